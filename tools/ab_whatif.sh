# what-if probe timing (bench's whatif_probe leg), two runs
for v in 1 2; do
  timeout 300 python bench.py --no-cpu --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for n,w in (('api64',d['whatif_probe']),('chat1024',d['extra_workloads']['chat1024']['whatif_probe'])): print(n, w['roofline']['kernel'], round(w['ms'],3), 'ms', round(w['roofline']['frac']*100,2), '%')"
done
