"""Print the key numbers of a bench.py JSON line: python tools/summ.py FILE"""
import json
import sys

l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])


def s(d, name):
    e = d['e2e'] if not isinstance(d['e2e'], dict) else d['e2e']['value']
    print(f"{name:10s} value {d['value']:9.0f} e2e {e:9.0f} lat {d.get('decision_latency_us', {}).get('p50')}/"
          f"{d.get('decision_latency_us', {}).get('p99')} parity {(d.get('parity') or {}).get('mismatches')} "
          f"roof {d['roofline']['frac']:.2e} traffic {d['roofline'].get('traffic')}")
    w = d.get('whatif_probe') or {}
    print(f"   whatif {w.get('roofline', {}).get('frac')} traffic {w.get('roofline', {}).get('traffic')} "
          f"k1 {d['k1_chain_keys']['roofline']['frac']:.3f} traffic {d['k1_chain_keys']['roofline'].get('traffic')}")


s(l, l['config']['workload'])
for k, v in (l.get('extra_workloads') or {}).items():
    s(v, k)
print('clocks', l['clocks'], 'launches', l['gpu_launches'], 'cpu', l.get('cpu_baseline', {}).get('value'),
      'port', l.get('cpu_port', {}).get('value'))
for r in l.get('route_api') or []:
    print('route', r['workload'], r['instances'], 'c_abi', round(r['c_abi']['p50_us'], 1), 'ours',
          round(r['ours']['p50_us'], 1), round(r['ours']['p99_us'], 1), 'ref',
          round(r.get('reference', {}).get('p50_us', 0), 1), r.get('parity'))
