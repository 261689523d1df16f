#!/bin/bash
# One round's measurement pass on the GPU box (tools/update_profiles.py TAG summarises it):
# bench line, ncu launch list of the bench, replay-kernel DRAM traffic, one --set full capture.
TAG=${1:-v31}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r1_launches_bench_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
for w in api64 chat1024; do
  timeout 400 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    -k regex:replay_kernel -c 1 --csv --log-file gpurun_out/r1_traffic_$w.csv \
    python bench.py --workload $w --extra "" --steps 1 --no-cpu > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -f \
  -o gpurun_out/prof_api64_$TAG python tools/profile_replay.py api64 5000 16 4 > /dev/null 2>&1
ls -la gpurun_out/
