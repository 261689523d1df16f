#!/bin/bash
# Round-2 measurement pass: bench line, ncu launch list of the bench, per-kernel DRAM/L2 counters
# (tools/profile_r2.sh), one --set full capture of the replay kernel (api64 slice) and of the
# what-if probe (chat1024). Summarise with tools/update_traffic.py + tools/ncu_hot.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --route-api "" --extra chat1024 > /dev/null 2>&1
bash tools/profile_r2.sh > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -f \
  -o gpurun_out/r2_prof_api64 python tools/profile_replay.py api64 5000 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:probe_scan_kernel -c 1 -f \
  -o gpurun_out/r2_prof_whatif_chat1024 python bench.py --workload chat1024 --extra "" --route-api "" --steps 1 --warmup 3 --no-cpu --no-parity > /dev/null 2>&1
ls -la gpurun_out/
