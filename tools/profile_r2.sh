#!/bin/bash
# Round-2 counter pass: DRAM bytes + L2 sectors/hit rate of every kernel the bench line carries a
# roofline for (replay, K1, what-if probes), a few launches each; tools/update_traffic.py
# summarises them into profiles/kernel_traffic.json (read by bench.py for roofline.traffic).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for w in ${WORKLOADS:-api64 chat1024 agent256}; do
  timeout 600 ncu --metrics $M --clock-control none -c 6 -k regex:"replay_kernel|k1_chain_keys" \
    --csv --log-file gpurun_out/r2_traffic_$w.csv \
    python bench.py --workload $w --extra "" --route-api "" --steps 1 --warmup 0 --no-cpu --no-parity --whatif 0 > /dev/null 2> gpurun_out/r2_traffic_$w.err
  timeout 600 ncu --metrics $M --clock-control none -c 2 -k regex:"probe_scan_kernel" \
    --csv --log-file gpurun_out/r2_traffic_whatif_$w.csv \
    python bench.py --workload $w --extra "" --route-api "" --steps 1 --warmup 0 --no-cpu --no-parity > /dev/null 2> gpurun_out/r2_traffic_whatif_$w.err
done
ls -la gpurun_out/
