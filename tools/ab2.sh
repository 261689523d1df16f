#!/bin/bash
# Interleaved A/B of librsim builds: tools/ab2.sh "lib1 lib2 ..." "workload:n ..." [passes]
# (lib = a directory under build/variants holding librsim.so, or "cur" for the in-tree build)
cd "$(dirname "$0")/.."
for pass in $(seq ${3:-2}); do
  for w in $2; do
    IFS=: read name n <<< "$w"
    for v in $1; do
      if [ "$v" = cur ]; then L=paper_2603_15202_b200/librsim.so; else L=build/variants/$v/librsim.so; fi
      RSIM_LIB=$L timeout 200 python tools/profile_replay.py $name $n 2>&1 | grep "us/decision" | sed "s/ctas=0 warps=0: total [0-9.]* ms  replay [0-9.]* ms//; s/^/[$v p$pass] /"
    done
  done
done
