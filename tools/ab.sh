#!/bin/bash
# A/B timing of librsim variants: tools/ab.sh "variant..." "workload:n:ctas:warps ..."
cd "$(dirname "$0")/.."
for v in $1; do
  for w in $2; do
    IFS=: read name n c wp <<< "$w"
    RSIM_LIB=build/variants/$v/librsim.so timeout 120 python tools/profile_replay.py $name $n $c $wp 2>&1 | sed "s/^/[$v] /"
  done
done
