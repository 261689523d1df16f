#!/bin/bash
# Build librsim variants for A/B timing: tools/variants.sh name "-DFLAG=1 ..." ...
# Output: build/variants/<name>/librsim.so (select with RSIM_LIB=...).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p "$ROOT/build/variants/$name"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo -std=c++17 \
    -Xcompiler -fPIC -shared $flags -o "$ROOT/build/variants/$name/librsim.so" "$ROOT/paper_2603_15202_b200/csrc/rsim.cu" &
done
wait
