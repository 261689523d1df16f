#!/bin/bash
# Snapshot the current csrc as a named variant and build it: tools/variant_src.sh name ["-DFLAGS"]
# -> build/variants/<name>/librsim.so (time with RSIM_LIB=..., tools/ab.sh)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; flags=${2:-}
V="$ROOT/build/variants/$name"
mkdir -p "$V/pkg/csrc" "$V/include"
cp "$ROOT"/paper_2603_15202_b200/csrc/*.cu* "$V/pkg/csrc/"
cp "$ROOT"/include/*.h "$V/include/"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared $flags -o "$V/librsim.so" "$V/pkg/csrc/rsim.cu"
