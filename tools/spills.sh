#!/bin/bash
# Per-kernel registers / stack / spills of librsim (ptxas -v): tools/spills.sh [extra nvcc flags]
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared \
  -Xptxas -v "$@" -o /tmp/spills_$$.so paper_2603_15202_b200/csrc/rsim.cu 2>&1 | python3 -c '
import sys, re
fn = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function .(\S+).", line) or re.search(r"Function properties for (\S+)", line)
    if m: fn = m.group(1)
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and fn and int(m.group(2)): print(f"{fn[:60]:60s} stack {m.group(1):>5s} spill st {m.group(2):>5s} ld {m.group(3):>5s}")
    m = re.search(r"Used (\d+) registers", line)
    if m and fn and "replay" in fn: print(f"{fn[:60]:60s} regs {m.group(1)}")
'
rm -f /tmp/spills_$$.so
