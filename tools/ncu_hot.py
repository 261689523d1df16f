"""Summarise an ncu report's source page: stall reasons overall and hottest lines.

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, lines = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] == "Function Name" or hdr is None or len(r) < len(hdr):
        continue
    if r[2] == "-":
        d = dict(zip(hdr[2:], r[2:]))
        lines.append((cur, r[0], r[1].strip()[:70], d))
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
for _, _, _, d in lines:
    for c in stall_cols:
        tot[c] += int(d.get(c) or 0)
S = sum(tot.values())
print(f"total stall samples {S}")
for c, v in tot.most_common(10):
    print(f"  {c:24s} {v:7d} {100 * v / max(S, 1):5.1f}%")
print(f"\ntop {top} lines by samples (file:line samples instr | top reasons)")
key = lambda x: -int(x[3].get("Warp Stall Sampling (All Samples)") or 0)
for f, ln, src, d in sorted(lines, key=key)[:top]:
    s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    ins = int(d.get("Instructions Executed") or 0)
    rs = sorted(((int(d.get(c) or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{f}:{ln:<5s}{s:6d} {ins:9d} | {' '.join(f'{n}={v}' for v, n in rs if v)}  {src}")
