"""Summarise a round's ncu captures (gpurun_out/) into profiles/ (tracked).

    python tools/update_profiles.py TAG     # TAG: kernel version label, e.g. v30
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, PR = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1]

rows = [r for r in csv.reader(open(os.path.join(G, f"r1_launches_bench_{tag}.csv"))) if len(r) > 10]
hdr = rows[0]
d = defaultdict(list)
for r in rows[1:]:
    d[r[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "")].append(float(r[-1]))
tot = sum(sum(v) for v in d.values())
out = [f"ncu launch list of `python bench.py --steps 3 --warmup 3 --no-cpu` (api64 headline + chat1024 extra), kernel {tag},",
       "--metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised per-launch times (shares, not absolutes)",
       f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'mean ms':>10s} {'share':>7s}"]
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    out.append(f"{k[:28]:28s} {len(v):8d} {sum(v) / 1e6:10.2f} {sum(v) / len(v) / 1e6:10.3f} {100 * sum(v) / tot:6.2f}%")
open(os.path.join(PR, "r1_launches_bench_summary.txt"), "w").write("\n".join(out) + "\n")
os.replace(os.path.join(G, f"r1_launches_bench_{tag}.csv"), os.path.join(PR, "r1_launches_bench.csv"))

tr = {}
for w in ("api64", "chat1024"):
    rr = [r for r in csv.reader(open(os.path.join(G, f"r1_traffic_{w}.csv"))) if len(r) > 10]
    m = {r[-3]: float(r[-1]) for r in rr[1:]}
    tr[w] = {"dram_bytes": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
             "dram_read": int(m["dram__bytes_read.sum"]), "dram_write": int(m["dram__bytes_write.sum"]),
             "l2_hit_pct": m["lts__t_sector_hit_rate.pct"], "launch_ns_under_ncu": int(m["gpu__time_duration.sum"]),
             "kernel": tag,
             "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:replay_kernel -c 1 "
                       f"python bench.py --workload {w} --steps 1 (first replay launch)"}
json.dump(tr, open(os.path.join(PR, "replay_traffic.json"), "w"), indent=1)

rep = os.path.join(G, f"prof_api64_{tag}.ncu-rep")
hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "40"], capture_output=True, text=True).stdout
open(os.path.join(PR, "r1_ncu_replay_api64_hotlines.txt"), "w").write(
    f"ncu --set full --import-source on, replay_kernel, api64 5,000-request slice, C=16 W=4, kernel {tag}\n" + hot)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
lines = [f"ncu --set full metrics, replay_kernel, api64 5,000-request slice, kernel {tag}"]
if len(rows) > 2:
    h, unit, val = rows[0], rows[1], rows[2]
    for w in want:
        if w in h:
            lines.append(f"{w:62s} {val[h.index(w)]:>16s} {unit[h.index(w)]}")
open(os.path.join(PR, "r1_ncu_replay_api64_metrics.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(out)); print(json.dumps(tr, indent=1)); print("\n".join(lines))
