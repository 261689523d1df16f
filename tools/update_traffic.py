"""Summarise tools/profile_r2.sh's ncu counter captures (gpurun_out/r2_traffic_*.csv) into
profiles/kernel_traffic.json: per workload and kernel, DRAM bytes (read + write), L2 sectors and
L2 hit rate of one launch (the median launch of that kernel; for the replay kernel the median of
the full-trace launches, not the short drain launches). bench.py reads it for roofline.traffic.

    python tools/update_traffic.py [TAG]
"""
import csv
import json
import os
import statistics
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, PR = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
OUT = os.path.join(PR, "kernel_traffic.json")


def launches(path):
    rows = [r for r in csv.DictReader(line for line in open(path) if line.startswith('"'))]
    by = defaultdict(dict)
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
        by[(int(r["ID"]), name)][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return by


def summarise(recs):
    med = lambda k: statistics.median(m[k] for m in recs)  # noqa: E731
    rd, wr = med("dram__bytes_read.sum"), med("dram__bytes_write.sum")
    return {"dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
            "l2_sectors": int(med("lts__t_sectors.sum")), "l2_hit_pct": med("lts__t_sector_hit_rate.pct"),
            "launch_ns_under_ncu": int(med("gpu__time_duration.sum")), "launches_captured": len(recs)}


def main():
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for w in ("api64", "chat1024", "agent256", "large4096"):
        ent = out.get(w, {})
        for fname in (f"r2_traffic_{w}.csv", f"r2_traffic_whatif_{w}.csv"):
            p = os.path.join(G, fname)
            if not os.path.exists(p):
                continue
            per = defaultdict(list)
            for (_, name), m in sorted(launches(p).items()):
                per[name].append(m)
            for name, recs in per.items():
                if name == "replay_kernel":           # full replays, not the drain launches after them
                    longest = max(m["gpu__time_duration.sum"] for m in recs)
                    recs = [m for m in recs if m["gpu__time_duration.sum"] > 0.5 * longest]
                s = summarise(recs)
                s["source"] = (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,"
                               f"lts__t_sector_hit_rate.pct --clock-control none, python bench.py --workload {w} "
                               f"--steps 1 (tools/profile_r2.sh, {tag}); median of the captured launches")
                ent[name] = s
        if ent:
            out[w] = ent
    json.dump(out, open(OUT, "w"), indent=1)
    for w, ent in out.items():
        for k, v in ent.items():
            print(f"{w:10s} {k:20s} dram {v['dram_bytes'] / 1e6:10.1f} MB  L2 sectors {v['l2_sectors'] * 32 / 1e6:10.1f} MB"
                  f"  hit {v['l2_hit_pct']:5.1f} %")


if __name__ == "__main__":
    main()
