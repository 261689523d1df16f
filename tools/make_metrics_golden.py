"""Golden exports: the REFERENCE's run + metrics.export (metrics.py:399-497) on golden
cases, run in this container; records every file's sha256 and summary.json.

    python tools/make_metrics_golden.py    # writes tests/golden/metrics_exports.json
"""
import hashlib
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from make_golden import CASES, build_case  # noqa: E402
from refcompat import import_reference, to_ref_config, to_ref_records  # noqa: E402

NAMES = ["cfg1_chatbot_full", "det_hot_n16", "stale_5ms", "policy_simulate", "adv_out1", "cost_small_batch"]


def main():
    rs = import_reference()
    from routesim.metrics import export
    out = {}
    for name in NAMES:
        expr, prefix = CASES[name]
        trace, cfg = build_case(expr, prefix)
        rep = rs.run(to_ref_records(trace), to_ref_config(cfg))
        files = {}
        for rw in (False, True):
            with tempfile.TemporaryDirectory() as d:
                for p in export(rep, d, request_weighted_hits=rw):
                    files[f"{'rw/' if rw else ''}{os.path.basename(p)}"] = hashlib.sha256(open(p, "rb").read()).hexdigest()
                if not rw:
                    summary = open(os.path.join(d, "summary.json")).read()
        out[name] = {"files": files, "summary": summary}
        print(name, len(files), flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "metrics_exports.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
