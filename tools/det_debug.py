"""Diagnostics: first decision where the device detector and the oracle disagree.

    RSIM_DET_DEBUG=1 python tools/det_debug.py <golden case>
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_cases as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2603_15202_b200.cluster import ClusterSim  # noqa: E402

name = sys.argv[1]
if name.startswith("random:"):                 # random:<seed>:<trial> of the random detector sweep
    _, sd, tr_i = name.split(":")
    trace, cfg = G.random_detector_case(int(sd), int(tr_i))
    print(cfg)
else:
    trace, cfg = G.build(name)
n = len(trace)
N = cfg.n_instances
ob = np.full((n, 8 + N), -1, np.int64)
O.lib().orc_set_det_debug.argtypes = [C.c_void_p]
O.lib().orc_set_det_debug(ob.ctypes.data)
ref = O.run_oracle(trace, cfg)
O.lib().orc_set_det_debug(None)
sim = ClusterSim(cfg)
rep = sim.run_trace(trace)
db = np.full((n, 8 + N), -1, np.int64)
h = sim._handle
h._L.rsim_detector_debug(h._h, db.ctypes.data, n)
cols = ["code", "nh", "pmin", "psum", "hit_tok", "prod_c", "held_c"]
bad = np.nonzero((db[:, :7] != ob[:, :7]).any(1) | (rep.chosen != ref.chosen))[0]
print(name, "requests", n, "mismatching", len(bad))
for i in bad[:6]:
    print(f"k={i} t={trace.arrival_us[i]} chosen dev {rep.chosen[i]} ref {ref.chosen[i]}")
    print("   dev", dict(zip(cols, db[i, :7].tolist())), "nl", db[i, 7])
    print("   ref", dict(zip(cols, ob[i, :7].tolist())))
    d = np.nonzero(db[i, 8:] != ob[i, 8:])[0]
    print("   products differ at instances", d.tolist(), "dev", db[i, 8 + d].tolist(), "ref", ob[i, 8 + d].tolist())
