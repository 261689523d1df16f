"""Print the first mismatching request of a stateful API session vs the reference golden."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import make_api_golden as M
from paper_2603_15202_b200 import workloads as W
from paper_2603_15202_b200.cluster import ClusterSim
from paper_2603_15202_b200.config import DuplicateRequestError
name = sys.argv[1]
want = json.load(open(os.path.join(ROOT, "tests", "golden", "api_sessions.json")))[name]
cfg, steps = M.SESSIONS[name]
trace = W.config1_chatbot()[0].slice(600)
got = json.loads(json.dumps(M.run_session(cfg, steps, trace, (ClusterSim, lambda t: t.records(), DuplicateRequestError))))
for i, (g, w) in enumerate(zip(got, want)):
    if g == w:
        continue
    print("step", i, steps[i])
    if g[0] == "run":
        for j, (a, b) in enumerate(zip(g[1], w[1])):
            if a != b:
                print(" first request mismatch", j, "got", a, "want", b)
                print(" next:", [(x, y) for x, y in zip(g[1][j:j+6], w[1][j:j+6])])
                break
        print(" hash", g[2] == w[2], "nsteps", g[3], w[3], "queued", g[4], w[4], "end", g[5], w[5])
    else:
        print(" got", str(g)[:400]); print(" want", str(w)[:400])
    break
else:
    print("all equal")
