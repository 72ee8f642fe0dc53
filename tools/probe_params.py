"""probe: c3 solve time / counts under parameter variants (certified stop)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_03749_b200 import pins as P
from workloads import make
name = sys.argv[1] if len(sys.argv) > 1 else "c3_gmm10k"
w = make(name)
gold = json.load(open(f"tests/golden/exact_{name}.json"))["obj"]
pb = P.DeviceProblem.from_workload(w)
ws = P.Workspace()
base = dict(K=200000, outer_rule=3, outer_tol=1e-7, newton_tol=1e-8)
variants = [{}, {"cg_forcing": 0.3}, {"cg_forcing": 0.5}, {"warm_start": 2}, {"warm_start": 2, "cg_forcing": 0.3}]
P.solve(pb, P.default_params(**base), ws=ws)
for v in variants:
    prm = P.default_params(**base, **v)
    ts = []
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        r = P.solve(pb, prm, ws=ws)
        torch.cuda.synchronize(); ts.append(time.time() - t0)
    print(json.dumps({"variant": v, "sec": min(ts), "outer": r["outer_iters"], "newton": r["newton_iters"],
                      "cg": r["cg_iters"], "sweeps": r["sweeps"], "status": r["status"],
                      "relerr": abs(r["obj"] - gold) / gold, "gap": r["gap"]}), flush=True)
