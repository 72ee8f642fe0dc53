"""probe: certified stop on the full-size configs, with the certificate trace."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
from paper_2502_03749_b200 import pins as P
from workloads import make
os.environ["PINS_CERT_TRACE"] = "1"
names = sys.argv[1:] or ["c2_img4k", "c1_rand1k"]
for name in names:
    w = make(name)
    gold = json.load(open(f"tests/golden/exact_{name}.json"))["obj"]
    pb = P.DeviceProblem.from_workload(w)
    torch.cuda.synchronize()
    t0 = time.time()
    r = P.solve(pb, P.default_params(K=200000, outer_rule=3, outer_tol=1e-7, newton_tol=1e-8))
    torch.cuda.synchronize()
    print(name, "sec", time.time() - t0, {k: r[k] for k in ("status", "outer_iters", "obj", "kkt", "gap", "lp_dual_obj", "dual_inf", "certificates", "cert_tree")},
          "relerr", abs(r["obj"] - gold) / gold, flush=True)
