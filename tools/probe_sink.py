"""probe: pins_sinkhorn final residual vs a fresh evaluation (chunk-skip check)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_03749_b200 import pins as P
from oracle import pins_oracle as po
from workloads import make

def T(x):
    return torch.as_tensor(np.asarray(x), dtype=torch.float64, device="cuda").contiguous()

for name, sc in [("c4_l1rect", 0.012), ("c3_gmm10k", 0.013), ("c4_l1rect_r", 0.012)]:
    w = make(name, scale=sc)
    C = po.cost_matrix(w)
    r = po.pins(C, w.a, w.b, po.Params(eta=w.eta, K=2, outer_tol=0.0, newton_tol=1e-10))
    f = r.f + np.random.default_rng(5).normal(0, 2 * w.eta, w.m)
    for noskip in (0, 1):
        if noskip:
            os.environ["PINS_NO_TILESKIP"] = "1"
        else:
            os.environ.pop("PINS_NO_TILESKIP", None)
        pb = P.DeviceProblem.from_workload(w)
        ws = P.Workspace()
        fd, gd = T(f), T(r.g)
        t, res = P.sinkhorn(ws, pb, T(r.phi), T(r.psi), r.s_next, fd, gd, 1e-6, 5000)
        ev = P.evaluate(P.Workspace(), pb, T(r.phi), T(r.psi), r.s_next, fd, gd)
        Ck = po.shifted_cost(C, r.logX, w.eta)
        ro = po.residual_l1(fd.cpu().numpy(), gd.cpu().numpy(), Ck, w.a, w.b, w.eta)
        print(name, "noskip", noskip, "sweeps", t, "res(phase)", res, "res(fresh eval)", ev["grad_l1"], "oracle res of gpu state", ro, flush=True)
