"""Short, deterministic targets for `ncu --set full` (one kernel family per mode).

    python tools/ncu_target.py sweep|eval|cg|late [config]
sweep: 30 Sinkhorn sweeps from X^0 (lse_pass_kernel); eval: 10 evaluations with
sparsify (sum_pass_kernel); cg: a PINS solve capped at 10 outer iterations;
late: a PINS solve capped at 300 outer iterations (late-phase tree-PCG calls).
Inputs: the seeded workload.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_03749_b200 import pins
from workloads import make

mode = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "c3_gmm10k"
w = make(name)
pb = pins.DeviceProblem.from_workload(w)
if mode in ("sweep", "eval"):
    phi, psi, s = pins.center_init(pb)
    f = torch.zeros(w.m, dtype=torch.float64, device="cuda")
    g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    ws = pins.Workspace()
    # one device-side Sinkhorn phase (argmax seeds and chunk-skip certificates carry
    # across its sweeps, as inside pins_solve)
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, 30 if mode == "sweep" else 20)
    if mode == "eval":
        for _ in range(10):
            pins.evaluate(ws, pb, phi, psi, s, f, g, tau=1e-4 / (w.m * w.n))
else:
    K = 10 if mode == "cg" else 300
    r = pins.solve(pb, pins.default_params(K=K, outer_tol=0.0, newton_tol=1e-8))
torch.cuda.synchronize()
print("ok", mode, name)
