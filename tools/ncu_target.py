"""Short, deterministic targets for `ncu --set full` (one kernel family per mode).

    python tools/ncu_target.py sweep|eval|cg|late|dense|spmv|ksweep [config]
sweep: 30 Sinkhorn sweeps from X^0 in one device-side phase (lse_pass_kernel);
eval: 20 sweeps then 10 evaluations with sparsify (sum_pass_kernel); cg: a PINS
solve capped at 10 outer iterations; late: a PINS solve capped at 300 outer
iterations (late-phase tree-PCG calls); dense: c3's cost materialised densely
(10^4 x 10^4 fp64, 800 MB), 10 sweeps and 2 evaluations (TMA-staged dense
passes); spmv: the grid CG on a 2.4e7-entry support, 50 iterations.
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
if mode != "ksweep":
    os.environ["PINS_KSWEEP"] = "0"      # the dense passes themselves (long phases default to kernel-matrix sweeps)
if mode == "ksweep":
    # 600 sweeps of one phase from X^0: dense sweeps while the potentials churn, then
    # absorbed kernel-matrix sweeps (lse_ksweep_kernel + fallback + merge)
    pb = pins.DeviceProblem.from_workload(w)
    phi, psi, s = pins.center_init(pb)
    f = torch.zeros(w.m, dtype=torch.float64, device="cuda")
    g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    ws = pins.Workspace()
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, 600)
elif mode in ("sweep", "eval"):
    pb = pins.DeviceProblem.from_workload(w)
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
elif mode == "dense":
    X = torch.as_tensor(w.X, dtype=torch.float64, device="cuda")
    Y = torch.as_tensor(w.Y, dtype=torch.float64, device="cuda")
    C = ((X * X).sum(1)[:, None] + (Y * Y).sum(1)[None, :] - 2.0 * X @ Y.T) * w.cost_scale
    C.clamp_(min=0.0)
    a = torch.as_tensor(w.a, dtype=torch.float64, device="cuda")
    b = torch.as_tensor(w.b, dtype=torch.float64, device="cuda")
    pb = pins.DeviceProblem(w.m, w.n, 0, a, b, w.eta, C=C)
    phi, psi, s = pins.center_init(pb)
    f = torch.zeros(w.m, dtype=torch.float64, device="cuda")
    g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    ws = pins.Workspace()
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, 10)
    pins.evaluate(ws, pb, phi, psi, s, f, g, tau=0.0)
    pins.evaluate(ws, pb, phi, psi, s, f, g, tau=1e-4 / (w.m * w.n))
elif mode == "spmv":
    m = n = 10000
    nnz_row = 2400
    gen = torch.Generator(device="cuda").manual_seed(7)
    cols = torch.rand(m, n, device="cuda", generator=gen).topk(nnz_row, dim=1).indices.sort(dim=1).values
    colidx = cols.reshape(-1).to(torch.int32)
    rowptr = torch.arange(0, m * nnz_row + 1, nnz_row, device="cuda", dtype=torch.int64)
    val = torch.rand(m * nnz_row, device="cuda", generator=gen, dtype=torch.float64) / (m * n)
    dr = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(
        0, torch.arange(m, device="cuda").repeat_interleave(nnz_row), val) * 1.5
    dc = torch.zeros(n, dtype=torch.float64, device="cuda").index_add_(0, colidx.long(), val) * 1.5
    rhs = torch.rand(m + n, device="cuda", generator=gen, dtype=torch.float64)
    ws = pins.Workspace()
    pins.cg(ws, m, n, rowptr, colidx, val, dr, dc, 1e-12, rhs, rtol=0.0, maxit=50)
else:
    pb = pins.DeviceProblem.from_workload(w)
    K = 10 if mode == "cg" else 300
    r = pins.solve(pb, pins.default_params(K=K, outer_tol=0.0, newton_tol=1e-8))
torch.cuda.synchronize()
print("ok", mode, name)
