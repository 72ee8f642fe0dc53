"""Dev probe: device time of one sweep / eval / eval+sparsify per config (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_03749_b200 import pins
from workloads import make

for name in sys.argv[1:]:
    w = make(name)
    pb = pins.DeviceProblem.from_workload(w)
    phi, psi, s = pins.center_init(pb)
    f = torch.zeros(w.m, dtype=torch.float64, device="cuda"); g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    ws = pins.Workspace()
    for _ in range(20):
        pins.sinkhorn_sweep(ws, pb, phi, psi, s, f, g)
    torch.cuda.synchronize()
    def t(fn, k=20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k
    ts = t(lambda: pins.sinkhorn_sweep(ws, pb, phi, psi, s, f, g))
    te = t(lambda: pins.evaluate(ws, pb, phi, psi, s, f, g))
    tau = 1e-4 / (w.m * w.n)
    tsp = t(lambda: pins.evaluate(ws, pb, phi, psi, s, f, g, tau=tau))
    ev = pins.evaluate(ws, pb, phi, psi, s, f, g, tau=tau)
    print(f"{name}: sweep {ts:.3f} ms  eval {te:.3f} ms  eval+sparsify {tsp:.3f} ms  nnz {ev['nnz']} grad {ev['grad_l1']:.3e}", flush=True)
