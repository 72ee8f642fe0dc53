"""Dev probe: per-class device time of repeated evaluate(tau) calls (library event profile)."""
import os, sys, time
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
    tau = 1e-4 / (w.m * w.n)
    for rep in range(3):
        pins.prof_reset(); pins.prof_enable(True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(10):
            pins.evaluate(ws, pb, phi, psi, s, f, g, tau=tau)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        pins.prof_enable(False)
        pr = pins.prof_read()
        print(name, rep, f"wall {1e3*(t1-t0)/10:.3f} ms/call", {k: (v['launches'], round(v['ms'], 3)) for k, v in pr.items() if v['launches']}, flush=True)
