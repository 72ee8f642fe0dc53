"""Dev probe: full-size pins_solve per config + per-call timings (not a bench)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_03749_b200 import pins
from workloads import make

name = sys.argv[1]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
w = make(name)
pb = pins.DeviceProblem.from_workload(w)
gold = None
gp = f"tests/golden/exact_{name}.json"
if os.path.exists(gp):
    gold = json.load(open(gp))["obj"]
# per-call timing
phi, psi, s = pins.center_init(pb)
f = torch.zeros(w.m, dtype=torch.float64, device="cuda"); g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
ws = pins.Workspace()
for _ in range(3):
    pins.sinkhorn_sweep(ws, pb, phi, psi, s, f, g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10):
    pins.sinkhorn_sweep(ws, pb, phi, psi, s, f, g)
e1.record(); torch.cuda.synchronize()
print(f"{name}: sweep {e0.elapsed_time(e1)/10:.3f} ms", flush=True)
t0 = time.time()
for _ in range(10):
    ev = pins.evaluate(ws, pb, phi, psi, s, f, g, tau=1e-4 / (w.m * w.n))
torch.cuda.synchronize()
print(f"{name}: eval+sparsify {(time.time()-t0)/10*1e3:.3f} ms nnz {ev['nnz']} grad {ev['grad_l1']:.3e}", flush=True)
prm = pins.default_params(K=K, outer_rule=1, outer_tol=1e-7, newton_tol=1e-10)
r = pins.solve(pb, prm, trace=True)
tr = r.pop("trace")
out = {k: v for k, v in r.items() if not torch.is_tensor(v) and v is not None}
out["rel_err"] = None if gold is None else abs(r["obj"] - gold) / gold
out["trace_tail"] = tr[-3:]
out["trace_sel"] = [tr[i] for i in range(0, len(tr), max(1, len(tr)//10))]
print(name, json.dumps(out), flush=True)
