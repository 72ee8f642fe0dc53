import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2502_03749_b200 import pins
from workloads import make
w = make("c4_l1rect", scale=0.04)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    pb = pins.DeviceProblem.from_workload(w)
    r = pins.solve(pb, pins.default_params(K=K, outer_tol=0.0))
    print("obj", repr(r["obj"]), r["sweeps"], r["cg_iters"], flush=True)
