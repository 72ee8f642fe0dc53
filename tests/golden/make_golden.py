"""Write tests/golden/exact_<config>.json: the exact LP optimum of each BASELINE
config, computed ONLY by oracle/ (network simplex on the dense cost built by
oracle.pins_oracle.cost_matrix) from the seeded generators in workloads/.

    python tests/golden/make_golden.py [config ...]

Each file records obj, the certificate (duality gap, min reduced cost, marginal
error), pivots and wall time.  Nothing here comes from the CUDA path.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.exact_lp import solve_exact  # noqa: E402
from oracle.pins_oracle import cost_matrix  # noqa: E402
from workloads import config_names, make  # noqa: E402


def main(names):
    for name in names:
        t0 = time.time()
        w = make(name)
        C = cost_matrix(w)
        r = solve_exact(C, w.a, w.b)
        X = r["X"]
        marg = float(np.abs(X.sum(1) - w.a).sum() + np.abs(X.sum(0) - w.b).sum())
        out = dict(config=name, m=w.m, n=w.n, obj=r["obj"],
                   dual_obj=float(w.a @ r["u"] + w.b @ r["v"]),
                   min_reduced_cost=r["min_rc"], marginal_l1=marg,
                   support=int((X > 0).sum()), pivots=r["pivots"],
                   seconds=time.time() - t0, source="oracle/netsimplex.c via tests/golden/make_golden.py")
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"exact_{name}.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or config_names())
