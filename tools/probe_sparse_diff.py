"""Dev probe: first outer iteration where the sparse-sweep path and the dense path differ."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2502_03749_b200 import pins
from workloads import make
w = make(sys.argv[1], scale=float(sys.argv[2]))
pb = pins.DeviceProblem.from_workload(w)
os.environ["PINS_TRACE"] = sys.argv[3]
r = pins.solve(pb, pins.default_params(K=int(sys.argv[4]), outer_tol=0.0), trace=True)
print(json.dumps({"trace": [float(x) for x in r["trace"]], "f": [float(x) for x in r["f"].cpu().numpy()[:5]]}))
'''
name, scale, K = sys.argv[1], sys.argv[2], sys.argv[3]
outs = []
for tag, env in (("dense", {"PINS_NO_SPARSE_SWEEP": "1"}), ("sparse", {})):
    e = dict(os.environ); e.update(env)
    r = subprocess.run([sys.executable, "-c", CHILD, name, scale, f"gpurun_out/trace_diff_{tag}.txt", K], env=e,
                       capture_output=True, text=True)
    print(tag, r.stderr[-500:])
    outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
for k, (a, b) in enumerate(zip(outs[0]["trace"], outs[1]["trace"])):
    print(k, a, b, "DIFF" if a != b else "")
for tag in ("dense", "sparse"):
    print(tag, open(f"gpurun_out/trace_diff_{tag}.txt").read())
