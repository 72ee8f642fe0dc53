"""Dev probe: one full-size solve with the per-outer trace (PINS_TRACE) and the launch profile."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_03749_b200 import pins
from workloads import make

name, tag = sys.argv[1], sys.argv[2]
over = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
w = make(name)
pb = pins.DeviceProblem.from_workload(w)
gp = f"tests/golden/exact_{name}.json"
gold = json.load(open(gp))["obj"] if os.path.exists(gp) else None
prm = dict(K=20000, outer_rule=1, outer_tol=1e-7, newton_tol=1e-10); prm.update(over)
os.environ["PINS_TRACE"] = f"gpurun_out/trace_{name}_{tag}.txt"
pins.prof_reset(); pins.prof_enable(True)
r = pins.solve(pb, pins.default_params(**prm))
pins.prof_enable(False)
prof = pins.prof_read()
out = {k: v for k, v in r.items() if not torch.is_tensor(v) and v is not None}
out["rel_err"] = None if gold is None else abs(r["obj"] - gold) / gold
out["prof"] = prof
out["params"] = prm
print(json.dumps(out), flush=True)
