"""A/B of library env knobs on full solves (device time by CUDA events, profiler off).

    python tools/ab_env.py CONFIG REPS 'ENV1=..,ENV2=..' ['ENV=..' ...]
Each setting runs in its own process (the knobs are read once per process); prints one
JSON line per setting: median seconds, counts, accuracy."""
import json, os, subprocess, sys

CHILD = r'''
import json, os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2502_03749_b200 import pins
from workloads import make
name, reps = sys.argv[1], int(sys.argv[2])
w = make(name)
pb = pins.DeviceProblem.from_workload(w)
gold = json.load(open(f"tests/golden/exact_{name}.json"))["obj"]
prm = pins.default_params(K=200000, outer_rule=3, outer_tol=1e-7, newton_tol=1e-8)
ws = pins.Workspace()
ts = []
for r in range(reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    res = pins.solve(pb, prm, ws=ws)
    e1.record(); torch.cuda.synchronize()
    if r: ts.append(e0.elapsed_time(e1) / 1e3)
out = {k: res[k] for k in ("outer_iters", "sweeps", "newton_iters", "cg_iters", "kkt", "gap", "status")}
out["rel_err"] = abs(res["obj"] - gold) / gold
out["s_med"] = statistics.median(ts); out["s_all"] = ts
print(json.dumps(out))
'''
cfg, reps = sys.argv[1], sys.argv[2]
for setting in sys.argv[3:]:
    env = dict(os.environ)
    if setting != "-":
        for kv in setting.split(","):
            k, v = kv.split("=", 1)
            env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD, cfg, reps], env=env, capture_output=True, text=True)
    line = (r.stdout.strip().splitlines() or ["{}"])[-1]
    print(json.dumps({"setting": setting, "cfg": cfg, **json.loads(line)}) if r.returncode == 0
          else json.dumps({"setting": setting, "error": r.stderr[-800:]}), flush=True)
