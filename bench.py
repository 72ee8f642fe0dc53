"""bench.py -- PINS on B200: seconds to KKT <= 1e-8 on BASELINE.json's n=10k config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3_gmm10k] [--no-cpu-baseline] [--quick]

A *step* is one complete pins_solve (Algorithm 2 of PAPER.md: every EPPA outer
iteration with its Sinkhorn sweeps, sparse-Newton/CG steps, line searches and
proximal-centre updates, plus the LP certificates of the certified outer stop)
on the seeded synthetic workload `--config` (default c3_gmm10k: m = n = 10000
points of an 8-component Gaussian mixture in R^10 on a 1/64 lattice,
squared-Euclidean cost recomputed on the fly, eta = 1e-3).
Inputs are resident in HBM when the timed region starts.  Parameters: PAPER.md
A.2 defaults with the certified outer stop (reading R11): primal residual
<= 1e-8 and certified LP gap <= 1e-7 |obj|; every step is also checked against
the exact LP optimum (tests/golden, written by the oracle's network simplex).

value  = max-over-ranks device time of the K timed steps / (K * N): seconds
         per solve at whole-job throughput (N ranks solve independent copies:
         replicas, no collective on the data path, "scaling": "weak").  The
         library's event profiler is OFF in the timed region.
e2e    = the same through pins_solve_host: instance copied from pinned host
         memory and the certified LP duals (u, v) copied back inside the timed
         region.
roofline = dominant kernel class of 2 extra PROFILED steps (pins_prof_*: CUDA
         events on the launching stream around every library launch); its
         bound and algorithmic work per launch are in DESIGN.md §7.
configs = one line per other BASELINE config (and the real-valued variants):
         device seconds to the same certified stop, accuracy vs the exact LP,
         Sinkhorn sweeps/s and half-sweep throughput, CG SpMV GB/s.
hbm    = the two HBM-bound kernels at HBM scale: the dense-cost half-sweep
         and sum pass on c3's cost materialised as a 10^4 x 10^4 fp64 C (800 MB),
         and the grid CG's SpMV on a 2.4e7-entry sparsified support.
cpu_baseline = the fp64 oracle (oracle/pins_oracle.py) as it stands: a
         measured complete oracle solve of small instances (c0, c1 at 1/4
         scale) beside the same solves on the GPU, and the c3 estimate from
         per-operation oracle times at full size scaled by this run's counts.

`--impl reference` runs only the oracle leg (rank 0; other ranks exit 0) and
prints the same JSON line with "impl": "reference"; its operation counts come
from the committed work profile profiles/workprofile_<config>.json (written by
this script's own arm from a measured GPU solve).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# PAPER.md A.2 (lines 477-485) defaults (newton_tol 1e-8, T1, T2, ...) except the outer stop:
# the certified rule (reading R11): certified LP gap <= 1e-7 |obj| (BASELINE.json's 1e-7 bar)
BENCH_PARAMS = dict(K=200000, outer_rule=3, outer_tol=1e-7, newton_tol=1e-8)
# the other BASELINE configurations (and the real-valued point variants), one line each
CONFIG_LINES = ["c0_pts64", "c1_rand1k", "c2_img4k", "c4_l1rect", "c0_pts64_r", "c3_gmm10k_r", "c4_l1rect_r"]
PROFILED_STEPS = 2
KKT_TARGET = 1e-8
OBJ_RTOL = 1e-7


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3_gmm10k")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=25.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--quick", action="store_true", help="skip the per-config and HBM-scale sections")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ work model
# SIMT work model of the dense passes over point costs: per entry the
# branch-free phase 1 of a chunk (x.y on the tensor cores, then FADD + FFMA for D, FFMA
# for the test value, FSETP + LOP3 for the survivor mask, FMNMX for the chunk maximum) is
# I1 issue slots; per SURVIVOR (entry evaluated exactly) the fp64 exponential and its
# accumulation cost I2 issue slots, F2 of them on the FP64 pipe (half the FP32 rate on
# B200: 64 lanes/clk/SM).  Survivors are counted on the device (pins_prof_read_work).
SWEEP_CLASSES = ("sweep_row", "sweep_col", "ksweep", "sweep_aux")
ALU_MODEL = {"sweep_row": dict(I1=6, I2=24, F2=16), "eval": dict(I1=6, I2=30, F2=19)}


def kernel_roofline(cls: str, w, launches: int, ms: float, clocks_mhz: float, peaks: dict,
                    work: float = 0.0) -> dict:
    """Roofline entry for one kernel class (DESIGN.md §7 gives every number used here).

    sweep_row / eval (dense passes over the m x n block; m*n entries per half-sweep,
    2*m*n per sum pass, both orientations in one launch):
      dense cost -> "hbm": 8 B of C read per entry and pass, peak = measured HBM copy GB/s.
      point cost -> "alu": t_min = max((I1 E + I2 S) / issue, F2 S / fp64) with E entries,
                    S measured survivors, issue = 148 SM x 128 lanes x clock, fp64 = 148 SM x
                    64 lanes x clock; achieved / peak in entries/s at that survivor fraction.
    cg (the Newton-system solvers, one launch per system): "hbm" bytes = per iteration
      (CSR + CSC: 2 x 12 B x nnz) + 10 vectors x 8 B x (m + n), x iterations; peak = HBM.
      Its working set is on chip (L2 / shared memory), so this fraction shows how
      latency-bound the iteration is, not a traffic limit."""
    avg_s = ms / max(1, launches) / 1e3
    src = "measured" if "hbm_gbs" in peaks else "fallback"
    if cls in ("sweep_row", "eval"):
        mult = 1.0 if cls == "sweep_row" else 2.0
        entries = mult * float(w.m) * float(w.n)
        if w.kind == 0:
            ach = 8.0 * entries / avg_s / 1e9
            peak = peaks.get("hbm_gbs", 6650.0)
            return {"kernel": cls, "bound": "hbm", "unit": "GB/s", "achieved": ach, "peak": peak,
                    "frac": ach / peak, "work_per_launch": f"{8 * entries:.3g} B (8 B/entry)",
                    "peak_source": f"{src} HBM copy"}
        md = ALU_MODEL[cls]
        surv = work / max(1, launches)
        f = clocks_mhz * 1e6
        t_min = max((md["I1"] * entries + md["I2"] * surv) / (148 * 128 * f), md["F2"] * surv / (148 * 64 * f))
        ach = entries / avg_s / 1e9
        peak = entries / t_min / 1e9
        return {"kernel": cls, "bound": "alu", "unit": "Gentries/s", "achieved": ach, "peak": peak,
                "frac": ach / peak, "work_per_launch": f"{entries:.3g} entries, {surv:.3g} survivors "
                f"({surv / entries:.3f})",
                "peak_source": f"derived (DESIGN.md §7): I1={md['I1']}, I2={md['I2']}, F2={md['F2']} per "
                               f"entry / survivor, 148 SM x 128 issue lanes (64 FP64) x {clocks_mhz:.0f} MHz"}
    if cls == "ksweep":
        # absorbed kernel-matrix half-sweep (ELL walk): streams 12 B per listed entry
        # (int32 column + fp64 kernel value); `work` = entries walked, counted on the device
        byts = 12.0 * work / max(1, launches)
        ach = byts / avg_s / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        return {"kernel": cls, "bound": "hbm", "unit": "GB/s", "achieved": ach, "peak": peak, "frac": ach / peak,
                "work_per_launch": f"{byts:.3g} B (12 B x {work / max(1, launches):.3g} listed entries)",
                "peak_source": f"{src} HBM copy"}
    if cls == "cg":
        byts = work / max(1, launches)
        ach = byts / avg_s / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        return {"kernel": cls, "bound": "hbm", "unit": "GB/s", "achieved": ach, "peak": peak, "frac": ach / peak,
                "work_per_launch": f"{byts:.3g} B (library-counted: 24 B x nnz + 80 B x (m+n) per CG iteration)",
                "peak_source": f"{src} HBM copy (working set on chip: latency-bound)"}
    return {"kernel": cls}


# ------------------------------------------------------------ cpu baseline
def oracle_rates(w, budget_s: float, cg_per_newton: float):
    """Time the oracle's own operations, as they stand, on the FULL instance at
    the first subproblem (k = 0, X^0 = a b^T): one Sinkhorn sweep, one residual
    evaluation, and one Newton direction with 10 and with 60 CG iterations (the
    difference gives the per-CG-iteration cost), plus one line-search trial.
    Returns seconds per operation."""
    import numpy as np
    from oracle import pins_oracle as po
    t0 = time.time()
    C = po.cost_matrix(w)
    t_cost = time.time() - t0
    logX0 = np.log(w.a)[:, None] + np.log(w.b)[None, :]
    Ck = po.shifted_cost(C, logX0, w.eta)
    f = np.zeros(w.m)
    g = np.zeros(w.n)
    t0 = time.time()
    f, g = po.sinkhorn_sweep(f, g, Ck, w.a, w.b, w.eta)
    t_sweep = time.time() - t0
    t0 = time.time()
    po.residual_l1(f, g, Ck, w.a, w.b, w.eta)
    t_eval = time.time() - t0
    spent = t_cost + t_sweep + t_eval
    out = dict(sweep=t_sweep, eval=t_eval, cost=t_cost)
    if spent + 6 * t_eval < budget_s:
        ts = []
        for its in (10, 60):
            prm = po.Params(eta=w.eta, cg_tol=0.0, cg_forcing=0.0, cg_maxit=its)
            t0 = time.time()
            df, dg, _ = po.newton_direction(f, g, Ck, w.a, w.b, w.eta, prm)
            ts.append(time.time() - t0)
        per_it = max(0.0, (ts[1] - ts[0]) / 50.0)
        t0 = time.time()
        po.dual_increase(f, g, df, dg, 1.0, Ck, w.a, w.b, w.eta)
        t_ls = time.time() - t0
        out["newton"] = max(0.0, ts[0] - 10 * per_it) + per_it * cg_per_newton + t_ls
        out["cg_it"] = per_it
    else:
        out["newton"] = 4 * t_eval      # plan + sparsify + one line-search trial, lower bound
        out["cg_it"] = None
    return out


def cpu_baseline(w, counts: dict, budget_s: float, cores: int):
    outer, sweeps, newton = counts["outer_iters"], counts["sweeps"], counts["newton_iters"]
    cgpn = counts["cg_iters"] / max(1, newton)
    r = oracle_rates(w, budget_s, cgpn)
    # oracle PINS per outer iteration: one residual (+ the objective), per sweep a
    # sweep + a residual, per Newton step a step + a residual
    est = outer * 2 * r["eval"] + sweeps * (r["sweep"] + r["eval"]) + newton * (r["newton"] + r["eval"])
    cg_txt = f", {r['cg_it'] * 1e3:.1f} ms per CG iteration" if r.get("cg_it") is not None else ""
    sample = (f"oracle fp64 numpy, full {w.m}x{w.n} instance at k=0: one Sinkhorn sweep "
              f"{r['sweep']:.2f}s, one residual {r['eval']:.2f}s, one Newton step {r['newton']:.2f}s"
              f"{cg_txt}; scaled by this solve's {outer} outer / {sweeps} sweeps / {newton} Newton steps "
              f"/ {cgpn:.0f} CG iterations per Newton step")
    return {"value": est, "unit": "s", "cores": cores, "kind": "oracle", "sample": sample}


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info()]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ multi-GPU
def max_over_ranks(local: float, world: int, device: str) -> float:
    """Device time of the job = the slowest rank's (timing rule: max over ranks)."""
    if world <= 1:
        return float(local)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(local)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def per_solve_value(total_s: float, steps: int, world: int) -> float:
    """Whole-job seconds per solve: N replicas each solve `steps` independent problems
    in total_s (max over ranks), so the job delivers steps * N solves in total_s."""
    return total_s / (steps * world)


# ------------------------------------------------------------------ main
def run_reference(args, rank):
    if rank != 0:
        return
    from workloads import make
    w = make(args.config)
    prof_path = os.path.join(ROOT, "profiles", f"workprofile_{args.config}.json")
    if not os.path.exists(prof_path):
        print(json.dumps({"impl": "reference", "unavailable": f"no work profile {prof_path}"}))
        return
    counts = json.load(open(prof_path))["counts"]
    cores = blas_threads()
    vals = []
    for _ in range(args.warmup):
        pass   # the oracle has no warm state; warm-up steps are not repeated
    for _ in range(args.steps):
        vals.append(cpu_baseline(w, counts, args.cpu_budget, cores))
    v = statistics.median([x["value"] for x in vals])
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": "s to KKT<1e-8 (n=10k, c3_gmm10k)", "value": v, "unit": "s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "m": w.m, "n": w.n, "eta": w.eta},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def golden_obj(name):
    p = os.path.join(ROOT, "tests", "golden", f"exact_{name}.json")
    return json.load(open(p))["obj"] if os.path.exists(p) else None


def check_solve(r, gold, name):
    ok = (r["status"] == 0 and r["kkt"] <= KKT_TARGET and r["gap"] <= OBJ_RTOL * abs(r["obj"])
          and (gold is None or abs(r["obj"] - gold) <= OBJ_RTOL * abs(gold)))
    if not ok:
        raise SystemExit(f"{name}: solve failed the accuracy bar: status {r['status']} kkt {r['kkt']:.3e} "
                         f"gap {r['gap']:.3e} obj {r['obj']!r} exact {gold!r}")


def prof_stats(pins, w, prof, clocks_mhz, peaks, steps):
    """Per-class device time, launches, and roofline entries of a profiled region."""
    total_ms = sum(v["ms"] for v in prof.values())
    kerns = {}
    for c in ("sweep_row", "sweep_col", "ksweep", "eval", "cg"):
        if prof[c]["launches"] and prof[c]["ms"] > 0:
            cls = "sweep_row" if c == "sweep_col" else c
            e = kernel_roofline(cls, w, prof[c]["launches"], prof[c]["ms"], clocks_mhz, peaks, prof[c]["work"])
            e.update(kernel=c, launches=prof[c]["launches"] // steps,
                     avg_launch_us=prof[c]["ms"] / prof[c]["launches"] * 1e3,
                     share_of_device_time=prof[c]["ms"] / max(total_ms, 1e-9), traffic=None)
            kerns[c] = e
    return kerns


def config_lines(pins, prm, peaks, mhz):
    """One solve per other BASELINE config (device-timed, profiler off) plus one profiled
    solve for the per-kernel numbers: sweeps/s, half-sweep throughput, CG SpMV GB/s."""
    import torch
    from workloads import make
    out = {}
    stream = torch.cuda.current_stream()
    for name in CONFIG_LINES:
        w = make(name)
        gold = golden_obj(name)
        pb = pins.DeviceProblem.from_workload(w)
        ws = pins.Workspace()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        r = pins.solve(pb, prm, want_duals=True, ws=ws)
        e1.record(stream)
        torch.cuda.synchronize()
        check_solve(r, gold, name)
        sec = e0.elapsed_time(e1) / 1e3
        pins.prof_reset()
        pins.prof_enable(True)
        r2 = pins.solve(pb, prm, want_duals=False, ws=ws)
        pins.prof_enable(False)
        prof = pins.prof_read()
        # every launch of the Sinkhorn phases: dense half-sweeps, ELL walks, and the list
        # modes' auxiliary launches (records, sort, ELL build, fallback, merge)
        sw_ms = sum(prof[c]["ms"] for c in SWEEP_CLASSES)
        sw_l = 2 * r2["sweeps"]
        kerns = prof_stats(pins, w, prof, mhz, peaks, 1)
        cg = kerns.get("cg", {})
        out[name] = {
            "m": w.m, "n": w.n, "cost": ["dense", "sqeuclid", "l1"][w.kind],
            "lattice": w.meta.get("lattice", w.kind == 0 or None), "eta": w.eta,
            "seconds": sec, "outer_iters": r["outer_iters"], "sweeps": r["sweeps"],
            "newton_iters": r["newton_iters"], "cg_iters": r["cg_iters"], "certificates": r["certificates"],
            "kkt": r["kkt"], "gap": r["gap"], "dual_inf": r["dual_inf"], "obj": r["obj"], "exact_obj": gold,
            "rel_err": None if gold is None else abs(r["obj"] - gold) / abs(gold),
            "sweeps_per_s": (sw_l / 2) / (sw_ms / 1e3) if sw_ms > 0 else None,
            "half_sweep_us": sw_ms / sw_l * 1e3 if sw_l else None,
            "half_sweep_roofline": {k: kerns["sweep_row"][k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                                                         "avg_launch_us", "launches")}
            if "sweep_row" in kerns else None,
            "ksweep_roofline": {k: kerns["ksweep"][k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                                                  "avg_launch_us", "launches")}
            if "ksweep" in kerns else None,
            "cg_spmv_gbs": cg.get("achieved"), "cg_frac_hbm": cg.get("frac"),
        }
        del ws
    return out


def hbm_section(pins, peaks):
    """The HBM-bound kernels at HBM scale.  (1) Dense passes on c3's cost materialised
    as a 10^4 x 10^4 fp64 C (800 MB > 126 MB L2): one Sinkhorn sweep (two half-sweeps)
    and one evaluation (sum pass, both orientations) at k = 0, 8 B of C per entry and
    pass.  (2) The grid CG on a sparsified support with 2.4e7 entries: SpMV bytes
    24 B x nnz + 80 B x (m + n) per iteration, fixed iteration count."""
    import numpy as np
    import torch
    from workloads import make
    peak = peaks.get("hbm_gbs", 6650.0)
    out = {}
    w = make("c3_gmm10k")
    X = torch.as_tensor(w.X, dtype=torch.float64, device="cuda")
    Y = torch.as_tensor(w.Y, dtype=torch.float64, device="cuda")
    C = ((X * X).sum(1)[:, None] + (Y * Y).sum(1)[None, :] - 2.0 * X @ Y.T) * w.cost_scale   # input prep
    C.clamp_(min=0.0)
    del X, Y
    a = torch.as_tensor(w.a, dtype=torch.float64, device="cuda")
    b = torch.as_tensor(w.b, dtype=torch.float64, device="cuda")
    pb = pins.DeviceProblem(w.m, w.n, 0, a, b, w.eta, C=C)
    phi, psi, s = pins.center_init(pb)
    f = torch.zeros(w.m, dtype=torch.float64, device="cuda")
    g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    ws = pins.Workspace()
    os.environ["PINS_KSWEEP"] = "0"                           # the dense half-sweeps themselves
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, 3)          # warm-up (and the argmax seeds)
    pins.prof_reset()
    pins.prof_enable(True)
    nsw = 20
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, nsw)
    pins.evaluate(ws, pb, phi, psi, s, f, g, tau=0.0)        # sums only: the C stream
    pins.prof_enable(False)
    prof = pins.prof_read()
    del os.environ["PINS_KSWEEP"]
    # the same phase continued with the absorbed kernel-matrix sweeps (the default of long
    # phases): ELL walks stream 12 B per listed entry
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, 400)        # past the cold start's churn; list growth
    pins.prof_reset()
    pins.prof_enable(True)
    nks = 200
    pins.sinkhorn(ws, pb, phi, psi, s, f, g, 0.0, nks)
    pins.prof_enable(False)
    prof_k = pins.prof_read()
    L, ms = prof_k["ksweep"]["launches"], prof_k["ksweep"]["ms"]
    if L and ms > 0:
        byk = 12.0 * prof_k["ksweep"]["work"] / L
        gbs = byk / (ms / L / 1e3) / 1e9
        allms = sum(prof_k[c]["ms"] for c in SWEEP_CLASSES)
        out["ksweep"] = {"launches": L, "avg_launch_us": ms / L * 1e3, "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "bytes_per_launch": byk, "entries_per_launch": byk / 12.0,
                         "dense_half_sweeps": prof_k["sweep_row"]["launches"] + prof_k["sweep_col"]["launches"],
                         "half_sweep_us_all_launches": allms / (2 * nks) * 1e3,
                         "config": f"the same dense-C instance, one phase of {nks} sweeps (each phase starts with "
                                   "7 dense sweeps, then kernel-matrix mode); half_sweep_us_all_launches = every "
                                   "launch of the phase (dense sweeps, records, ELL builds, walks, fallback, merge) "
                                   "per half-sweep, profiler events included"}
    pins.prof_reset()
    pins.prof_enable(True)
    ev = pins.evaluate(ws, pb, phi, psi, s, f, g, tau=1e-4 / (w.m * w.n))   # + sparsify
    pins.prof_enable(False)
    prof_sp = pins.prof_read()
    byt = 8.0 * w.m * w.n
    for c in ("sweep_row", "sweep_col", "eval"):
        L, ms = prof[c]["launches"], prof[c]["ms"]
        if not L:
            continue
        mult = 2.0 if c == "eval" else 1.0
        gbs = mult * byt / (ms / L / 1e3) / 1e9
        out[f"dense_{c}"] = {"launches": L, "avg_launch_us": ms / L * 1e3, "achieved": gbs, "peak": peak,
                             "unit": "GB/s", "frac": gbs / peak, "bytes_per_launch": mult * byt,
                             "survivors_per_launch": prof[c]["work"] / L if c != "sweep_col" else None}
    L, ms = prof_sp["eval"]["launches"], prof_sp["eval"]["ms"]
    if L:
        gbs = 2.0 * byt / (ms / L / 1e3) / 1e9
        out["dense_eval_sparsify"] = {"launches": L, "avg_launch_us": ms / L * 1e3, "achieved": gbs, "peak": peak,
                                      "unit": "GB/s", "frac": gbs / peak, "bytes_per_launch": 2.0 * byt,
                                      "kept_entries": ev["nnz"]}
    out["dense_config"] = ("c3_gmm10k cost materialised densely (10^4 x 10^4 fp64, 800 MB), k = 0, "
                           f"{nsw} Sinkhorn sweeps, 1 sum pass (sums only), 1 sum pass with sparsification "
                           f"(nnz {ev['nnz']})")
    del C, pb, ws
    torch.cuda.empty_cache()
    # (2) SpMV: random support with 2.4e7 entries (m = n = 10^4, ~12 % dense -- the k = 1
    # support size of early EPPA), weights of a plan
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
    cws = pins.Workspace()
    its_fixed = 50
    pins.cg(cws, m, n, rowptr, colidx, val, dr, dc, 1e-12, rhs, rtol=0.0, maxit=5)      # warm-up, CSC build
    pins.prof_reset()
    pins.prof_enable(True)
    x, its, rel = pins.cg(cws, m, n, rowptr, colidx, val, dr, dc, 1e-12, rhs, rtol=0.0, maxit=its_fixed)
    pins.prof_enable(False)
    prof = pins.prof_read()
    L, ms = prof["cg"]["launches"], prof["cg"]["ms"]
    nnz = m * nnz_row
    byts = its * (24.0 * nnz + 80.0 * (m + n))
    gbs = byts / (ms / 1e3) / 1e9
    out["spmv_cg_grid"] = {"iterations": its, "nnz": nnz, "ms": ms, "achieved": gbs, "peak": peak, "unit": "GB/s",
                           "frac": gbs / peak, "bytes_per_iteration": 24.0 * nnz + 80.0 * (m + n),
                           "config": "m = n = 10^4, 2400 entries per row (2.4e7), CSR + CSC, fixed 50 iterations"}
    return out


def oracle_anchors(budget_s: float):
    """Complete oracle solves (the oracle as it stands, fp64 numpy) of small instances,
    halving stop at 1e-7 (reading R6): measured CPU seconds."""
    from oracle import pins_oracle as po
    from workloads import make
    out = []
    for name, sc in (("c0_pts64", 1.0), ("c1_rand1k", 0.25)):
        w = make(name, scale=sc)
        C = po.cost_matrix(w)
        prm = po.Params(eta=w.eta, K=20000, outer_rule=1, outer_tol=1e-7, newton_tol=1e-8)
        t0 = time.time()
        r = po.pins(C, w.a, w.b, prm)
        out.append({"config": name, "scale": sc, "m": w.m, "n": w.n, "seconds": time.time() - t0,
                    "outer_iters": r.outer_iters, "obj": r.obj})
    return out


def gpu_anchor_times(pins, anchors):
    import torch
    from workloads import make
    for a in anchors:
        w = make(a["config"], scale=a["scale"])
        pb = pins.DeviceProblem.from_workload(w)
        prm = pins.default_params(K=20000, outer_rule=1, outer_tol=1e-7, newton_tol=1e-8)
        pins.solve(pb, prm)
        torch.cuda.synchronize()
        t0 = time.time()
        r = pins.solve(pb, prm)
        torch.cuda.synchronize()
        a["gpu_seconds"] = time.time() - t0
        a["gpu_outer_iters"] = r["outer_iters"]
        a["gpu_obj"] = r["obj"]


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist
    from paper_2502_03749_b200 import pins
    from workloads import make

    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = make(args.config)
    gold = golden_obj(args.config)
    pb = pins.DeviceProblem.from_workload(w)
    prm = pins.default_params(**BENCH_PARAMS)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 512 MB > 126 MB L2
    ws = pins.Workspace()                      # one caller workspace for every step (pins_solve_ws)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        check_solve(pins.solve(pb, prm, ws=ws), gold, args.config)
    # ---- timed region (device; library profiler OFF, launches still counted) ----
    sampler = ClockSampler(local)
    sampler.start()
    pins.prof_enable(False)
    pins.prof_reset()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    results = []
    barrier()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        r = pins.solve(pb, prm, want_duals=False, ws=ws)
        ev[k][1].record(stream)
        results.append(r)
    barrier()
    clocks = sampler.stop()
    launches = int(sum(v["launches"] for v in pins.prof_read().values()))
    step_ms = [a.elapsed_time(b) for a, b in ev]
    for r in results:
        check_solve(r, gold, args.config)
    T = max_over_ranks(sum(step_ms), world, "cuda") / 1e3
    value = per_solve_value(T, args.steps, world)

    # ---- profiled steps (outside the timed region): per-kernel device time ----
    pins.prof_reset()
    pins.prof_enable(True)
    for _ in range(PROFILED_STEPS):
        flush.zero_()
        pins.solve(pb, prm, want_duals=False, ws=ws)
    torch.cuda.synchronize()
    pins.prof_enable(False)
    prof = pins.prof_read()

    # ---- end to end through the host-buffer C-ABI call ----
    hp = pins.HostProblem(w)
    pins.solve_host(hp, prm)
    barrier()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    io = None
    for k in range(args.steps):
        flush.zero_()
        e2e_ev[k][0].record(stream)
        r = pins.solve_host(hp, prm)
        e2e_ev[k][1].record(stream)
        check_solve(r, gold, args.config)
        io = (r["h2d_bytes"], r["d2h_bytes"])
    barrier()
    e2e_value = per_solve_value(max_over_ranks(sum(a.elapsed_time(b) for a, b in e2e_ev), world, "cuda") / 1e3,
                                args.steps, world)

    if rank == 0:
        r0 = results[-1]
        counts = {k: r0[k] for k in ("outer_iters", "sweeps", "newton_iters", "cg_iters", "certificates")}
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        mhz = clocks["sm_mhz"] or 1965.0
        kerns = prof_stats(pins, w, prof, mhz, peaks, PROFILED_STEPS)
        dom = max(kerns, key=lambda c: kerns[c]["share_of_device_time"])
        roof = dict(kerns[dom])
        tr_path = os.path.join(ROOT, "profiles", "ncu_traffic_r2.json")
        if os.path.exists(tr_path):       # dram bytes per launch from one ncu --set full capture
            tr = json.load(open(tr_path))
            for c, e in kerns.items():
                if c in tr:
                    e["traffic"] = tr[c]["dram_bytes_per_launch"]
                    e["traffic_source"] = tr[c]["source"]
            roof["traffic"] = kerns[dom].get("traffic")
        line = {
            "metric": "s to KKT<1e-8 (n=10k, c3_gmm10k)", "value": value, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": T * 1e3 / args.steps, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "m": w.m, "n": w.n, "eta": w.eta,
                       "cost": ["dense", "sqeuclid", "l1"][w.kind], "points": "1/64 lattice (DESIGN.md §4)",
                       "params": BENCH_PARAMS, "l2": "flushed (512 MB write) before every timed step",
                       "profiler": f"off in the timed region; roofline from {PROFILED_STEPS} extra profiled steps",
                       "parallelism": f"replicas x{world}"},
            "accuracy": {"kkt": r0["kkt"], "obj": r0["obj"], "exact_obj": gold,
                         "rel_err": None if gold is None else abs(r0["obj"] - gold) / abs(gold),
                         "lp_dual_obj": r0["lp_dual_obj"], "gap": r0["gap"],
                         "rel_gap": r0["gap"] / abs(r0["obj"]), "dual_inf": r0["dual_inf"],
                         "cert_tree": r0["cert_tree"]},
            "counts": counts,
            "clocks": clocks,
            "roofline": roof,
            "roofline_kernels": kerns,
            "prof": {c: {"launches": v["launches"] // PROFILED_STEPS, "ms_per_step": v["ms"] / PROFILED_STEPS}
                     for c, v in prof.items()},
            "gpu_launches": launches // args.steps,
            "e2e": {"value": e2e_value, "unit": "s", "h2d_bytes_per_step": io[0], "d2h_bytes_per_step": io[1]},
        }
        if not args.quick and world == 1:
            line["configs"] = config_lines(pins, prm, peaks, mhz)
            line["hbm"] = hbm_section(pins, peaks)
        os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_baseline(w, counts, args.cpu_budget, blas_threads())
            if not args.quick:
                anchors = oracle_anchors(args.cpu_budget)
                gpu_anchor_times(pins, anchors)
                cb["measured_solves"] = anchors
            line["cpu_baseline"] = cb
        # the work profile the reference arm scales by (counts of this measured solve)
        with open(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "profiles",
                               f"workprofile_{args.config}.json"), "w") as fh:
            json.dump({"config": args.config, "counts": counts, "source": "bench.py GPU solve"}, fh)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
