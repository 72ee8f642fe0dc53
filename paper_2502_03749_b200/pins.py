"""Thin ctypes binding of libpins_b200.so (include/pins.h).  Argument marshalling
only: every step of the PINS path runs in the CUDA library.  There is no CPU
fallback -- if the library or a CUDA device is missing, calls raise.

Names follow the C ABI: ``sinkhorn_sweep`` -> ``pins_sinkhorn_sweep`` etc.
Tensors are torch CUDA tensors (fp64 unless stated); torch only provides
device memory and the current stream.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_void_p
from typing import Dict, Optional

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libpins_b200.so")

COST_DENSE, COST_SQEUCLID, COST_L1 = 0, 1, 2

EXPORTS = [
    "pins_default_params", "pins_workspace_create", "pins_workspace_destroy", "pins_last_error",
    "pins_center_init", "pins_center_update", "pins_sinkhorn_sweep", "pins_sinkhorn", "pins_evaluate",
    "pins_get_csr", "pins_sparsify_dense", "pins_cg", "pins_newton_step", "pins_residuals", "pins_lp_certificate", "pins_plan", "pins_solve",
    "pins_prof_enable", "pins_prof_reset", "pins_prof_read", "pins_prof_read_work", "pins_solve_host",
    "pins_solve_ws",
]


class Problem(ctypes.Structure):
    _fields_ = [("m", c_int64), ("n", c_int64), ("cost_kind", c_int32), ("d", c_int32),
                ("C", c_void_p), ("ldc", c_int64), ("x", c_void_p), ("y", c_void_p),
                ("cost_scale", c_double), ("a", c_void_p), ("b", c_void_p), ("eta", c_double)]


class Params(ctypes.Structure):
    _fields_ = [("K", c_int32), ("outer_rule", c_int32), ("outer_tol", c_double), ("T1", c_int32),
                ("sink_tol", c_double), ("T2", c_int32), ("newton_tol", c_double),
                ("theta", c_double), ("cg_tol", c_double), ("cg_forcing", c_double),
                ("cg_maxit", c_int32), ("mu_rel", c_double), ("armijo_c", c_double),
                ("beta", c_double), ("max_backtracks", c_int32), ("warm_start", c_int32)]


class Result(ctypes.Structure):
    _fields_ = [("f", c_void_p), ("g", c_void_p), ("phi", c_void_p), ("psi", c_void_p),
                ("u", c_void_p), ("v", c_void_p), ("s", c_double), ("obj", c_double),
                ("dual_obj", c_double), ("lp_dual_obj", c_double), ("kkt", c_double),
                ("dual_inf", c_double), ("gap", c_double), ("outer_iters", c_int32),
                ("sweeps", c_int32), ("newton_iters", c_int32), ("cg_iters", c_int32),
                ("status", c_int32), ("certificates", c_int32), ("cert_tree", c_int32),
                ("obj_trace_host", POINTER(c_double)), ("seconds", c_double)]


_lib = None


def load():
    """Load libpins_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                           "(python paper_2502_03749_b200/build.py)")
    lib = ctypes.CDLL(LIB_PATH)
    P, V, D, I32, I64 = POINTER(Problem), c_void_p, c_double, c_int32, c_int64
    sig = {
        "pins_default_params": (None, [POINTER(Params)]),
        "pins_workspace_create": (I32, [POINTER(c_void_p)]),
        "pins_workspace_destroy": (None, [V]),
        "pins_last_error": (ctypes.c_char_p, []),
        "pins_center_init": (I32, [P, V, V, POINTER(D), V]),
        "pins_center_update": (I32, [P, V, V, POINTER(D), V, V, V]),
        "pins_sinkhorn_sweep": (I32, [V, P, V, V, D, V, V, V]),
        "pins_sinkhorn": (I32, [V, P, V, V, D, V, V, D, I32, POINTER(I32), POINTER(D), V]),
        "pins_evaluate": (I32, [V, P, V, V, D, V, V, D, V, V, POINTER(D), V]),
        "pins_get_csr": (I32, [V, V, V, V, I64, POINTER(I64), POINTER(I64)]),
        "pins_sparsify_dense": (I32, [V, I64, I64, V, I64, D, V, V, V, I64, POINTER(I64), V]),
        "pins_cg": (I32, [V, I64, I64, V, V, V, I64, V, V, D, V, V, D, I32, POINTER(I32),
                          POINTER(D), V]),
        "pins_newton_step": (I32, [V, P, POINTER(Params), V, V, D, V, V, POINTER(D), V]),
        "pins_residuals": (I32, [V, P, V, V, D, V, V, V, V, POINTER(D), V]),
        "pins_plan": (I32, [P, V, V, D, V, V, V, I64, V]),
        "pins_lp_certificate": (I32, [V, P, POINTER(Params), V, V, D, V, V, V, V, POINTER(D), V]),
        "pins_solve": (I32, [P, POINTER(Params), POINTER(Result), V]),
        "pins_solve_ws": (I32, [V, P, POINTER(Params), POINTER(Result), V]),
        "pins_solve_host": (I32, [P, POINTER(Params), POINTER(Result), POINTER(I64), V]),
        "pins_prof_enable": (None, [I32]),
        "pins_prof_reset": (None, []),
        "pins_prof_read": (I32, [I32, POINTER(I64), POINTER(D)]),
        "pins_prof_read_work": (I32, [I32, POINTER(D)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int):
    if rc != 0:
        msg = load().pins_last_error().decode()
        raise RuntimeError(f"libpins_b200 error {rc}: {msg}")


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2502_03749_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _p(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream():
    return c_void_p(_torch().cuda.current_stream().cuda_stream)


def default_params(**overrides) -> Params:
    p = Params()
    load().pins_default_params(ctypes.byref(p))
    for k, v in overrides.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


class DeviceProblem:
    """Device copy of an OT instance + the C ``pins_problem`` describing it."""

    def __init__(self, m, n, kind, a, b, eta, C=None, x=None, y=None, cost_scale=1.0):
        self.m, self.n, self.kind, self.eta = int(m), int(n), int(kind), float(eta)
        self.a, self.b, self.C, self.x, self.y = a, b, C, x, y
        self.cost_scale = float(cost_scale)
        self.struct = Problem(
            m=self.m, n=self.n, cost_kind=self.kind, d=0 if x is None else int(x.shape[1]),
            C=_p(C), ldc=0 if C is None else int(C.stride(0)), x=_p(x), y=_p(y),
            cost_scale=self.cost_scale, a=_p(a), b=_p(b), eta=self.eta)

    @classmethod
    def from_workload(cls, w, device="cuda", eta=None):
        torch = _torch()
        t = lambda v: None if v is None else torch.as_tensor(v, dtype=torch.float64).to(device).contiguous()
        return cls(w.m, w.n, w.kind, t(w.a), t(w.b), w.eta if eta is None else eta,
                   C=t(w.C), x=t(w.X), y=t(w.Y), cost_scale=w.cost_scale)

    def ref(self):
        return ctypes.byref(self.struct)


class Workspace:
    def __init__(self):
        self.h = c_void_p()
        _check(load().pins_workspace_create(ctypes.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                load().pins_workspace_destroy(self.h)
        except Exception:
            pass


def center_init(pb: DeviceProblem):
    torch = _torch()
    phi = torch.empty(pb.m, dtype=torch.float64, device="cuda")
    psi = torch.empty(pb.n, dtype=torch.float64, device="cuda")
    s = c_double(0.0)
    _check(load().pins_center_init(pb.ref(), _p(phi), _p(psi), ctypes.byref(s), _stream()))
    return phi, psi, s.value


def center_update(pb: DeviceProblem, phi, psi, s: float, f, g) -> float:
    sc = c_double(s)
    _check(load().pins_center_update(pb.ref(), _p(phi), _p(psi), ctypes.byref(sc), _p(f), _p(g),
                                     _stream()))
    return sc.value


def sinkhorn_sweep(ws: Workspace, pb: DeviceProblem, phi, psi, s: float, f, g):
    _check(load().pins_sinkhorn_sweep(ws.h, pb.ref(), _p(phi), _p(psi), s, _p(f), _p(g), _stream()))


def sinkhorn(ws: Workspace, pb: DeviceProblem, phi, psi, s: float, f, g, tol: float, max_sweeps: int):
    """Sinkhorn phase (Alg. 2 lines 4-8) in place; returns (sweeps, final ||grad P||_1)."""
    t, r = c_int32(), c_double()
    _check(load().pins_sinkhorn(ws.h, pb.ref(), _p(phi), _p(psi), s, _p(f), _p(g), float(tol), int(max_sweeps),
                                ctypes.byref(t), ctypes.byref(r), _stream()))
    return t.value, r.value


def evaluate(ws: Workspace, pb: DeviceProblem, phi, psi, s, f, g, tau=0.0, want_sums=True) -> Dict:
    torch = _torch()
    r = torch.empty(pb.m, dtype=torch.float64, device="cuda") if want_sums else None
    c = torch.empty(pb.n, dtype=torch.float64, device="cuda") if want_sums else None
    out = (c_double * 8)()
    _check(load().pins_evaluate(ws.h, pb.ref(), _p(phi), _p(psi), s, _p(f), _p(g), float(tau),
                                _p(r), _p(c), out, _stream()))
    return dict(grad_l1=out[0], sum_x=out[1], cost=out[2], dual_obj=out[3], nnz=int(out[4]),
                max_z=out[5], r=r, c=c)


def get_csr(ws: Workspace):
    """Copy of the workspace CSR: (rowptr int64, colidx int32, val fp64) torch tensors."""
    torch = _torch()
    nnz, m = c_int64(), c_int64()
    lib = load()
    _check(lib.pins_get_csr(ws.h, None, None, None, 0, ctypes.byref(nnz), ctypes.byref(m)))
    rowptr = torch.empty(m.value + 1, dtype=torch.int64, device="cuda")
    colidx = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
    val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device="cuda")
    _check(lib.pins_get_csr(ws.h, _p(rowptr), _p(colidx), _p(val), colidx.numel(),
                            ctypes.byref(nnz), ctypes.byref(m)))
    return rowptr, colidx[:nnz.value], val[:nnz.value]


def sparsify_dense(ws: Workspace, P, tau: float):
    """CSR (rowptr, colidx, val) of a caller-given dense P: P_ij >= tau (warp-ballot
    compaction kernels of pins_sparsify_dense; the evaluation pass's own sparsifier is
    reached through evaluate(tau > 0) + get_csr)."""
    torch = _torch()
    m, n = P.shape
    lib = load()
    nnz = c_int64()
    _check(lib.pins_sparsify_dense(ws.h, m, n, _p(P), int(P.stride(0)), float(tau), None, None, None, 0,
                                   ctypes.byref(nnz), _stream()))
    rowptr = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    colidx = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
    val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device="cuda")
    _check(lib.pins_sparsify_dense(ws.h, m, n, _p(P), int(P.stride(0)), float(tau), _p(rowptr),
                                   _p(colidx), _p(val), colidx.numel(), ctypes.byref(nnz), _stream()))
    return rowptr, colidx[:nnz.value], val[:nnz.value]


def cg(ws: Workspace, m, n, rowptr, colidx, val, dr, dc, mu, rhs, rtol=1e-10, maxit=1000):
    torch = _torch()
    x = torch.empty(m + n, dtype=torch.float64, device="cuda")
    its = c_int32()
    rel = c_double()
    _check(load().pins_cg(ws.h, m, n, _p(rowptr), _p(colidx), _p(val), int(val.numel()), _p(dr),
                          _p(dc), float(mu), _p(rhs), _p(x), float(rtol), int(maxit),
                          ctypes.byref(its), ctypes.byref(rel), _stream()))
    return x, its.value, rel.value


def newton_step(ws: Workspace, pb: DeviceProblem, prm: Params, phi, psi, s, f, g) -> Dict:
    info = (c_double * 8)()
    _check(load().pins_newton_step(ws.h, pb.ref(), ctypes.byref(prm), _p(phi), _p(psi), s, _p(f),
                                   _p(g), info, _stream()))
    return dict(grad_before=info[0], grad_after=info[1], alpha=info[2], cg_iters=int(info[3]),
                cg_relres=info[4], nnz=int(info[5]), trials=int(info[6]))


def residuals(ws: Workspace, pb: DeviceProblem, phi, psi, s, f, g) -> Dict:
    torch = _torch()
    u = torch.empty(pb.m, dtype=torch.float64, device="cuda")
    v = torch.empty(pb.n, dtype=torch.float64, device="cuda")
    out = (c_double * 8)()
    _check(load().pins_residuals(ws.h, pb.ref(), _p(phi), _p(psi), s, _p(f), _p(g), _p(u), _p(v),
                                 out, _stream()))
    return dict(kkt=out[0], dual_inf=out[1], obj=out[2], lp_dual_obj=out[3], gap=out[4], u=u, v=v)


def lp_certificate(ws: Workspace, pb: DeviceProblem, prm: Params, phi, psi, s, f, g) -> Dict:
    """LP certificate of X~(f, g) (reading R11): certified duals u, v and the LP KKT."""
    torch = _torch()
    u = torch.empty(pb.m, dtype=torch.float64, device="cuda")
    v = torch.empty(pb.n, dtype=torch.float64, device="cuda")
    out = (c_double * 8)()
    _check(load().pins_lp_certificate(ws.h, pb.ref(), ctypes.byref(prm), _p(phi), _p(psi), s, _p(f), _p(g),
                                      _p(u), _p(v), out, _stream()))
    return dict(primal=out[0], pobj=out[1], dual_obj=out[2], gap=out[3], dual_inf=out[4],
                tree_edges=int(out[5]), used_tree=int(out[6]), nnz=int(out[7]), u=u, v=v)


def plan(pb: DeviceProblem, phi, psi, s, f, g):
    torch = _torch()
    X = torch.empty(pb.m, pb.n, dtype=torch.float64, device="cuda")
    _check(load().pins_plan(pb.ref(), _p(phi), _p(psi), s, _p(f), _p(g), _p(X), pb.n, _stream()))
    return X


def solve(pb: DeviceProblem, prm: Optional[Params] = None, trace: bool = False, want_duals=True,
          ws: Optional["Workspace"] = None) -> Dict:
    torch = _torch()
    prm = prm or default_params()
    dev = dict(dtype=torch.float64, device="cuda")
    f, g = torch.empty(pb.m, **dev), torch.empty(pb.n, **dev)
    phi, psi = torch.empty(pb.m, **dev), torch.empty(pb.n, **dev)
    u = torch.empty(pb.m, **dev) if want_duals else None
    v = torch.empty(pb.n, **dev) if want_duals else None
    res = Result(f=_p(f), g=_p(g), phi=_p(phi), psi=_p(psi), u=_p(u), v=_p(v))
    tr = (c_double * max(1, prm.K))() if trace else None
    if trace:
        res.obj_trace_host = ctypes.cast(tr, POINTER(c_double))
    if ws is None:
        _check(load().pins_solve(pb.ref(), ctypes.byref(prm), ctypes.byref(res), _stream()))
    else:
        _check(load().pins_solve_ws(ws.h, pb.ref(), ctypes.byref(prm), ctypes.byref(res), _stream()))
    out = {k: getattr(res, k) for k in ("s", "obj", "dual_obj", "lp_dual_obj", "kkt", "dual_inf", "gap",
                                        "outer_iters", "sweeps", "newton_iters", "cg_iters", "status",
                                        "certificates", "cert_tree", "seconds")}
    out.update(f=f, g=g, phi=phi, psi=psi, u=u, v=v)
    if trace:
        out["trace"] = [tr[i] for i in range(res.outer_iters)]
    return out


PROF_CLASSES = ["sweep_row", "sweep_col", "eval", "reduce", "csr", "cg", "vec", "plan", "ksweep", "sweep_aux"]


def prof_enable(on: bool = True):
    load().pins_prof_enable(1 if on else 0)


def prof_reset():
    load().pins_prof_reset()


def prof_read() -> Dict[str, Dict]:
    """{class: {"launches": L, "ms": device ms}} since the last prof_reset (synchronises)."""
    lib = load()
    out = {}
    for c, name in enumerate(PROF_CLASSES):
        n, ms = c_int64(), c_double()
        _check(lib.pins_prof_read(c, ctypes.byref(n), ctypes.byref(ms)))
        wk = c_double()
        _check(lib.pins_prof_read_work(c, ctypes.byref(wk)))
        out[name] = {"launches": n.value, "ms": ms.value, "work": wk.value}
    return out


class HostProblem:
    """Host (pinned) copy of an OT instance for the end-to-end path ``solve_host``."""

    def __init__(self, w, eta=None):
        torch = _torch()
        pin = lambda v: None if v is None else torch.as_tensor(v, dtype=torch.float64).contiguous().pin_memory()
        self.m, self.n = int(w.m), int(w.n)
        self.a, self.b, self.C, self.x, self.y = pin(w.a), pin(w.b), pin(w.C), pin(w.X), pin(w.Y)
        self.struct = Problem(
            m=self.m, n=self.n, cost_kind=int(w.kind), d=0 if w.X is None else int(w.X.shape[1]),
            C=_p(self.C), ldc=0 if self.C is None else int(self.C.stride(0)), x=_p(self.x), y=_p(self.y),
            cost_scale=float(w.cost_scale), a=_p(self.a), b=_p(self.b), eta=float(w.eta if eta is None else eta))
        self.u = torch.empty(self.m, dtype=torch.float64).pin_memory()
        self.v = torch.empty(self.n, dtype=torch.float64).pin_memory()


def solve_host(hp: HostProblem, prm: Optional[Params] = None) -> Dict:
    """End-to-end pins_solve_host: inputs copied from pinned host memory, LP duals u, v
    copied back into hp.u / hp.v; returns the scalars plus h2d / d2h byte counts."""
    prm = prm or default_params()
    res = Result(u=_p(hp.u), v=_p(hp.v))
    io = (c_int64 * 2)()
    _check(load().pins_solve_host(ctypes.byref(hp.struct), ctypes.byref(prm), ctypes.byref(res), io, _stream()))
    out = {k: getattr(res, k) for k in ("s", "obj", "dual_obj", "lp_dual_obj", "kkt", "dual_inf", "gap",
                                        "outer_iters", "sweeps", "newton_iters", "cg_iters", "status",
                                        "certificates", "cert_tree", "seconds")}
    out.update(h2d_bytes=io[0], d2h_bytes=io[1])
    return out
