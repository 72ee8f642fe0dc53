"""Exact LP oracle for PAPER.md Eq. (1) (lines 41-46) -- TEST INFRASTRUCTURE ONLY.

* :func:`solve_exact` -- hand-written network simplex (``oracle/netsimplex.c``),
  compiled with gcc on first use, loaded with ctypes.  Returns an optimal vertex
  plan, its cost and LP duals (u, v) with u_i + v_j <= C_ij.
* :func:`brute_force_assignment` -- exhaustive minimum over all permutations
  for uniform square instances (n <= 8).  PAPER.md Thm 4.3 proof (line 362):
  for m = n the feasible set is the Birkhoff polytope "whose vertices are
  precisely the permutation matrices", and the LP optimum is attained at a
  vertex, so OPT = (1/n) min_sigma sum_i C_{i,sigma(i)}.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
import sys
from typing import Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "netsimplex.c")
_LIB = os.path.join(_HERE, "_netsimplex.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile netsimplex.c into oracle/_netsimplex.so (plain gcc, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.ns_solve.restype = ctypes.c_int
        lib.ns_solve.argtypes = [ctypes.c_longlong, ctypes.c_longlong, dp, dp, dp, dp, dp, dp,
                                 dp, dp, ctypes.c_longlong]
        _lib = lib
    return _lib


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def solve_exact(C: np.ndarray, a: np.ndarray, b: np.ndarray, max_pivots: int = 10 ** 12,
                want_plan: bool = True):
    """Network simplex on Eq. (1).  Returns dict(obj, X, u, v, pivots, max_art, min_rc)."""
    lib = _load()
    C = np.ascontiguousarray(C, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    m, n = C.shape
    X = np.empty((m, n), dtype=np.float64)
    u = np.empty(m, dtype=np.float64)
    v = np.empty(n, dtype=np.float64)
    obj = ctypes.c_double(0.0)
    stats = np.zeros(4, dtype=np.float64)
    rc = lib.ns_solve(m, n, _ptr(C), _ptr(a), _ptr(b), _ptr(X), _ptr(u), _ptr(v),
                      ctypes.byref(obj), _ptr(stats), int(max_pivots))
    if rc != 0:
        raise RuntimeError(f"network simplex failed (status {rc})")
    out = dict(obj=obj.value, u=u, v=v, pivots=int(stats[0]), max_art=float(stats[1]),
               min_rc=float(stats[2]))
    out["X"] = X if want_plan else None
    return out


def brute_force_assignment(C: np.ndarray) -> Tuple[Tuple[int, ...], float]:
    """min over permutations of (1/n) sum_i C[i, sigma(i)]; lexicographic tie-break."""
    C = np.asarray(C, dtype=np.float64)
    n = C.shape[0]
    if C.shape != (n, n) or n > 8:
        raise ValueError("brute force needs a square matrix with n <= 8")
    best, best_p = np.inf, None
    for p in itertools.permutations(range(n)):
        s = 0.0
        for i in range(n):
            s += C[i, p[i]]
        if s < best:
            best, best_p = s, p
    return best_p, best / n


if __name__ == "__main__":  # pragma: no cover - manual check
    build(force=True)
    print("built", _LIB, file=sys.stderr)
