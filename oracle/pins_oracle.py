"""Plain fp64 CPU PINS -- the parity oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It shares no code with the CUDA path
(paper_2502_03749_b200/): it is written from PAPER.md, dense and unblocked, in
the paper's notation, with numpy primitives (exp, log, sum, sparse matvec) as
its only library steps.

Every function cites the PAPER.md line range and the equation / algorithm line
it restates.  Readings of ambiguous passages are listed in DESIGN.md §3 and are
marked "reading R<k>" here.

Notation (§3.2):
  C         cost, m x n                         (Eq. (1), line 44)
  X^k       proximal centre, carried as log X^k (Eq. (5))
  C^k       = C - eta log X^k                   (Alg. 2 line 3)
  f, g      dual potentials of subproblem (6)
  X~(f,g)   = exp((f e^T + e g^T - C^k - eta E)/eta)          (Eq. (7), :226-229)
  P^k(f,g)  = <a,f> + <b,g> - eta <E, X~(f,g)>               (Eq. (8), :232-237)
  grad P^k  = (a - X~ e_n, b - X~^T e_m)                      (Eq. (9), :241-243)
  hess P^k  = -(1/eta) [[diag(X~ e_n), X~], [X~^T, diag(X~^T e_m)]]  (Eq. (9), :244-248)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import scipy.sparse as sp

from workloads.gen import COST_DENSE, COST_L1, COST_SQEUCLID, Workload


# --------------------------------------------------------------------------- cost
def cost_matrix(w: Workload) -> np.ndarray:
    """Dense C for a workload (input definition): C_ij = D_ij * scale.

    D_ij = sum_d (x_id - y_jd)^2 (squared Euclidean) or sum_d |x_id - y_jd| (L1),
    evaluated pair by pair by broadcasting; dense workloads carry C directly.
    """
    if w.kind == COST_DENSE:
        return np.array(w.C, dtype=np.float64, copy=True)
    X, Y = w.X, w.Y
    C = np.empty((w.m, w.n), dtype=np.float64)
    bs = max(1, 4_000_000 // max(1, w.n * w.d))
    for s in range(0, w.m, bs):
        diff = X[s:s + bs, None, :] - Y[None, :, :]
        D = (diff * diff).sum(-1) if w.kind == COST_SQEUCLID else np.abs(diff).sum(-1)
        C[s:s + bs] = D * w.cost_scale
    return C


# ------------------------------------------------------------------ Eq. (7)-(9)
def shifted_cost(C: np.ndarray, logX: np.ndarray, eta: float) -> np.ndarray:
    """C^k = C - eta log X^k.  Alg. 2 line 3; §3.2."""
    return C - eta * logX


def log_plan(f, g, Ck, eta):
    """log X~^{k*}(f,g) = (f e^T + e g^T - C^k - eta E) / eta.  Eq. (7)."""
    return (f[:, None] + g[None, :] - Ck - eta) / eta


def plan(f, g, Ck, eta):
    """X~^{k*}(f,g), Eq. (7)."""
    return np.exp(log_plan(f, g, Ck, eta))


def dual_objective(f, g, Ck, a, b, eta) -> float:
    """P^k(f,g) = <a,f> + <b,g> - eta <E, X~(f,g)>.  Eq. (8)."""
    return float(a @ f + b @ g - eta * plan(f, g, Ck, eta).sum())


def dual_gradient(f, g, Ck, a, b, eta):
    """(grad_f P^k, grad_g P^k) = (a - X~ e_n, b - X~^T e_m).  Eq. (9)."""
    X = plan(f, g, Ck, eta)
    return a - X.sum(axis=1), b - X.sum(axis=0)


def hessian_dense(f, g, Ck, eta) -> np.ndarray:
    """Full (m+n)x(m+n) Hessian of P^k.  Eq. (9), PAPER.md:244-248 (small cases only)."""
    X = plan(f, g, Ck, eta)
    top = np.hstack([np.diag(X.sum(axis=1)), X])
    bot = np.hstack([X.T, np.diag(X.sum(axis=0))])
    return -np.vstack([top, bot]) / eta


def logsumexp(A: np.ndarray, axis: int) -> np.ndarray:
    """log sum exp along an axis, with the usual max shift (an exact identity)."""
    mx = A.max(axis=axis, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    return (mx + np.log(np.exp(A - mx).sum(axis=axis, keepdims=True))).squeeze(axis)


# ---------------------------------------------------------------- Sinkhorn (6)
def sinkhorn_sweep(f, g, Ck, a, b, eta):
    """One log-domain Sinkhorn sweep, Alg. 2 lines 5-6, = Alg. 1 lines 3-4.

      f^{t+1} = f^t + eta (log a - log(X~(f^t, g^t) e_n))
      g^{t+1} = g^t + eta (log b - log(X~(f^{t+1}, g^t)^T e_m))

    log of a row/column sum of X~ is the logsumexp of the matching row/column of
    log X~ ("log-domain version").
    """
    f1 = f + eta * (np.log(a) - logsumexp(log_plan(f, g, Ck, eta), axis=1))
    g1 = g + eta * (np.log(b) - logsumexp(log_plan(f1, g, Ck, eta), axis=0))
    return f1, g1


# ------------------------------------------------------------ Sparsification
def sparsify_threshold(P: np.ndarray, tau: float) -> np.ndarray:
    """Keep-mask of the transport-plan block: P_ij >= tau.

    §3.2 "Sparsification" and Alg. 2 line 11;
    reading R3: a value threshold on P = X~ (BASELINE north star:
    "thresholds P ... into a CSR pattern"); diagonal blocks are kept exact.
    """
    return P >= tau


def sparsify_topk(P: np.ndarray, rho: float) -> np.ndarray:
    """Paper-literal variant: keep the ceil(rho*m*n) largest entries (PAPER.md:256,
    "truncate the (1-rho) n^2-smallest entries"); ties -> smaller (row, col) first."""
    m, n = P.shape
    k = int(math.ceil(rho * m * n))
    flat = P.ravel()
    order = np.lexsort((np.arange(flat.size), -flat))  # value desc, index asc
    mask = np.zeros(flat.size, dtype=bool)
    mask[order[:k]] = True
    return mask.reshape(m, n)


def csr_from_mask(P: np.ndarray, mask: np.ndarray):
    """Row-major CSR (rowptr, colidx, values) of P restricted to mask, columns ascending."""
    rows, cols = np.nonzero(mask)
    rowptr = np.zeros(P.shape[0] + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    return rowptr, cols.astype(np.int64), P[rows, cols]


# --------------------------------------------------------------- CG (§3.2)
def cg(matvec, rhs: np.ndarray, tol: float, maxit: int, diag: Optional[np.ndarray] = None):
    """Conjugate gradients (Fletcher & Reeves citation), Jacobi
    preconditioned when ``diag`` is given (reading R5).  Stops when
    ||r||_2 <= tol ||rhs||_2.  Returns (x, iterations, relative residual)."""
    x = np.zeros_like(rhs)
    r = rhs.copy()
    nb = float(np.linalg.norm(rhs))
    if nb == 0.0:
        return x, 0, 0.0
    z = r / diag if diag is not None else r.copy()
    p = z.copy()
    rz = float(r @ z)
    it = 0
    res = 1.0
    while it < maxit:
        res = float(np.linalg.norm(r)) / nb
        if res <= tol:
            break
        Ap = matvec(p)
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            break
        alpha = rz / pAp
        x = x + alpha * p
        r = r - alpha * Ap
        z = r / diag if diag is not None else r.copy()
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
    res = float(np.linalg.norm(r)) / nb
    return x, it, res


@dataclass
class Params:
    """Solver parameters (shared semantics with include/pins.h ``pins_params``).

    Defaults follow PAPER.md Appendix A.2 (lines 477-485) where it states them.
    """
    eta: float = 1e-2
    K: int = 500                  # max EPPA iterations (A.2: 500)
    outer_tol: float = 1e-4       # A.2 "relative error threshold of 1e-4"
    outer_rule: int = 0           # 0: relative change, 1: halving, 2: geometric tail (reading R6)
    T1: int = 50000               # max Sinkhorn sweeps per subproblem (A.2)
    sink_tol: float = 6.3e-4      # A.2 "absolute error threshold of approximately 6.3e-4"
    T2: int = 20                  # max Newton iterations (A.2)
    newton_tol: float = 1e-8      # A.2 "absolute error threshold of 1e-8"
    theta: float = 1e-4           # sparsify threshold tau = theta/(m n) (reading R3)
    cg_tol: float = 1e-6          # floor of the CG relative tolerance
    cg_forcing: float = 0.5       # reading R5: rtol = clamp(cg_forcing*newton_tol/||grad||_1, cg_tol, 0.5)
    cg_maxit: int = 1000
    mu_rel: float = 1e-10         # Tikhonov damping relative to max diagonal (reading R5)
    armijo_c: float = 1e-4        # reading R4
    beta: float = 0.5
    max_backtracks: int = 30
    warm_start: int = 1           # reading R7: 1 carry (f,g), 2 extrapolate (safeguarded), 0 zero


def residual_l1(f, g, Ck, a, b, eta) -> float:
    """||X~ e_n - a||_1 + ||X~^T e_m - b||_1 (= ||grad P^k||_1, Eq. (9))."""
    gf, gg = dual_gradient(f, g, Ck, a, b, eta)
    return float(np.abs(gf).sum() + np.abs(gg).sum())


def newton_direction(f, g, Ck, a, b, eta, prm: Params):
    """Alg. 2 lines 10-12.

    Hessian by Eq. (9); H^t = Sparsify(hess, rho) keeps the diagonal blocks and
    the thresholded transport-plan block; CG solves H^t (df, dg) = -grad P.
    With H^t = -(1/eta) M this is  M (df, dg) = eta grad P,
    M = [[diag(X~ e), X^],[X^^T, diag(X~^T e)]] + mu I   (reading R5).
    """
    m, n = Ck.shape
    X = plan(f, g, Ck, eta)
    r = X.sum(axis=1)
    c = X.sum(axis=0)
    grad = np.concatenate([a - r, b - c])
    tau = prm.theta / (m * n)
    mask = sparsify_threshold(X, tau)
    Xs = sp.csr_matrix(np.where(mask, X, 0.0))
    mu = prm.mu_rel * max(float(r.max()), float(c.max()))
    diag = np.concatenate([r, c]) + mu

    def matvec(p):
        return np.concatenate([r * p[:m] + Xs @ p[m:], Xs.T @ p[:m] + c * p[m:]]) + mu * p

    rtol = cg_rtol(float(np.abs(grad).sum()), prm)
    d, its, res = cg(matvec, eta * grad, rtol, prm.cg_maxit, diag=diag)
    return d[:m], d[m:], dict(grad=grad, nnz=int(mask.sum()), cg_iters=its, cg_res=res, tau=tau)


def cg_rtol(gnorm1: float, prm: Params) -> float:
    """Inexact-Newton forcing term (reading R5): the CG relative tolerance is
    clamp(cg_forcing * newton_tol / ||grad P||_1, cg_tol, 0.5)."""
    if prm.cg_forcing <= 0.0 or gnorm1 <= 0.0:
        return prm.cg_tol
    return min(0.5, max(prm.cg_tol, prm.cg_forcing * prm.newton_tol / gnorm1))


def dual_increase(f, g, df, dg, alpha, Ck, a, b, eta) -> float:
    """P^k(f + alpha df, g + alpha dg) - P^k(f, g), from Eq. (8) rearranged:

      = alpha (<a,df> + <b,dg>) - eta sum_ij X~_ij expm1(alpha (df_i + dg_j)/eta)

    (an exact identity; evaluating the difference instead of two values of P
    keeps it meaningful when it is far below the ulp of P itself, reading R4).
    """
    X = plan(f, g, Ck, eta)
    w = alpha * (df[:, None] + dg[None, :]) / eta
    with np.errstate(over="ignore", invalid="ignore"):
        s = float((X * np.expm1(w)).sum())
    return float(alpha * (a @ df + b @ dg) - eta * s)


def line_search(f, g, df, dg, Ck, a, b, eta, prm: Params):
    """Backtracking line search, §3.2, ascent form for max P^k:
    largest alpha in {1, beta, beta^2, ...} with
    P(x + alpha d) >= P(x) + c alpha grad P^T d   (reading R4: c = armijo_c,
    the difference P(x + alpha d) - P(x) taken from :func:`dual_increase`).
    Returns (alpha, increase); alpha = 0.0 when no trial is accepted."""
    gf, gg = dual_gradient(f, g, Ck, a, b, eta)
    slope = float(gf @ df + gg @ dg)
    alpha = 1.0
    for _ in range(prm.max_backtracks):
        inc = dual_increase(f, g, df, dg, alpha, Ck, a, b, eta)
        if np.isfinite(inc) and inc >= prm.armijo_c * alpha * slope:
            return alpha, inc
        alpha *= prm.beta
    return 0.0, 0.0


def newton_step(f, g, Ck, a, b, eta, prm: Params):
    """One sparse Newton iteration, Alg. 2 lines 10-14."""
    df, dg, info = newton_direction(f, g, Ck, a, b, eta, prm)
    alpha, _ = line_search(f, g, df, dg, Ck, a, b, eta, prm)
    info["alpha"] = alpha
    return f + alpha * df, g + alpha * dg, info


# ------------------------------------------------------------ KKT / objective
def kkt(C, logX, a, b, u, v) -> Dict[str, float]:
    """Residuals of the OT LP, Eq. (1): primal ||Xe-a||_1+||X^Te-b||_1, dual
    infeasibility max(0, max_ij u_i+v_j-C_ij), duality gap <C,X>-<a,u>-<b,v>."""
    X = np.exp(logX)
    primal = float(np.abs(X.sum(1) - a).sum() + np.abs(X.sum(0) - b).sum())
    dual_inf = float(max(0.0, (u[:, None] + v[None, :] - C).max()))
    pobj = float((C * X).sum())
    dobj = float(a @ u + b @ v)
    return dict(primal=primal, dual_inf=dual_inf, pobj=pobj, dobj=dobj, gap=pobj - dobj)


@dataclass
class Result:
    logX: np.ndarray
    f: np.ndarray
    g: np.ndarray
    u: np.ndarray
    v: np.ndarray
    obj: float
    dual_obj: float
    kkt: Dict[str, float]
    outer_iters: int
    phi: np.ndarray          # eta log a + sum_t f^t      (centre of the next subproblem:
    psi: np.ndarray          # eta log b + sum_t (g^t-eta)  C^K = s_next C - phi (+) psi)
    s_next: float
    sweeps: int
    newton_iters: int
    cg_iters: int
    trace: List[Dict] = field(default_factory=list)


def pins(C: np.ndarray, a: np.ndarray, b: np.ndarray, prm: Params, trace: bool = False) -> Result:
    """PINS, Algorithm 2.

    X^0 = a b^T (reading R1).  For k = 0..K-1:
      C^k = C - eta log X^k                                   (line 3)
      Sinkhorn sweeps until ||grad P^k||_1 <= sink_tol or T1  (lines 4-8)
      sparse Newton until ||grad P^k||_1 <= newton_tol or T2  (lines 9-15)
      X^{k+1} = X~^{k*}(f, g)                                 (line 16)
    stop when the outer rule fires (reading R6).  The LP duals reported are
    u = (eta log a + sum_t f^t)/s, v = (eta log b + sum_t g^t - k eta)/s with
    s = k+1, so that log X^{k+1} = s (u e^T + e v^T - C)/eta exactly
    (Eq. (7) unrolled).
    """
    m, n = C.shape
    eta = prm.eta
    logX = np.log(a)[:, None] + np.log(b)[None, :]
    f = np.zeros(m)
    g = np.zeros(n)
    fsum = eta * np.log(a)
    gsum = eta * np.log(b)
    objs: List[float] = []
    sweeps = newton_its = cg_its = 0
    tr: List[Dict] = []
    k = 0
    Ck = shifted_cost(C, logX, eta)
    f_prev = g_prev = None
    for k in range(prm.K):
        Ck = shifted_cost(C, logX, eta)
        if not prm.warm_start:
            f = np.zeros(m)
            g = np.zeros(n)
        # warm_start 2 (reading R7): linear extrapolation 2 x^k - x^{k-1} of the last two
        # subproblem solutions, kept only if it needs no Sinkhorn phase
        f_sol, g_sol = f, g
        if prm.warm_start == 2 and f_prev is not None:
            f, g = 2.0 * f_sol - f_prev, 2.0 * g_sol - g_prev
        res = residual_l1(f, g, Ck, a, b, eta)
        if prm.warm_start == 2 and f_prev is not None and res > prm.sink_tol:
            f, g = f_sol, g_sol
            res = residual_l1(f, g, Ck, a, b, eta)
        if k >= 1:
            f_prev, g_prev = f_sol, g_sol
        t = 0
        while res > prm.sink_tol and t < prm.T1:
            f, g = sinkhorn_sweep(f, g, Ck, a, b, eta)
            res = residual_l1(f, g, Ck, a, b, eta)
            t += 1
        sweeps += t
        tn = 0
        while res > prm.newton_tol and tn < prm.T2:
            f, g, info = newton_step(f, g, Ck, a, b, eta, prm)
            cg_its += info["cg_iters"]
            res = residual_l1(f, g, Ck, a, b, eta)
            tn += 1
            if info["alpha"] == 0.0:
                break
        newton_its += tn
        logX = log_plan(f, g, Ck, eta)
        fsum = fsum + f
        gsum = gsum + g - eta
        obj = float((C * np.exp(logX)).sum())
        objs.append(obj)
        if trace:
            tr.append(dict(k=k, sweeps=t, newton=tn, res=res, obj=obj))
        if outer_converged(objs, prm):
            break
    s = k + 1
    u = fsum / s
    v = gsum / s
    dual = dual_objective(f, g, Ck, a, b, eta)
    return Result(logX=logX, f=f, g=g, u=u, v=v, obj=objs[-1], dual_obj=dual,
                  kkt=kkt(C, logX, a, b, u, v), outer_iters=k + 1, phi=fsum, psi=gsum,
                  s_next=float(k + 2), sweeps=sweeps,
                  newton_iters=newton_its, cg_iters=cg_its, trace=tr)


def outer_converged(objs: List[float], prm: Params) -> bool:
    """Outer stopping rule (reading R6 of A.2's "relative error threshold").

    rule 0: |obj_k - obj_{k-1}| <= tol |obj_k|
    rule 1: obj_{ceil(k/2)} - obj_k <= tol |obj_k|   (halving estimator: exact
            whenever the error decays at least like 1/k, Thm 4.1 monotonicity)
    rule 2: geometric tail.  With W = max(5, k//4), D1 = obj_{k-2W} - obj_{k-W},
            D2 = obj_{k-W} - obj_k, r = D2/D1: the remaining error of a sequence
            decaying like A q^k is D2 r/(1-r); stop when that is <= tol |obj_k|
            (r >= 1, i.e. no geometric decay yet, never stops).
    """
    k = len(objs)
    if k < 2:
        return False
    cur = objs[-1]
    scale = max(abs(cur), 1e-300)
    if prm.outer_rule == 0:
        return abs(cur - objs[-2]) <= prm.outer_tol * scale
    if prm.outer_rule == 1:
        half = objs[(k - 1) // 2]
        return (half - cur) <= prm.outer_tol * scale and k >= 4
    W = max(5, k // 4)
    if k < 2 * W + 1:
        return False
    D1 = objs[-1 - 2 * W] - objs[-1 - W]
    D2 = objs[-1 - W] - cur
    if D2 <= 0.0:
        return D1 >= 0.0 and abs(D2) <= prm.outer_tol * scale
    if D1 <= 0.0:
        return False
    r = D2 / D1
    if r >= 1.0:
        return False
    return D2 * r / (1.0 - r) <= prm.outer_tol * scale


def bregman(X: np.ndarray, Y: np.ndarray) -> float:
    """D_phi(X, Y) with phi(X) = sum X (log X - 1), 0 log 0 = 0."""
    with np.errstate(divide="ignore", invalid="ignore"):
        xlogx = np.where(X > 0, X * np.log(np.where(X > 0, X, 1.0)), 0.0)
    phiX = float((xlogx - X).sum())
    phiY = float((Y * (np.log(Y) - 1.0)).sum())
    return phiX - phiY - float((np.log(Y) * (X - Y)).sum())
