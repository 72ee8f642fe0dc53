"""Pins of the CPU oracle against things other than itself (no GPU).

Each test names the PAPER.md passage whose mathematics fixes the expected
value: closed forms, finite differences, invariants, brute force and the
independent exact LP (network simplex).
"""
import math

import numpy as np
import pytest

from oracle import pins_oracle as po
from oracle.exact_lp import brute_force_assignment, solve_exact

E1 = math.exp(-1.0)


# ---------------------------------------------------------------- Eq. (7)-(9)
def test_plan_closed_form():
    # Eq. (7) with f=g=0, C^k=0, eta=1: every entry exp(-1)
    X = po.plan(np.zeros(2), np.zeros(3), np.zeros((2, 3)), 1.0)
    assert np.allclose(X, E1, rtol=0, atol=1e-16)


def test_dual_objective_and_gradient_closed_form():
    # Eq. (8): P = 0 + 0 - 1 * 4 e^-1 ; Eq. (9): grad_f = 0.5 - 2 e^-1
    a = b = np.array([0.5, 0.5])
    P = po.dual_objective(np.zeros(2), np.zeros(2), np.zeros((2, 2)), a, b, 1.0)
    assert abs(P - (-4 * E1)) < 1e-15
    gf, gg = po.dual_gradient(np.zeros(2), np.zeros(2), np.zeros((2, 2)), a, b, 1.0)
    assert np.allclose(gf, 0.5 - 2 * E1, atol=1e-15) and np.allclose(gg, 0.5 - 2 * E1, atol=1e-15)


def test_gauge_invariance():
    # (f + c e, g - c e) leaves X~ unchanged and P unchanged when sum a = sum b = 1
    rng = np.random.default_rng(5)
    C = rng.random((4, 3)); a = np.full(4, .25); b = np.full(3, 1 / 3)
    f, g = rng.normal(size=4), rng.normal(size=3)
    X1 = po.plan(f, g, C, 0.3); X2 = po.plan(f + 0.7, g - 0.7, C, 0.3)
    assert np.allclose(X1, X2, rtol=1e-13)
    assert abs(po.dual_objective(f, g, C, a, b, .3) - po.dual_objective(f + .7, g - .7, C, a, b, .3)) < 1e-13


@pytest.mark.parametrize("eta", [1.0, 0.1])
def test_gradient_matches_finite_differences(eta):
    rng = np.random.default_rng(11)
    for _ in range(10):
        m, n = rng.integers(2, 7), rng.integers(2, 6)
        C = rng.random((m, n)); a = po_norm(rng.random(m) + .1); b = po_norm(rng.random(n) + .1)
        f, g = rng.normal(0, .3, m), rng.normal(0, .3, n)
        gf, gg = po.dual_gradient(f, g, C, a, b, eta)
        h = 1e-6
        for i in range(m):
            e = np.zeros(m); e[i] = h
            fd = (po.dual_objective(f + e, g, C, a, b, eta) - po.dual_objective(f - e, g, C, a, b, eta)) / (2 * h)
            assert abs(fd - gf[i]) <= 1e-6 * (1 + abs(gf).max())
        for j in range(n):
            e = np.zeros(n); e[j] = h
            fd = (po.dual_objective(f, g + e, C, a, b, eta) - po.dual_objective(f, g - e, C, a, b, eta)) / (2 * h)
            assert abs(fd - gg[j]) <= 1e-6 * (1 + abs(gg).max())


@pytest.mark.parametrize("eta", [1.0, 0.1])
def test_hessian_matches_finite_differences(eta):
    rng = np.random.default_rng(12)
    for _ in range(10):
        m, n = rng.integers(2, 7), rng.integers(2, 6)
        C = rng.random((m, n)); a = po_norm(rng.random(m) + .1); b = po_norm(rng.random(n) + .1)
        f, g = rng.normal(0, .3, m), rng.normal(0, .3, n)
        H = po.hessian_dense(f, g, C, eta)
        h = 1e-5
        for k in range(m + n):
            d = np.zeros(m + n); d[k] = h
            gp = np.concatenate(po.dual_gradient(f + d[:m], g + d[m:], C, a, b, eta))
            gm = np.concatenate(po.dual_gradient(f - d[:m], g - d[m:], C, a, b, eta))
            fd = (gp - gm) / (2 * h)
            assert np.abs(fd - H[:, k]).max() <= 1e-5 * (1 + np.abs(H).max())


def test_hessian_null_vector():
    # Eq. (9): [[diag(Xe), X],[X^T, diag(X^T e)]] (e_m, -e_n) = 0
    rng = np.random.default_rng(3)
    C = rng.random((5, 4)); f, g = rng.normal(size=5), rng.normal(size=4)
    H = po.hessian_dense(f, g, C, 0.5)
    z = np.concatenate([np.ones(5), -np.ones(4)])
    assert np.abs(H @ z).max() <= 1e-12 * np.abs(H).max()


def po_norm(v):
    return v / v.sum()


# ------------------------------------------------------------------- Sinkhorn
def test_sinkhorn_marginals_exact_after_updates():
    # Alg. 2 line 5: after the f-update the rows of X~(f^{t+1}, g^t) sum to a;
    # line 6: after the g-update the columns sum to b.
    rng = np.random.default_rng(8)
    C = rng.random((10, 10)); a = po_norm(rng.random(10) + .1); b = po_norm(rng.random(10) + .1)
    f, g = np.zeros(10), np.zeros(10)
    prev = -np.inf
    for _ in range(200):
        f1, g1 = po.sinkhorn_sweep(f, g, C, a, b, 0.05)
        rows = po.plan(f1, g, C, 0.05).sum(1)
        assert np.abs(rows - a).sum() <= 1e-12
        cols = po.plan(f1, g1, C, 0.05).sum(0)
        assert np.abs(cols - b).sum() <= 1e-12
        P = po.dual_objective(f1, g1, C, a, b, 0.05)
        assert P >= prev - 1e-12          # exact alternating maximisation
        prev, f, g = P, f1, g1


def test_sinkhorn_constant_cost_gives_product_plan():
    # C = c E: one sweep lands on X = a b^T (rank-one scaling stays rank one)
    rng = np.random.default_rng(1)
    a = po_norm(rng.random(6) + .1); b = po_norm(rng.random(4) + .1)
    C = np.full((6, 4), 0.37)
    f, g = po.sinkhorn_sweep(np.zeros(6), np.zeros(4), C, a, b, 0.1)
    assert np.allclose(po.plan(f, g, C, 0.1), np.outer(a, b), rtol=1e-13, atol=0)


def test_sinkhorn_single_cell():
    f, g = po.sinkhorn_sweep(np.zeros(1), np.zeros(1), np.array([[0.4]]), np.ones(1), np.ones(1), 0.01)
    assert abs(po.plan(f, g, np.array([[0.4]]), 0.01)[0, 0] - 1.0) < 1e-14


# ------------------------------------------------------------- sparsify / CG
def test_sparsify_threshold_and_topk():
    P = np.array([[4.0, 1.0], [3.0, 2.0]])
    assert (po.sparsify_topk(P, 0.5) == np.array([[True, False], [True, False]])).all()
    assert po.sparsify_topk(P, 1.0).all()
    assert (po.sparsify_threshold(P, 2.0) == np.array([[True, False], [True, True]])).all()
    rp, ci, v = po.csr_from_mask(P, po.sparsify_threshold(P, 2.0))
    assert list(rp) == [0, 1, 3] and list(ci) == [0, 0, 1] and list(v) == [4.0, 3.0, 2.0]


def test_cg_small_spd():
    A = np.array([[4.0, 1.0], [1.0, 3.0]])
    x, its, res = po.cg(lambda p: A @ p, np.array([1.0, 2.0]), 1e-14, 10)
    assert np.allclose(x, [1 / 11, 7 / 11], atol=1e-14)
    rng = np.random.default_rng(2)
    B = rng.normal(size=(30, 30)); A = B @ B.T + 30 * np.eye(30); rhs = rng.normal(size=30)
    x, its, res = po.cg(lambda p: A @ p, rhs, 1e-12, 200, diag=np.diag(A))
    assert np.allclose(x, np.linalg.solve(A, rhs), rtol=1e-9, atol=1e-12)


def test_newton_direction_is_exact_newton_without_sparsification():
    # With theta = 0 (keep everything), mu -> 0 and a tight CG, the direction
    # solves the Newton system of Eq. (9):  hess P d = -grad P  (min-norm sense).
    rng = np.random.default_rng(4)
    m, n, eta = 6, 5, 0.2
    C = rng.random((m, n)); a = po_norm(rng.random(m) + .1); b = po_norm(rng.random(n) + .1)
    f, g = np.zeros(m), np.zeros(n)
    for _ in range(5):
        f, g = po.sinkhorn_sweep(f, g, C, a, b, eta)
    prm = po.Params(theta=0.0, cg_tol=1e-12, cg_forcing=0.0, cg_maxit=500)
    df, dg, info = po.newton_direction(f, g, C, a, b, eta, prm)
    H = po.hessian_dense(f, g, C, eta)
    grad = np.concatenate(po.dual_gradient(f, g, C, a, b, eta))
    d = np.concatenate([df, dg])
    assert np.abs(H @ d + grad).max() <= 1e-10
    # quadratic convergence: two Newton steps shrink the gradient sharply
    res0 = np.abs(grad).sum()
    f1, g1, _ = po.newton_step(f, g, C, a, b, eta, prm)
    f2, g2, _ = po.newton_step(f1, g1, C, a, b, eta, prm)
    assert po.residual_l1(f2, g2, C, a, b, eta) < 1e-4 * res0


# ------------------------------------------------------------------ PINS (Alg. 2)
def test_pins_identity_with_annealed_entropic_ot():
    # Eq. (5)-(7): with X^0 = a b^T and subproblems solved to high accuracy,
    # X^{k} = argmin <C,X> + (eta/k) sum X log X over the polytope (the shifted
    # costs C^k are k C up to separable terms).  Independent check: plain
    # Sinkhorn on C with regularisation eta/k.
    rng = np.random.default_rng(9)
    m, n, eta, K = 7, 6, 0.2, 4
    C = rng.random((m, n)); a = po_norm(rng.random(m) + .1); b = po_norm(rng.random(n) + .1)
    prm = po.Params(eta=eta, K=K, outer_tol=0.0, sink_tol=1e-13, T1=100000, newton_tol=1e-14)
    r = po.pins(C, a, b, prm)
    epsk = eta / K
    f, g = np.zeros(m), np.zeros(n)
    for _ in range(20000):
        f, g = po.sinkhorn_sweep(f, g, C, a, b, epsk)
    Xent = po.plan(f, g, C, epsk)
    assert np.abs(np.exp(r.logX) - Xent).max() <= 1e-9


def test_pins_uniform_square_matches_brute_force():
    rng = np.random.default_rng(21)
    for n in (3, 5, 6):
        C = rng.random((n, n)); a = np.full(n, 1.0 / n)
        _, opt = brute_force_assignment(C)
        prm = po.Params(eta=0.05, K=4000, outer_rule=1, outer_tol=1e-8, newton_tol=1e-12)
        r = po.pins(C, a, a.copy(), prm, trace=True)
        assert abs(r.obj - opt) <= 1e-7 * abs(opt)
        assert r.kkt["primal"] <= 1e-8
        objs = [t["obj"] for t in r.trace]
        # Thm 4.1 proof: <C,X^{k+1}> <= <C,X^k>
        assert all(objs[i + 1] <= objs[i] + 1e-12 for i in range(len(objs) - 1)), max(np.diff(objs))


def test_pins_rectangular_matches_network_simplex_and_bregman_monotone():
    rng = np.random.default_rng(22)
    m, n = 9, 7
    C = rng.random((m, n)); a = po_norm(rng.random(m) + .1); b = po_norm(rng.random(n) + .1)
    ex = solve_exact(C, a, b)
    prm = po.Params(eta=0.05, K=3000, outer_rule=1, outer_tol=1e-8, newton_tol=1e-12)
    r = po.pins(C, a, b, prm, trace=True)
    assert abs(r.obj - ex["obj"]) <= 1e-7 * abs(ex["obj"])
    # Bregman monotonicity toward X* (Thm 4.1 proof): re-run
    # the outer loop step by step and track D(X*, X^k)
    Xs = ex["X"]
    prm2 = po.Params(eta=0.05, K=1, outer_tol=0.0, newton_tol=1e-13)
    logX = np.log(a)[:, None] + np.log(b)[None, :]
    f, g = np.zeros(m), np.zeros(n)
    prev = po.bregman(Xs, np.exp(logX))
    for _ in range(30):
        Ck = po.shifted_cost(C, logX, 0.05)
        for _ in range(200):
            f, g = po.sinkhorn_sweep(f, g, Ck, a, b, 0.05)
        for _ in range(5):
            f, g, _ = po.newton_step(f, g, Ck, a, b, 0.05, prm2)
        logX = po.log_plan(f, g, Ck, 0.05)
        D = po.bregman(Xs, np.exp(logX))
        assert D <= prev + 1e-9
        prev = D


def test_kkt_of_exact_solution_is_zero():
    rng = np.random.default_rng(23)
    C = rng.random((6, 8)); a = po_norm(rng.random(6) + .1); b = po_norm(rng.random(8) + .1)
    ex = solve_exact(C, a, b)
    X = ex["X"]
    assert np.abs(X.sum(1) - a).sum() + np.abs(X.sum(0) - b).sum() <= 1e-14
    assert (ex["u"][:, None] + ex["v"][None, :] - C).max() <= 1e-12
    assert abs((C * X).sum() - a @ ex["u"] - b @ ex["v"]) <= 1e-13


def test_outer_rules():
    prm = po.Params(outer_rule=0, outer_tol=1e-4)
    assert po.outer_converged([1.0, 1.0], prm)
    assert not po.outer_converged([1.0, 0.99989], prm)   # SPEC example: change 1.1e-4
    prm1 = po.Params(outer_rule=1, outer_tol=1e-3)
    seq = [1 + 1.0 / (k + 1) for k in range(4000)]
    k_stop = next(k for k in range(2, 4000) if po.outer_converged(seq[:k], prm1))
    # error 1/k halves when k doubles: the halving estimate is exact for 1/k
    assert abs(1.0 / k_stop - 1e-3) < 2e-4


@pytest.mark.parametrize("warm", [0, 1, 2])
def test_pins_warm_start_variants_reach_exact_lp(warm):
    # every warm-start reading (R7: zero, carry, safeguarded extrapolation) is only an
    # initial point of subproblem (6); PINS must still reach the exact optimum of Eq. (1)
    rng = np.random.default_rng(21)
    m, n = 9, 7
    C = rng.random((m, n))
    a = rng.random(m) + 0.2; a /= a.sum()
    b = rng.random(n) + 0.2; b /= b.sum()
    ex = solve_exact(C, a, b)
    r = po.pins(C, a, b, po.Params(eta=0.05, K=4000, outer_rule=1, outer_tol=1e-9, newton_tol=1e-11,
                                    warm_start=warm))
    assert abs(r.obj - ex["obj"]) <= 1e-7 * abs(ex["obj"])
    assert r.kkt["primal"] <= 1e-9


# ------------------------------------------------------------------ remaining pins
def test_cost_matrix_closed_form_and_scaling():
    # input definition: squared-Euclidean / L1 distances of lattice points,
    # scaled so that the largest entry is 1; 3-4-5 triangle gives D = 25 (sq) and 7 (L1)
    from workloads.gen import _points_workload, COST_SQEUCLID, COST_L1
    X = np.array([[0.0, 0.0], [3.0, 4.0]])
    Y = np.array([[0.0, 0.0], [3.0, 0.0]])
    a = b = np.array([0.5, 0.5])
    w = _points_workload("t", X, Y, COST_SQEUCLID, a, b, 0.1)
    C = po.cost_matrix(w)
    np.testing.assert_allclose(C * 25.0, [[0.0, 9.0], [25.0, 16.0]], rtol=0, atol=1e-13)
    w = _points_workload("t", X, Y, COST_L1, a, b, 0.1)
    C = po.cost_matrix(w)
    np.testing.assert_allclose(C * 7.0, [[0.0, 3.0], [7.0, 4.0]], rtol=0, atol=1e-13)
    assert C.max() == 1.0


def test_logsumexp_identities():
    # log sum exp = log(sum(exp)) for moderate values; exact shift invariance for huge ones
    rng = np.random.default_rng(3)
    A = rng.normal(size=(5, 7))
    np.testing.assert_allclose(po.logsumexp(A, 1), np.log(np.exp(A).sum(1)), rtol=1e-14)
    np.testing.assert_allclose(po.logsumexp(A + 1000.0, 0), np.log(np.exp(A).sum(0)) + 1000.0, rtol=1e-14)
    B = np.array([[-np.inf, 0.0], [-np.inf, -np.inf]])
    with np.errstate(divide="ignore"):
        L = po.logsumexp(B, 1)
    assert L[0] == 0.0 and L[1] == -np.inf


def test_inexact_newton_direction_meets_its_forcing_residual():
    # Reading R5 (inexact Newton): the direction returned by newton_direction solves the
    # damped sparsified Newton system M d = eta grad P to the forcing tolerance.  The
    # residual is recomputed here from a DENSE assembly of M (Eq. (9) blocks, diagonal
    # blocks exact, off-diagonal thresholded at tau), independently of the oracle's matvec.
    rng = np.random.default_rng(21)
    m, n, eta = 9, 7, 0.1
    Ck = rng.random((m, n))
    a = po_norm(rng.random(m) + 0.1); b = po_norm(rng.random(n) + 0.1)
    f, g = rng.normal(0, 0.05, m), rng.normal(0, 0.05, n)
    for forcing, newton_tol in ((0.1, 1e-3), (0.0, 1e-8)):
        prm = po.Params(eta=eta, cg_forcing=forcing, newton_tol=newton_tol, cg_tol=1e-9, theta=1e-2)
        df, dg, info = po.newton_direction(f, g, Ck, a, b, eta, prm)
        X = np.exp((f[:, None] + g[None, :] - Ck - eta) / eta)
        tau = 1e-2 / (m * n)
        Xs = np.where(X >= tau, X, 0.0)
        r, c = X.sum(1), X.sum(0)
        mu = 1e-10 * max(r.max(), c.max())
        M = np.block([[np.diag(r), Xs], [Xs.T, np.diag(c)]]) + mu * np.eye(m + n)
        rhs = eta * np.concatenate([a - r, b - c])
        d = np.concatenate([df, dg])
        rel = np.linalg.norm(M @ d - rhs) / np.linalg.norm(rhs)
        gnorm = np.abs(a - r).sum() + np.abs(b - c).sum()
        want = min(0.5, max(1e-9, forcing * newton_tol / gnorm)) if forcing > 0 else 1e-9
        assert rel <= want * (1 + 1e-6) + 1e-13
        if forcing > 0:
            assert want > 1e-6 and info["cg_iters"] < m + n      # a loose solve stops early


def test_dual_increase_matches_direct_difference():
    # Eq. (8) rearranged (reading R4) equals P(x + alpha d) - P(x) where the direct
    # difference is well conditioned
    rng = np.random.default_rng(8)
    m, n, eta = 4, 5, 0.3
    Ck = rng.random((m, n))
    a = po_norm(rng.random(m) + 0.1); b = po_norm(rng.random(n) + 0.1)
    f, g = rng.normal(0, 0.2, m), rng.normal(0, 0.2, n)
    df, dg = rng.normal(0, 0.1, m), rng.normal(0, 0.1, n)
    for alpha in (1.0, 0.25):
        direct = (po.dual_objective(f + alpha * df, g + alpha * dg, Ck, a, b, eta)
                  - po.dual_objective(f, g, Ck, a, b, eta))
        assert abs(po.dual_increase(f, g, df, dg, alpha, Ck, a, b, eta) - direct) <= 1e-14


def test_line_search_returns_largest_armijo_step():
    # backtracking (reading R4): the accepted alpha satisfies the
    # Armijo condition and 2 alpha (if tried) does not
    rng = np.random.default_rng(9)
    m, n, eta = 6, 5, 0.05
    Ck = rng.random((m, n))
    a = po_norm(rng.random(m) + 0.1); b = po_norm(rng.random(n) + 0.1)
    f, g = np.zeros(m), np.zeros(n)
    prm = po.Params(eta=eta)
    gf, gg = po.dual_gradient(f, g, Ck, a, b, eta)
    df, dg = 40.0 * gf, 40.0 * gg            # an over-long ascent direction forces backtracking
    alpha, inc = po.line_search(f, g, df, dg, Ck, a, b, eta, prm)
    slope = float(gf @ df + gg @ dg)
    assert 0.0 < alpha < 1.0
    assert inc >= prm.armijo_c * alpha * slope
    big = 2.0 * alpha
    assert po.dual_increase(f, g, df, dg, big, Ck, a, b, eta) < prm.armijo_c * big * slope


def test_kkt_of_exact_lp_solution():
    # residuals of Eq. (1) at the network simplex optimum and its dual certificate:
    # feasible plan, dual feasible up to rounding, zero duality gap
    rng = np.random.default_rng(12)
    m, n = 7, 9
    C = rng.random((m, n))
    a = po_norm(rng.random(m) + 0.1); b = po_norm(rng.random(n) + 0.1)
    ex = solve_exact(C, a, b)
    with np.errstate(divide="ignore"):
        logX = np.log(ex["X"])
    k = po.kkt(C, logX, a, b, ex["u"], ex["v"])
    assert k["primal"] <= 1e-14 and k["dual_inf"] <= 1e-13 and abs(k["gap"]) <= 1e-13


def test_outer_rule_geometric_tail_is_exact_for_geometric_sequences():
    # rule 2 (reading R6): for obj_k = L + A q^k the estimator D2 r / (1 - r) equals the
    # true remaining error obj_k - L exactly, so the rule stops at the FIRST k whose true
    # error is <= tol |obj_k| (and not earlier), once k >= 2W + 1
    L, A, q, tol = 0.37, 0.05, 0.8, 1e-6
    prm = po.Params(outer_rule=2, outer_tol=tol)
    objs, stop = [], None
    for k in range(400):
        objs.append(L + A * q ** k)
        if po.outer_converged(objs, prm):
            stop = len(objs)
            break
    assert stop is not None
    W = max(5, stop // 4)
    err = lambda K: objs[K - 1] - L
    assert err(stop) <= tol * objs[stop - 1] * (1 + 1e-9)
    # the step before either had a larger true error or was too short for the estimator
    prev = stop - 1
    assert err(prev) > tol * objs[prev - 1] * (1 - 1e-9) or prev < 2 * max(5, prev // 4) + 1
    # monotone sequences (Thm 4.1) decaying slower than any q^k never stop at this tol
    objs = [L + A / (k + 1) for k in range(300)]
    assert not any(po.outer_converged(objs[:K], prm) for K in range(2, 300))
    # a sequence that is still decreasing by more than tol per window never stops
    objs = [L + A * (1 - 1e-3 * k) for k in range(300)]
    assert not any(po.outer_converged(objs[:K], prm) for K in range(2, 300))


def test_bregman_divergence_closed_forms():
    # D_phi(X, Y) with phi = sum X (log X - 1) is the generalised KL
    # divergence sum X log(X/Y) - X + Y (0 log 0 = 0): pinned on hand-computed values
    Y = np.full((2, 2), 0.25)
    X = np.array([[0.5, 0.0], [0.0, 0.5]])
    assert po.bregman(X, Y) == pytest.approx(np.log(2.0), rel=1e-15)          # 2 (0.5 log 2) - 1 + 1
    assert po.bregman(Y, Y) == 0.0 or abs(po.bregman(Y, Y)) <= 1e-16
    X2 = np.array([[1.0, 2.0], [3.0, 4.0]])
    Y2 = np.array([[2.0, 1.0], [1.0, 1.0]])
    hand = (1 * np.log(0.5) + 2 * np.log(2) + 3 * np.log(3) + 4 * np.log(4)) - 10.0 + 5.0
    assert po.bregman(X2, Y2) == pytest.approx(hand, rel=1e-14)
    # scaling: D(cX, cY) = c D(X, Y); and D(X, Y) > 0 for X != Y
    assert po.bregman(3 * X2, 3 * Y2) == pytest.approx(3 * hand, rel=1e-14)
    assert po.bregman(Y2, X2) > 0
