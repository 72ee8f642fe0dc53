"""GPU parity: every hot-path call through the C ABI against the CPU oracle on
the same seeded inputs (Eq. (7)-(9), Alg. 1/2, §3.2).

Subproblem states (centre X^k and warm potentials) are produced by running
the ORACLE's PINS for k outer iterations; the GPU receives the centre in its
factored log form (phi, psi, s), the oracle keeps its dense C^k = C - eta log X^k.
Agreement therefore also checks the factorisation identity of DESIGN.md §2.

Tolerances (derived in DESIGN.md §6): plan entries and sums are fp64 with
exponents of magnitude |z| <= s max C / eta, so relative errors are bounded by
~1e-16 * |z|; we allow 1e-11 relative (+ small absolute floors).
"""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pins_oracle as po  # noqa: E402
from oracle import lp_certificate as lc  # noqa: E402
from oracle.exact_lp import solve_exact  # noqa: E402
from workloads import make  # noqa: E402
from workloads.gen import COST_DENSE, Workload  # noqa: E402

SKIP = math.exp(-80.0)     # sum-pass skip threshold on X~ (pins_pass.cuh kSumCut)
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def P():
    from paper_2502_03749_b200 import build as b
    b.build()
    from paper_2502_03749_b200 import pins
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return pins


def T(x):
    return torch.as_tensor(np.asarray(x), dtype=torch.float64, device="cuda").contiguous()


def H(t):
    return t.detach().cpu().numpy()


def ragged(m, n, seed, kind="dense", d=3, real=False):
    """Ragged-size instance (not multiples of the 128-row tile / 32-column chunk);
    real=True draws real-valued points (fp64 cost paths), else lattice points."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.1, 1, m); a /= a.sum()
    b = rng.uniform(0.1, 1, n); b /= b.sum()
    if kind == "dense":
        return Workload("ragged", m, n, COST_DENSE, a, b, 0.05, C=rng.random((m, n)))
    X = rng.random((m, d)) * 1024; Y = rng.random((n, d)) * 1024
    if real:
        X, Y = X / 1024.0 - 0.5, Y / 1024.0 - 0.5
    else:
        X, Y = np.floor(X), np.floor(Y)
    from workloads.gen import _points_workload, COST_SQEUCLID, COST_L1
    return _points_workload("ragged_pts", X, Y, COST_SQEUCLID if kind == "sq" else COST_L1, a, b, 0.05)


CASES = [
    ("c0", lambda: make("c0_pts64")),
    ("c1s", lambda: make("c1_rand1k", scale=0.11)),
    ("c2s", lambda: make("c2_img4k", scale=0.06)),
    ("c3s", lambda: make("c3_gmm10k", scale=0.013)),
    ("c4s", lambda: make("c4_l1rect", scale=0.012)),
    ("rag_dense", lambda: ragged(37, 1029, 5)),           # odd pitch: thread-staged dense path
    ("c1t", lambda: make("c1_rand1k", scale=0.125)),      # 128 x 128: TMA-staged dense path
    ("rag_dense_t", lambda: ragged(37, 1030, 15)),        # even pitch, ragged: TMA path, partial tiles
    ("rag_sq", lambda: ragged(70, 515, 6, "sq", 10)),
    ("rag_l1", lambda: ragged(33, 17, 7, "l1", 3)),
    # real-valued point sets (BASELINE.json as written): fp64 cost paths PC_SQ64 / PC_L164
    ("c0r", lambda: make("c0_pts64_r")),
    ("c3rs", lambda: make("c3_gmm10k_r", scale=0.013)),
    ("c4rs", lambda: make("c4_l1rect_r", scale=0.012)),
    ("rag_sq_r", lambda: ragged(70, 515, 16, "sq", 10, real=True)),
    ("rag_l1_r", lambda: ragged(133, 47, 17, "l1", 3, real=True)),
]
# Newton-step cases: the five configurations (scaled) plus the real-valued variants
NEWTON_CASES = CASES[:5] + [c for c in CASES if c[0] in ("c0r", "c3rs", "c4rs")]


def oracle_state(w, k, **kw):
    """Oracle PINS after k outer iterations: (C, C^k dense, phi, psi, s, f, g)."""
    C = po.cost_matrix(w)
    prm = po.Params(eta=w.eta, K=k, outer_tol=0.0, newton_tol=1e-10, **kw)
    r = po.pins(C, w.a, w.b, prm)
    Ck = po.shifted_cost(C, r.logX, w.eta)
    return C, Ck, r.phi, r.psi, r.s_next, r.f, r.g


@pytest.mark.parametrize("name,mk", CASES)
@pytest.mark.parametrize("k", [0, 3])
def test_plan_and_evaluate(P, name, mk, k):
    w = mk()
    if k == 0:
        C = po.cost_matrix(w)
        Ck = po.shifted_cost(C, np.log(w.a)[:, None] + np.log(w.b)[None, :], w.eta)
        phi, psi, s = w.eta * np.log(w.a), w.eta * np.log(w.b), 1.0
        rng = np.random.default_rng(1)
        f, g = rng.normal(0, 0.3 * w.eta, w.m), rng.normal(0, 0.3 * w.eta, w.n)
    else:
        C, Ck, phi, psi, s, f, g = oracle_state(w, k)
    pb = P.DeviceProblem.from_workload(w)
    X = H(P.plan(pb, T(phi), T(psi), s, T(f), T(g)))
    Xo = po.plan(f, g, Ck, w.eta)
    scale = max(1.0, s * C.max() / w.eta)
    np.testing.assert_allclose(X, Xo, rtol=4e-15 * scale, atol=1e-300)
    ws = P.Workspace()
    ev = P.evaluate(ws, pb, T(phi), T(psi), s, T(f), T(g))
    gf, gg = po.dual_gradient(f, g, Ck, w.a, w.b, w.eta)
    # entries below e^-80 are not evaluated (skip rule): absolute floor n e^-80
    np.testing.assert_allclose(H(ev["r"]), Xo.sum(1), rtol=4e-15 * scale, atol=w.n * SKIP)
    np.testing.assert_allclose(H(ev["c"]), Xo.sum(0), rtol=4e-15 * scale, atol=w.m * SKIP)
    gn = np.abs(gf).sum() + np.abs(gg).sum()
    assert abs(ev["grad_l1"] - gn) <= 1e-14 * scale * (1 + gn)
    assert abs(ev["sum_x"] - Xo.sum()) <= 1e-14 * scale * Xo.sum()
    assert abs(ev["cost"] - (C * Xo).sum()) <= 1e-13 * scale * abs((C * Xo).sum()) + 1e-300
    Po = po.dual_objective(f, g, Ck, w.a, w.b, w.eta)
    # P^k itself is large relative to its changes; compare in the scale of its terms
    assert abs(ev["dual_obj"] - Po) <= 1e-13 * (abs(w.a @ f) + abs(w.b @ g) + w.eta * Xo.sum() + 1)


@pytest.mark.parametrize("name,mk", CASES)
def test_sparsify_pattern_in_eval_matches_threshold(P, name, mk):
    # The PRODUCTION sparsifier (sum pass compaction + csr_build, Alg. 2
    # line 11) on identical P: pins_plan materialises X~(f, g) with the same exponent
    # expression and exp as the sum pass (pins_pass.cuh plan_kernel), so the CSR of
    # pins_evaluate(tau) must equal the oracle's threshold of THAT plan bit for bit --
    # rowptr, colidx and values -- with no tolerance band, including entries exactly at tau.
    w = mk()
    C, Ck, phi, psi, s, f, g = oracle_state(w, 2)
    pb = P.DeviceProblem.from_workload(w)
    Pg = H(P.plan(pb, T(phi), T(psi), s, T(f), T(g)))
    tau0 = 1e-4 / (w.m * w.n)
    # planted threshold: an actual entry value, so ties X~_ij == tau occur (kept: >= tau)
    cand = np.sort(Pg[Pg >= tau0].ravel())
    taus = [tau0] + ([float(cand[len(cand) // 2])] if len(cand) else [])
    for tau in taus:
        ws = P.Workspace()
        ev = P.evaluate(ws, pb, T(phi), T(psi), s, T(f), T(g), tau=tau)
        rp, ci, va = (H(t_) for t_ in P.get_csr(ws))
        rpo, cio, vao = po.csr_from_mask(Pg, po.sparsify_threshold(Pg, tau))
        assert np.array_equal(rp, rpo)
        assert np.array_equal(ci, cio)
        assert np.array_equal(va.view(np.uint64), vao.view(np.uint64))
        assert ev["nnz"] == len(ci)
        if tau != tau0:
            assert np.count_nonzero(Pg == tau) >= 1 and np.count_nonzero(va == tau) == np.count_nonzero(Pg == tau)
    # and the plan itself is the oracle's (Eq. (7)) to rounding: patterns agree away from tau
    Xo = po.plan(f, g, Ck, w.eta)
    scale = max(1.0, s * C.max() / w.eta)
    near = np.abs(Xo - tau0) <= 4e-14 * scale * tau0
    assert np.array_equal(po.sparsify_threshold(Xo, tau0) & ~near, po.sparsify_threshold(Pg, tau0) & ~near)


@pytest.mark.parametrize("shape", [(1, 1), (3, 700), (64, 64), (37, 1029), (300, 5)])
def test_sparsify_dense_bit_exact(P, shape):
    # identical P on both sides: the CSR pattern must match bit for bit,
    # including entries exactly equal to tau (kept: P >= tau).
    m, n = shape
    rng = np.random.default_rng(m * 1000 + n)
    Pm = rng.random((m, n)) ** 4
    tau = 0.3
    Pm[rng.random((m, n)) < 0.05] = tau
    ws = P.Workspace()
    rp, ci, va = (H(t) for t in P.sparsify_dense(ws, T(Pm), tau))
    rpo, cio, vao = po.csr_from_mask(Pm, po.sparsify_threshold(Pm, tau))
    assert np.array_equal(rp, rpo) and np.array_equal(ci, cio) and np.array_equal(va, vao)


@pytest.mark.parametrize("name,mk", CASES)
@pytest.mark.parametrize("k", [0, 2])
def test_sinkhorn_sweep(P, name, mk, k):
    w = mk()
    if k == 0:
        C = po.cost_matrix(w)
        Ck = po.shifted_cost(C, np.log(w.a)[:, None] + np.log(w.b)[None, :], w.eta)
        phi, psi, s = w.eta * np.log(w.a), w.eta * np.log(w.b), 1.0
        f, g = np.zeros(w.m), np.zeros(w.n)
    else:
        C, Ck, phi, psi, s, f, g = oracle_state(w, k)
    pb = P.DeviceProblem.from_workload(w)
    ws = P.Workspace()
    fd, gd = T(f), T(g)
    for _ in range(3):
        P.sinkhorn_sweep(ws, pb, T(phi), T(psi), s, fd, gd)
        f, g = po.sinkhorn_sweep(f, g, Ck, w.a, w.b, w.eta)
    scale = max(1.0, s * C.max() / w.eta)
    tol = 1e-14 * scale * w.eta * 10
    np.testing.assert_allclose(H(fd), f, rtol=0, atol=tol * (1 + np.abs(f).max() / w.eta))
    np.testing.assert_allclose(H(gd), g, rtol=0, atol=tol * (1 + np.abs(g).max() / w.eta))


@pytest.mark.parametrize("name,mk", [c for c in CASES if c[0] in ("c0", "c1s", "c3s", "c4s", "c3rs", "rag_l1_r")])
def test_sinkhorn_phase(P, name, mk):
    # Alg. 2 lines 4-8: sweeps until ||grad P^k||_1 <= tol, run on the
    # device (pins_sinkhorn); stops at exactly the oracle's sweep count
    w = mk()
    C, Ck, phi, psi, s, f, g = oracle_state(w, 2)
    f = f + np.random.default_rng(5).normal(0, 2 * w.eta, w.m)      # away from the optimum
    tol = 1e-6
    pb = P.DeviceProblem.from_workload(w)
    ws = P.Workspace()
    fd, gd = T(f), T(g)
    t_gpu, res_gpu = P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, tol, 5000)
    t_o, res_o = 0, po.residual_l1(f, g, Ck, w.a, w.b, w.eta)
    while res_o > tol and t_o < 5000:
        f, g = po.sinkhorn_sweep(f, g, Ck, w.a, w.b, w.eta)
        res_o = po.residual_l1(f, g, Ck, w.a, w.b, w.eta)
        t_o += 1
    assert t_o > 1
    assert t_gpu == t_o
    assert abs(res_gpu - res_o) <= 1e-3 * tol + 1e-8 * res_o
    assert res_gpu <= tol or t_gpu == 5000          # converged, or both hit the sweep budget
    scale = max(1.0, s * C.max() / w.eta)
    tol_f = 1e-13 * scale * w.eta * (1 + t_o)
    np.testing.assert_allclose(H(fd), f, rtol=0, atol=tol_f * (1 + np.abs(f).max() / w.eta))
    np.testing.assert_allclose(H(gd), g, rtol=0, atol=tol_f * (1 + np.abs(g).max() / w.eta))


def test_cg_against_direct_solve(P):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    w = make("c1_rand1k", scale=0.1)
    C, Ck, phi, psi, s, f, g = oracle_state(w, 2)
    Xo = po.plan(f, g, Ck, w.eta)
    tau = 1e-4 / (w.m * w.n)
    rp, ci, va = po.csr_from_mask(Xo, po.sparsify_threshold(Xo, tau))
    r, c = Xo.sum(1), Xo.sum(0)
    m, n = w.m, w.n
    mu = 1e-8
    Xs = sp.csr_matrix((va, ci, rp), shape=(m, n))
    M = sp.bmat([[sp.diags(r), Xs], [Xs.T, sp.diags(c)]]).tocsc() + mu * sp.eye(m + n)
    rhs = np.random.default_rng(3).normal(size=m + n)
    x_ref = spla.spsolve(M, rhs)
    ws = P.Workspace()
    x, its, rel = P.cg(ws, m, n, torch.as_tensor(rp, device="cuda"), torch.as_tensor(ci.astype(np.int32), device="cuda"),
                       T(va), T(r), T(c), mu, T(rhs), rtol=1e-12, maxit=20000)
    assert rel <= 1e-12
    res = np.linalg.norm(M @ H(x) - rhs) / np.linalg.norm(rhs)
    # true residual vs the recursive one: q = M z + beta q drifts by O(its * eps * cond)
    assert res <= 1e-10
    # oracle CG (same algorithm, same preconditioner) reaches the same solution
    xo, _, _ = po.cg(lambda p: M @ p, rhs, 1e-12, 20000, diag=np.concatenate([r, c]) + mu)
    np.testing.assert_allclose(H(x), xo, rtol=1e-6, atol=1e-9 * np.abs(xo).max())
    np.testing.assert_allclose(H(x), x_ref, rtol=1e-6, atol=1e-9 * np.abs(x_ref).max())


@pytest.mark.parametrize("cg", ["tree", "treecl", "cluster", "grid"])
@pytest.mark.parametrize("name,mk", NEWTON_CASES)
def test_newton_step(P, name, mk, cg, monkeypatch):
    # the three Newton-system solvers: spanning-tree PCG (one CTA),
    # Jacobi-Schur CG (one cluster), Jacobi CG on the full system (cooperative grid)
    monkeypatch.setenv("PINS_CG", cg)
    w = mk()
    C, Ck, phi, psi, s, f, g = oracle_state(w, 2)
    # start away from the subproblem optimum: one plain sweep from the warm start
    prm_o = po.Params(eta=w.eta, cg_tol=1e-12, cg_forcing=0.0, cg_maxit=5000)
    prm_g = P.default_params(cg_tol=1e-12, cg_forcing=0.0, cg_maxit=5000)
    pb = P.DeviceProblem.from_workload(w)
    ws = P.Workspace()
    fd, gd = T(f), T(g)
    for _ in range(2):
        info = P.newton_step(ws, pb, prm_g, T(phi), T(psi), s, fd, gd)
        f2, g2, io = po.newton_step(f, g, Ck, w.a, w.b, w.eta, prm_o)
        assert info["alpha"] == io["alpha"]
        assert info["nnz"] == io["nnz"] or abs(info["nnz"] - io["nnz"]) <= 2
        dnorm = np.abs(f2 - f).max() + np.abs(g2 - g).max()
        np.testing.assert_allclose(H(fd), f2, rtol=0, atol=1e-7 * dnorm + 1e-13)
        np.testing.assert_allclose(H(gd), g2, rtol=0, atol=1e-7 * dnorm + 1e-13)
        res_o = po.residual_l1(f2, g2, Ck, w.a, w.b, w.eta)
        assert abs(info["grad_after"] - res_o) <= 1e-6 * info["grad_before"] + 1e-13
        f, g = f2, g2


def test_center_update_and_residuals(P):
    w = make("c1_rand1k", scale=0.08)
    C, Ck, phi, psi, s, f, g = oracle_state(w, 3)
    pb = P.DeviceProblem.from_workload(w)
    ph, ps = T(phi), T(psi)
    s2 = P.center_update(pb, ph, ps, s, T(f), T(g))
    assert s2 == s + 1
    # X^{k+1} = X~(f, g) (Alg. 2 line 16) and C^{k+1} = C - eta log X^{k+1} (line 3)
    logX = po.log_plan(f, g, Ck, w.eta)
    Ck1 = po.shifted_cost(C, logX, w.eta)
    Ck1_gpu = s2 * C - H(ph)[:, None] - H(ps)[None, :]
    np.testing.assert_allclose(Ck1_gpu, Ck1, rtol=0, atol=1e-13 * s2 * C.max())
    ws = P.Workspace()
    rr = P.residuals(ws, pb, T(phi), T(psi), s, T(f), T(g))
    u, v = (f + phi) / s, (g + psi - w.eta) / s
    ko = po.kkt(C, logX, w.a, w.b, u, v)
    np.testing.assert_allclose(H(rr["u"]), u, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(H(rr["v"]), v, rtol=1e-14, atol=1e-15)
    assert abs(rr["kkt"] - ko["primal"]) <= 1e-12
    assert abs(rr["obj"] - ko["pobj"]) <= 1e-13
    assert abs(rr["lp_dual_obj"] - ko["dobj"]) <= 1e-13
    assert abs(rr["dual_inf"] - ko["dual_inf"]) <= 1e-12


@pytest.mark.parametrize("name,mk", [c for c in CASES if c[0] in ("c0", "c1s", "c2s", "c3s", "c4s", "rag_dense",
                                                                 "c0r", "c3rs", "c4rs", "rag_l1_r")])
@pytest.mark.parametrize("k", [3, 30])
def test_lp_certificate_matches_oracle(P, name, mk, k):
    # reading R11: basis forest of the sparsified plan (Boruvka on the GPU, Kruskal in the
    # oracle, same strict order), tree duals by the contraction replay (GPU) vs BFS
    # (oracle), row / column c-transforms; the entropic duals are the second candidate.
    # The oracle certifies the GPU's own plan (pins_plan: the sum pass's bits), so both
    # sides see the same support and the same forest.
    w = mk()
    C, Ck, phi, psi, s, f, g = oracle_state(w, k)
    pb = P.DeviceProblem.from_workload(w)
    prm = P.default_params()
    ws = P.Workspace()
    cg = P.lp_certificate(ws, pb, prm, T(phi), T(psi), s, T(f), T(g))
    Pg = H(P.plan(pb, T(phi), T(psi), s, T(f), T(g)))
    tau = 1e-12 / (w.m * w.n)                    # the certificate's support (pins.h)
    o = lc.certify(C, w.a, w.b, Pg, tau, duals0=((f + phi) / s, (g + psi - w.eta) / s))
    assert cg["tree_edges"] == len(o["forest"])
    cmax = np.abs(C).max()
    assert abs(cg["dual_obj"] - o["dual_obj"]) <= 1e-12 * (abs(o["dual_obj"]) + cmax)
    assert abs(cg["primal"] - o["primal"]) <= 1e-12 + 1e-10 * o["primal"]
    assert abs(cg["pobj"] - o["pobj"]) <= 1e-12 * abs(o["pobj"]) + 1e-300
    assert abs(cg["gap"] - o["gap"]) <= 1e-12 * (abs(o["dual_obj"]) + cmax)
    # certified: dual feasible on the oracle's own cost matrix (rounding only)
    u, v = H(cg["u"]), H(cg["v"])
    assert (u[:, None] + v[None, :] - C).max() <= 4e-16 * cmax * 4
    assert 0.0 <= cg["dual_inf"] <= 4e-15 * cmax
    # gauge-fixed element-wise agreement (one component once the support is connected)
    if len(o["forest"]) == w.m + w.n - 1 and cg["used_tree"] == o["used_tree"]:
        c0 = u[0] - o["u"][0]
        np.testing.assert_allclose(u - c0, o["u"], rtol=0, atol=1e-12 * cmax)
        np.testing.assert_allclose(v + c0, o["v"], rtol=0, atol=1e-12 * cmax)
    # weak duality against the exact LP optimum (network simplex)
    lp = solve_exact(C, w.a, w.b)["obj"]
    assert cg["dual_obj"] <= lp + 1e-13 * lp


@pytest.mark.parametrize("name,scale,warm,K", [("c1_rand1k", 0.1, 1, 25), ("c1_rand1k", 0.1, 2, 25),
                                                ("c3_gmm10k", 0.03, 1, 12), ("c3_gmm10k_r", 0.03, 1, 12),
                                                ("c4_l1rect", 0.025, 1, 8)])
def test_solve_matches_oracle_fixed_iterations(P, name, scale, warm, K):
    # warm_start 1: carry (f, g); 2: safeguarded linear extrapolation (reading R7).
    # The point cases have m n >= 65536, so pins_solve permutes them into Morton order,
    # solves, and scatters f, g, phi, psi, u, v back: the trace and the gauge-fixed duals
    # compared here are the scattered ones (element-wise parity of the Morton path).
    w = make(name, scale=scale)
    if w.kind != COST_DENSE:
        assert w.m * w.n >= 65536
    C = po.cost_matrix(w)
    o = po.pins(C, w.a, w.b, po.Params(eta=w.eta, K=K, outer_tol=0.0, newton_tol=1e-11, warm_start=warm),
                trace=True)
    pb = P.DeviceProblem.from_workload(w)
    prm = P.default_params(K=K, outer_tol=0.0, newton_tol=1e-11, warm_start=warm)
    r = P.solve(pb, prm, trace=True)
    assert r["outer_iters"] == K
    to = np.array([t["obj"] for t in o.trace])
    np.testing.assert_allclose(np.array(r["trace"]), to, rtol=1e-9)
    assert r["kkt"] <= 1e-11 and o.kkt["primal"] <= 1e-11
    # the centre (phi, psi) = the running sums of the subproblem potentials, element-wise.
    # Potentials are unique only up to the gauge (f + c, g - c) (sum a = sum b = 1, Eq. (8)):
    # the Newton direction's component along the Hessian's null vector (e, -e) depends on
    # the linear solver, so compare gauge-fixed values (reading R5).  The
    # entropic LP dual estimates u = phi / K, v = psi / K (reading R8) follow.
    s_o = o.s_next
    assert r["s"] == s_o
    np.testing.assert_allclose(H(r["phi"]) - H(r["phi"])[0], o.phi - o.phi[0], rtol=0, atol=1e-9 * s_o)
    np.testing.assert_allclose(H(r["psi"]) + H(r["phi"])[0], o.psi + o.phi[0], rtol=0, atol=1e-9 * s_o)
    # the returned (u, v) are the certified duals (reading R11): feasible, a lower bound
    u, v = H(r["u"]), H(r["v"])
    assert (u[:, None] + v[None, :] - C).max() <= 1e-14
    assert abs(r["lp_dual_obj"] - (w.a @ u + w.b @ v)) <= 1e-14
    assert r["lp_dual_obj"] <= solve_exact(C, w.a, w.b)["obj"] + 1e-14
    assert r["gap"] == r["obj"] - r["lp_dual_obj"]


def test_workspace_reuse_and_no_leak(P):
    # one workspace, two problems at the SAME device addresses (points updated in place):
    # pins_solve_ws must rebuild every derived datum, giving exactly the fresh-workspace
    # results; repeated solves must not grow device memory (leaks, stale keys)
    wa = make("c3_gmm10k", scale=0.03)
    wb = make("c3_gmm10k", scale=0.03, seed=11)
    prm = P.default_params(K=6, outer_tol=0.0)
    pb = P.DeviceProblem.from_workload(wa)
    ws = P.Workspace()
    ra = P.solve(pb, prm, ws=ws)
    pb.x.copy_(T(wb.X)); pb.y.copy_(T(wb.Y)); pb.a.copy_(T(wb.a)); pb.b.copy_(T(wb.b))
    pb.struct.cost_scale = wb.cost_scale
    rb = P.solve(pb, prm, ws=ws)
    rb_fresh = P.solve(P.DeviceProblem.from_workload(wb), prm)
    ra_fresh = P.solve(P.DeviceProblem.from_workload(wa), prm)
    # every kernel is deterministic (pull-form tree solve, fixed-order reductions)
    assert rb["obj"] == rb_fresh["obj"] and ra["obj"] == ra_fresh["obj"]
    assert abs(rb["obj"] - ra["obj"]) > 1e-6 * abs(ra["obj"])
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        P.solve(pb, prm)
        P.solve(pb, prm, ws=ws)
    torch.cuda.synchronize()
    assert abs(torch.cuda.mem_get_info()[0] - free0) <= 4 << 20


def test_evaluate_exact_out_array(P):
    # pins.h: out_host holds >= 6 doubles ([5] = max z); call with exactly 6 through ctypes
    import ctypes
    w = make("c1_rand1k", scale=0.05)
    pb = P.DeviceProblem.from_workload(w)
    phi, psi, s = P.center_init(pb)
    f = torch.zeros(w.m, dtype=torch.float64, device="cuda")
    g = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    ws = P.Workspace()
    out = (ctypes.c_double * 6)(*([-7.0] * 6))
    lib = P.load()
    rc = lib.pins_evaluate(ws.h, pb.ref(), phi.data_ptr(), psi.data_ptr(), s, f.data_ptr(), g.data_ptr(),
                           0.0, None, None, out, P._stream())
    assert rc == 0 and out[4] == 0.0 and out[5] != -7.0 and out[1] > 0.0


BENCH = dict(K=20000, outer_rule=1, outer_tol=1e-7, newton_tol=1e-10)
BENCH_A2 = dict(K=200000, outer_rule=3, outer_tol=1e-7, newton_tol=1e-8)   # bench.py BENCH_PARAMS


@pytest.mark.parametrize("name", ["c0_pts64", "c1_rand1k", "c2_img4k", "c3_gmm10k", "c4_l1rect", "c0_pts64_r",
                                  "c3_gmm10k_r", "c4_l1rect_r"])
def test_solve_full_size_reaches_exact_lp(P, name):
    # BASELINE.json full sizes, the bench parameters (A.2 defaults + the certified outer
    # stop, reading R11): primal residual <= 1e-8, certified LP gap <= 1e-7 |obj|, measured
    # dual infeasibility at rounding level, and the objective equal to the exact LP
    # optimum of the oracle's network simplex to 1e-7 -- the SAME parameters for all configs
    gold = json.load(open(os.path.join(GOLD, f"exact_{name}.json")))
    w = make(name)
    pb = P.DeviceProblem.from_workload(w)
    r = P.solve(pb, P.default_params(**BENCH_A2))
    assert r["status"] == 0
    assert r["kkt"] <= 1e-8
    assert r["gap"] <= 1e-7 * abs(r["obj"])
    assert r["lp_dual_obj"] <= gold["obj"] * (1 + 1e-12)            # weak duality, certified
    assert 0.0 <= r["dual_inf"] <= 1e-14
    assert abs(r["obj"] - gold["obj"]) <= 1e-7 * abs(gold["obj"])
    if w.m * w.n <= 1 << 20:                                         # duals feasible on the oracle's C
        C = po.cost_matrix(w)
        u, v = H(r["u"]), H(r["v"])
        assert (u[:, None] + v[None, :] - C).max() <= 1e-14


@pytest.mark.parametrize("name,scale", [("c1_rand1k", 0.125), ("c2_img4k", 0.06), ("c4_l1rect", 0.01),
                                        ("c3_gmm10k", 0.01)])
def test_solve_small_scale_reaches_exact_lp(P, name, scale):
    w = make(name, scale=scale)
    ex = solve_exact(po.cost_matrix(w), w.a, w.b)
    pb = P.DeviceProblem.from_workload(w)
    r = P.solve(pb, P.default_params(**BENCH), trace=True)
    assert r["kkt"] <= 1e-8
    assert abs(r["obj"] - ex["obj"]) <= 1e-7 * abs(ex["obj"])
    tr = np.array(r["trace"])
    # Thm 4.1: <C, X^{k+1}> <= <C, X^k> for exact subproblem solves.  The
    # solves stop at ||grad P^k||_1 <= newton_tol, i.e. each plan's marginals are off by at
    # most newton_tol in l1, which moves <C, X> by at most newton_tol max C: slack 2 newton_tol max C
    cmax = po.cost_matrix(w).max()
    assert np.all(np.diff(tr) <= 2 * BENCH["newton_tol"] * cmax)


def test_edge_cases(P):
    # single cell: the only feasible plan is [[1]]
    w = Workload("one", 1, 1, COST_DENSE, np.ones(1), np.ones(1), 0.01, C=np.array([[0.3]]))
    r = P.solve(P.DeviceProblem.from_workload(w), P.default_params(K=5))
    assert abs(r["obj"] - 0.3) <= 1e-12 and r["kkt"] <= 1e-12
    # single row / column: plan is forced (a b^T)
    rng = np.random.default_rng(0)
    b = rng.random(300) + 0.1; b /= b.sum()
    w = Workload("row", 1, 300, COST_DENSE, np.ones(1), b, 0.01, C=rng.random((1, 300)))
    r = P.solve(P.DeviceProblem.from_workload(w), P.default_params(K=5))
    assert abs(r["obj"] - (w.C[0] @ b)) <= 1e-10 and r["kkt"] <= 1e-8
    # invalid arguments fail loudly (no fallback)
    bad = P.DeviceProblem(0, 4, 0, T(np.ones(1)), T(np.ones(4) / 4), 0.1, C=T(np.zeros((1, 4))))
    with pytest.raises(RuntimeError):
        P.solve(bad)
    bad = P.DeviceProblem(2, 2, 0, T(np.ones(2) / 2), T(np.ones(2) / 2), -1.0, C=T(np.zeros((2, 2))))
    with pytest.raises(RuntimeError):
        P.solve(bad)


@pytest.mark.parametrize("name,mk", [("c3s", lambda: make("c3_gmm10k", scale=0.05)),
                                     ("c2s", lambda: make("c2_img4k", scale=0.1)),
                                     ("rag_sq", lambda: ragged(301, 517, 9, "sq", 10))])
def test_tensor_core_cross_term_bit_identical(P, name, mk, monkeypatch):
    # x.y on tcgen05 (fp16 operands, fp32 accumulate) is exact for integer points with
    # |x| <= 2048 and partial sums < 2^24 (pins_tc.cuh), so every pass must reproduce the
    # SIMT fp32 path bit for bit: sums, objective, CSR pattern and values, sweeps
    w = mk()
    C, Ck, phi, psi, s, f, g = oracle_state(w, 1)
    tau = 1e-4 / (w.m * w.n)
    out = []
    for no_tc in (False, True):
        if no_tc:
            monkeypatch.setenv("PINS_NO_TC", "1")
        pb = P.DeviceProblem.from_workload(w)
        ws = P.Workspace()
        ev = P.evaluate(ws, pb, T(phi), T(psi), s, T(f), T(g), tau=tau)
        csr = [H(t) for t in P.get_csr(ws)]
        fd, gd = T(f), T(g)
        for _ in range(2):
            P.sinkhorn_sweep(ws, pb, T(phi), T(psi), s, fd, gd)
        out.append((H(ev["r"]), H(ev["c"]), ev["cost"], ev["grad_l1"], csr, H(fd), H(gd)))
    a, b = out
    for x, y in zip(a[:2], b[:2]):
        assert np.array_equal(x, y)
    assert a[2] == b[2] and a[3] == b[3]
    for x, y in zip(a[4], b[4]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[5], b[5]) and np.array_equal(a[6], b[6])


@pytest.mark.parametrize("name,mk", [("c1t", lambda: make("c1_rand1k", scale=0.3125)),
                                     ("rag_dense_t", lambda: ragged(301, 1030, 19)),
                                     ("tall", lambda: ragged(1030, 66, 20))])
def test_tma_staged_dense_passes_bit_identical(P, name, mk, monkeypatch):
    # dense C tiles staged by TMA (cp.async.bulk.tensor, 128-byte swizzle for the row
    # orientation) feed the same arithmetic in the same order as the thread-staged path:
    # every pass must agree bit for bit (PINS_NO_TMA=1 selects the thread-staged path)
    w = mk()
    assert w.n % 2 == 0
    C, Ck, phi, psi, s, f, g = oracle_state(w, 1)
    tau = 1e-4 / (w.m * w.n)
    out = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("PINS_NO_TMA", "1")
        pb = P.DeviceProblem.from_workload(w)
        ws = P.Workspace()
        ev = P.evaluate(ws, pb, T(phi), T(psi), s, T(f), T(g), tau=tau)
        csr = [H(t_) for t_ in P.get_csr(ws)]
        fd, gd = T(f), T(g)
        P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, 0.0, 7)
        out.append((H(ev["r"]), H(ev["c"]), ev["cost"], ev["grad_l1"], csr, H(fd), H(gd)))
    a, b = out
    for x, y in zip(a[:2], b[:2]):
        assert np.array_equal(x, y)
    assert a[2] == b[2] and a[3] == b[3]
    for x, y in zip(a[4], b[4]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[5], b[5]) and np.array_equal(a[6], b[6])


@pytest.mark.parametrize("name,mk", [("c3s", lambda: make("c3_gmm10k", scale=0.05)),
                                     ("c4s", lambda: make("c4_l1rect", scale=0.05)),
                                     ("rag_sq", lambda: ragged(301, 517, 9, "sq", 10)),
                                     ("rag_l1", lambda: ragged(517, 301, 3, "l1", 11))])
def test_tile_skip_bit_identical(P, name, mk, monkeypatch):
    # whole-chunk skipping (R10, tile form) drops a chunk only when the drift certificate
    # proves that the per-entry fp32 test rejects every entry of it, so every pass -- and
    # hence every whole solve -- must be bit-identical with and without it
    w = mk()
    C, Ck, phi, psi, s, f, g = oracle_state(w, 1)
    tau = 1e-4 / (w.m * w.n)
    out = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("PINS_NO_TILESKIP", "1")
        pb = P.DeviceProblem.from_workload(w)
        ws = P.Workspace()
        ev = P.evaluate(ws, pb, T(phi), T(psi), s, T(f), T(g), tau=tau)
        csr = [H(t) for t in P.get_csr(ws)]
        fd, gd = T(f), T(g)
        # 40 sweeps in ONE device-side Sinkhorn phase: the first passes record the drift
        # certificates, the later ones skip chunks (tol 0: never stops early)
        P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, 0.0, 40)
        r = P.solve(pb, P.default_params(K=6, outer_tol=0.0))
        out.append((H(ev["r"]), H(ev["c"]), ev["cost"], ev["grad_l1"], csr, H(fd), H(gd),
                    r["obj"], H(r["u"]), H(r["v"])))
    a, b = out
    for x, y in zip(a[:2], b[:2]):
        assert np.array_equal(x, y)
    assert a[2] == b[2] and a[3] == b[3]
    for x, y in zip(a[4], b[4]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[5], b[5]) and np.array_equal(a[6], b[6])
    assert a[7] == b[7] and np.array_equal(a[8], b[8]) and np.array_equal(a[9], b[9])


@pytest.mark.parametrize("name,scale", [("c3_gmm10k", 0.04), ("c4_l1rect", 0.03), ("c1_rand1k", 0.2),
                                        ("c3_gmm10k_r", 0.03)])
def test_solve_is_bit_reproducible(P, name, scale):
    # repeated pins_solve calls give identical bits: no atomics decide any floating-point
    # sum (the tree factor / solve gather in pull form; all reductions have a fixed order)
    w = make(name, scale=scale)
    pb = P.DeviceProblem.from_workload(w)
    prm = P.default_params(K=30, outer_tol=0.0)
    r1 = P.solve(pb, prm)
    r2 = P.solve(pb, prm)
    assert r1["obj"] == r2["obj"] and r1["cg_iters"] == r2["cg_iters"]
    for k in ("f", "g", "phi", "psi", "u", "v"):
        assert np.array_equal(H(r1[k]), H(r2[k])), k


@pytest.mark.parametrize("name,mk", [("c3s", lambda: make("c3_gmm10k", scale=0.05)),
                                     ("c4s", lambda: make("c4_l1rect", scale=0.04)),
                                     ("c1t", lambda: make("c1_rand1k", scale=0.125)),
                                     ("rag_dense", lambda: ragged(37, 1029, 5)),
                                     ("c3rs", lambda: make("c3_gmm10k_r", scale=0.03)),
                                     ("rag_l1_r", lambda: ragged(133, 47, 17, "l1", 3, real=True)),
                                     ("rag_sq", lambda: ragged(301, 517, 9, "sq", 10))])
def test_sparse_sweeps_bit_identical(P, name, mk, monkeypatch):
    # The Sinkhorn phase walks certified candidate lists (lse_sparse_kernel) instead of the
    # dense m x n block; the certificate proves that no entry outside a list can pass the
    # dense pass's fp32 test, and the lists are walked with the dense pass's chunk
    # thresholds and survivor pairing -- so f, g and the sweep count must be bit-identical
    # to the dense sweeps.  The third setting forces list overflow (capacity 2: regrowth)
    # and failing certificates (margin 0.01: dense fallback rows and re-records).
    w = mk()
    out = []
    for k in (0, 1):
        if k == 0:
            phi, psi, s = w.eta * np.log(w.a), w.eta * np.log(w.b), 1.0
            f, g = np.zeros(w.m), np.zeros(w.n)
        else:
            C, Ck, phi, psi, s, f, g = oracle_state(w, 1)
            f = f + np.random.default_rng(3).normal(0, 3 * w.eta, w.m)
        res = []
        for env in ({"PINS_KSWEEP": "0"}, {"PINS_SPARSE_SWEEP": "1"},
                    {"PINS_SPARSE_SWEEP": "1", "PINS_LIST_CAP": "2", "PINS_LIST_MARGIN": "0.01"}):
            for key in ("PINS_SPARSE_SWEEP", "PINS_LIST_CAP", "PINS_LIST_MARGIN", "PINS_KSWEEP"):
                monkeypatch.delenv(key, raising=False)
            for key, v in env.items():
                monkeypatch.setenv(key, v)
            pb = P.DeviceProblem.from_workload(w)
            ws = P.Workspace()
            fd, gd = T(f), T(g)
            t, r = P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, 0.0, 70)
            t2, r2 = P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, 1e-3, 400)   # stops on the tolerance
            res.append((t, r, t2, r2, H(fd), H(gd)))
        d = res[0]
        for o in res[1:]:
            assert o[0] == d[0] and o[2] == d[2], (name, k, o[:4], d[:4])
            assert o[1] == d[1] and o[3] == d[3]
            assert np.array_equal(o[4], d[4]) and np.array_equal(o[5], d[5])
        out.append(d[2])
    # and whole solves
    objs = []
    for env in ({"PINS_KSWEEP": "0"}, {"PINS_SPARSE_SWEEP": "1"}):
        for key in ("PINS_SPARSE_SWEEP", "PINS_LIST_CAP", "PINS_LIST_MARGIN", "PINS_KSWEEP"):
            monkeypatch.delenv(key, raising=False)
        for key, v in env.items():
            monkeypatch.setenv(key, v)
        pb = P.DeviceProblem.from_workload(w)
        r = P.solve(pb, P.default_params(K=5, outer_tol=0.0))
        objs.append((r["obj"], r["sweeps"], H(r["u"]), H(r["v"])))
    assert objs[0][0] == objs[1][0] and objs[0][1] == objs[1][1]
    assert np.array_equal(objs[0][2], objs[1][2]) and np.array_equal(objs[0][3], objs[1][3])


KS_KEYS = ("PINS_SPARSE_SWEEP", "PINS_LIST_CAP", "PINS_LIST_MARGIN", "PINS_KSWEEP", "PINS_KSWEEP_START",
           "PINS_KSWEEP_NOCOOL", "PINS_LIST_BUDGET")


@pytest.mark.parametrize("name,mk", [("c3s", lambda: make("c3_gmm10k", scale=0.05)),
                                     ("c4s", lambda: make("c4_l1rect", scale=0.04)),
                                     ("c1t", lambda: make("c1_rand1k", scale=0.125)),
                                     ("rag_dense", lambda: ragged(37, 1029, 5)),
                                     ("c3rs", lambda: make("c3_gmm10k_r", scale=0.03)),
                                     ("rag_l1_r", lambda: ragged(133, 47, 17, "l1", 3, real=True)),
                                     ("rag_sq", lambda: ragged(301, 517, 9, "sq", 10))])
def test_kernel_matrix_sweeps(P, name, mk, monkeypatch):
    # Absorbed kernel-matrix sweeps (lse_ksweep_kernel, the default of long Sinkhorn phases):
    # exp(x_ij - r) = K_ij u_j with K fixed since the record pass -- the same sums as the
    # log-domain pass (Alg. 2 l.5-6) with a different rounding, so f, g agree with the dense
    # sweeps and with the oracle to the sweep tolerance and the phase stops at the same
    # sweep.  Settings: from the first sweep on; from sweep 7 (the default); without the
    # churn control (the phase stays in kernel-matrix mode however many units fall back);
    # and forced list overflow (capacity 2: regrowth) with failing certificates (margin
    # 0.01: dense fallback units and re-records).
    w = mk()
    for k in (0, 1):
        if k == 0:
            C = po.cost_matrix(w)
            Ck = po.shifted_cost(C, np.log(w.a)[:, None] + np.log(w.b)[None, :], w.eta)
            phi, psi, s = w.eta * np.log(w.a), w.eta * np.log(w.b), 1.0
            f, g = np.zeros(w.m), np.zeros(w.n)
        else:
            C, Ck, phi, psi, s, f, g = oracle_state(w, 1)
            f = f + np.random.default_rng(3).normal(0, 3 * w.eta, w.m)
        res = []
        for env in ({"PINS_KSWEEP": "0"}, {"PINS_KSWEEP_START": "0"}, {},
                    {"PINS_KSWEEP_START": "0", "PINS_KSWEEP_NOCOOL": "1"},
                    {"PINS_KSWEEP_START": "0", "PINS_LIST_BUDGET": "4096"},    # lists declined: dense sweeps
                    {"PINS_KSWEEP_START": "0", "PINS_LIST_CAP": "2", "PINS_LIST_MARGIN": "0.01",
                     "PINS_KSWEEP_NOCOOL": "1"}):
            for key in KS_KEYS:
                monkeypatch.delenv(key, raising=False)
            for key, v in env.items():
                monkeypatch.setenv(key, v)
            pb = P.DeviceProblem.from_workload(w)
            ws = P.Workspace()
            fd, gd = T(f), T(g)
            t, r = P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, 0.0, 40)
            f40, g40 = H(fd).copy(), H(gd).copy()
            t2, r2 = P.sinkhorn(ws, pb, T(phi), T(psi), s, fd, gd, 1e-3, 400)   # stops on the tolerance
            res.append((t, r, t2, r2, f40, g40, H(fd), H(gd)))
        # the oracle's 40 sweeps
        fo, go = f.copy(), g.copy()
        for _ in range(40):
            fo, go = po.sinkhorn_sweep(fo, go, Ck, w.a, w.b, w.eta)
        scale = max(1.0, s * C.max() / w.eta)
        tol_f = 1e-13 * scale * w.eta * 41
        d = res[0]
        assert np.array_equal(res[4][6], d[6]) and np.array_equal(res[4][7], d[7])   # declined = dense, bit for bit
        for o in res:
            assert o[0] == d[0] and o[2] == d[2], (name, k, o[:4], d[:4])
            assert abs(o[1] - d[1]) <= 1e-9 * abs(d[1]) + 1e-15
            np.testing.assert_allclose(o[4], fo, rtol=0, atol=tol_f * (1 + np.abs(fo).max() / w.eta))
            np.testing.assert_allclose(o[5], go, rtol=0, atol=tol_f * (1 + np.abs(go).max() / w.eta))
            tol2 = 1e-13 * scale * w.eta * (41 + d[2])
            np.testing.assert_allclose(o[6], d[6], rtol=0, atol=tol2 * (1 + np.abs(d[6]).max() / w.eta))
            np.testing.assert_allclose(o[7], d[7], rtol=0, atol=tol2 * (1 + np.abs(d[7]).max() / w.eta))
    # and whole solves
    objs = []
    for env in ({"PINS_KSWEEP": "0"}, {"PINS_KSWEEP_START": "0"}):
        for key in KS_KEYS:
            monkeypatch.delenv(key, raising=False)
        for key, v in env.items():
            monkeypatch.setenv(key, v)
        pb = P.DeviceProblem.from_workload(w)
        r = P.solve(pb, P.default_params(K=5, outer_tol=0.0))
        ph, ps = H(r["phi"]), H(r["psi"])
        objs.append((r["obj"], r["sweeps"], ph - ph[0], ps + ph[0]))
    assert objs[0][1] == objs[1][1]
    # each subproblem is solved to newton_tol, not to rounding: the two runs agree like the
    # GPU and the oracle traces do (test_solve_trace_matches_oracle: rtol 1e-9)
    assert abs(objs[0][0] - objs[1][0]) <= 1e-9 * abs(objs[0][0])
    np.testing.assert_allclose(objs[1][2], objs[0][2], rtol=0, atol=1e-9 * 6)
    np.testing.assert_allclose(objs[1][3], objs[0][3], rtol=0, atol=1e-9 * 6)


@pytest.mark.parametrize("name,scale", [("c4_l1rect", 0.04), ("c3_gmm10k", 0.05), ("c1_rand1k", 0.2)])
def test_no_uninitialised_reads(P, name, scale, monkeypatch):
    # every device buffer the library allocates is filled with a garbage byte first
    # (PINS_POISON, dev switch): a solve that read memory before writing it would change
    # (or fault); results must be bit-identical to the unpoisoned solve.  (Regression: the
    # tree workspace was once reallocated at the same address and its stale factor reused.)
    w = make(name, scale=scale)
    out = []
    # kernel-matrix sweeps from the first sweep on, so their buffers (lists, ELL tiles, unit
    # records, packing offsets) are covered as well
    monkeypatch.setenv("PINS_KSWEEP_START", "0")
    for z in (None, "165", "0"):
        monkeypatch.delenv("PINS_POISON", raising=False)
        if z is not None:
            monkeypatch.setenv("PINS_POISON", z)
        pb = P.DeviceProblem.from_workload(w)
        r = P.solve(pb, P.default_params(K=4, outer_tol=0.0))
        out.append((r["obj"], r["cg_iters"], r["sweeps"], H(r["u"]), H(r["v"]), H(r["f"])))
    for o in out[1:]:
        assert o[0] == out[0][0] and o[1] == out[0][1] and o[2] == out[0][2]
        for x, y in zip(o[3:], out[0][3:]):
            assert np.array_equal(x, y)
