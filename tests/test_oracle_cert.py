"""Pins of the LP-certificate oracle (oracle/lp_certificate.py, reading R11):
spanning forest vs brute force, tree duals vs the network simplex duals,
c-transforms on hand-computed values, weak duality, zero gap at the optimum."""
import itertools

import numpy as np
import pytest

from oracle import lp_certificate as lc
from oracle.exact_lp import brute_force_assignment, solve_exact


def norm(v):
    return v / v.sum()


def csr(mask, X):
    rows, cols = np.nonzero(mask)
    rowptr = np.zeros(mask.shape[0] + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    return np.cumsum(rowptr), cols, X[rows, cols]


def is_forest(edges, m, n):
    parent = list(range(m + n))

    def find(x):
        while parent[x] != x:
            x = parent[x]
        return x
    for i, j in edges:
        a, b = find(i), find(m + j)
        if a == b:
            return False
        parent[a] = b
    return True


@pytest.mark.parametrize("seed", range(6))
def test_max_spanning_forest_is_the_brute_force_maximum(seed):
    rng = np.random.default_rng(seed)
    m, n = 3, 3
    mask = rng.random((m, n)) < 0.7
    X = rng.random((m, n))
    rp, ci, va = csr(mask, X)
    forest = lc.max_spanning_forest(rp, ci, va, m, n)
    edges = [(int(i), int(j)) for i, j in zip(*np.nonzero(mask))]
    # components of the support graph fix the size of every spanning forest
    best = max((sum(X[i, j] for i, j in sub), sub) for k in range(len(edges) + 1)
               for sub in itertools.combinations(edges, k) if is_forest(sub, m, n))
    got = [(i, j) for i, j, _ in forest]
    assert is_forest(got, m, n)
    assert len(got) == len(best[1])
    assert sum(X[i, j] for i, j in got) == pytest.approx(best[0], rel=1e-15)
    assert sorted(got) == sorted(best[1])


def test_tree_duals_satisfy_the_basis_equations_and_gauge():
    rng = np.random.default_rng(3)
    m, n = 6, 5
    C = rng.random((m, n))
    # a random spanning tree of K_{m,n}: attach each new node to an earlier one of the other side
    edges, order = [], rng.permutation(m + n)
    placed = [order[0]]
    for x in order[1:]:
        cand = [y for y in placed if (y < m) != (x < m)]
        if not cand:
            cand = [y for y in placed if (y < m) != (x < m)] or placed
        y = cand[rng.integers(len(cand))] if cand and (cand[0] < m) != (x < m) else None
        if y is None:
            continue
        i, j = (x, y - m) if x < m else (y, x - m)
        edges.append((int(i), int(j), 0))
        placed.append(x)
    u, v = lc.tree_duals(C, edges, m, n)
    for i, j, _ in edges:
        assert u[i] + v[j] == pytest.approx(C[i, j], abs=1e-14)
    # gauge: the smallest node index of the component has z = 0
    comp_nodes = sorted({i for i, _, _ in edges} | {m + j for _, j, _ in edges})
    r = comp_nodes[0]
    assert (u[r] if r < m else -v[r - m]) == 0.0


def test_ctransform_hand_values():
    C = np.array([[1.0, 2.0], [3.0, 0.0]])
    u = lc.ctransform_rows(C, np.zeros(2))
    assert list(u) == [1.0, 0.0]
    v = lc.ctransform_cols(C, u)
    assert list(v) == [0.0, 0.0]
    a = b = np.array([0.5, 0.5])
    # LP optimum: the diagonal plan, cost 0.5 (brute force over the two permutations)
    assert a @ u + b @ v == 0.5 == brute_force_assignment(C)[1]
    # v = (1, -1): u = min_j (C_ij - v_j) = (min(0, 3), min(2, 1)) = (0, 1)
    assert list(lc.ctransform_rows(C, np.array([1.0, -1.0]))) == [0.0, 1.0]


@pytest.mark.parametrize("seed", range(5))
def test_weak_duality_for_any_ctransformed_duals(seed):
    rng = np.random.default_rng(100 + seed)
    m, n = 8, 11
    C = rng.random((m, n))
    a, b = norm(rng.random(m) + 0.1), norm(rng.random(n) + 0.1)
    lp = solve_exact(C, a, b)["obj"]
    for _ in range(5):
        v = rng.normal(0, 1, n)
        u = lc.ctransform_rows(C, v)
        v2 = lc.ctransform_cols(C, u)
        assert (u[:, None] + v2[None, :] <= C + 1e-15).all()
        assert a @ u + b @ v2 <= lp + 1e-14
        assert a @ u + b @ v2 >= a @ u + b @ v - 1e-14      # the column transform only raises v


@pytest.mark.parametrize("seed", range(5))
def test_certificate_of_the_exact_optimum_has_zero_gap(seed):
    # non-degenerate random instance: the optimal vertex's support is a spanning tree
    # (m + n - 1 positive flows); its tree duals are optimal, the c-transforms change
    # nothing, and the certified lower bound equals LP* (network simplex)
    rng = np.random.default_rng(200 + seed)
    m, n = 9, 12
    C = rng.random((m, n))
    a, b = norm(rng.random(m) + 0.1), norm(rng.random(n) + 0.1)
    ex = solve_exact(C, a, b)
    X = ex["X"]
    assert int((X > 0).sum()) == m + n - 1
    cert = lc.certify(C, a, b, X, tau=1e-300)
    assert len(cert["forest"]) == m + n - 1
    assert cert["rows_changed"] == 0 and cert["cols_changed"] == 0
    assert cert["dual_obj"] == pytest.approx(ex["obj"], rel=1e-13)
    assert abs(cert["gap"]) <= 1e-14 and cert["primal"] <= 1e-14 and cert["dual_inf"] <= 1e-15
    # the tree duals are the network simplex duals up to the gauge (c, -c)
    c = cert["u_tree"][0] - ex["u"][0]
    np.testing.assert_allclose(cert["u_tree"] - c, ex["u"], atol=1e-13)
    np.testing.assert_allclose(cert["v_tree"] + c, ex["v"], atol=1e-13)


def test_certificate_of_a_perturbed_plan_is_a_valid_bound():
    # an entropically smoothed optimum (a near-optimal interior plan): the forest of its
    # heaviest entries is still the optimal basis, so the bound is still exact; a plan far
    # from optimal still gives a valid (lower) bound
    rng = np.random.default_rng(7)
    m, n = 10, 10
    C = rng.random((m, n))
    a, b = norm(rng.random(m) + 0.1), norm(rng.random(n) + 0.1)
    ex = solve_exact(C, a, b)
    X = ex["X"] + 1e-9 * rng.random((m, n))
    cert = lc.certify(C, a, b, X, tau=0.0)
    assert cert["dual_obj"] == pytest.approx(ex["obj"], rel=1e-12)
    Xbad = np.outer(a, b)                    # the product plan X^0
    bad = lc.certify(C, a, b, Xbad, tau=0.0)
    assert bad["dual_obj"] <= ex["obj"] + 1e-14 and bad["gap"] > 1e-3
    assert bad["dual_inf"] <= 1e-15


def test_certificate_on_a_degenerate_assignment_is_a_valid_bound():
    # uniform marginals: the optimum is a permutation (Birkhoff), a
    # degenerate vertex; the certificate's bound never exceeds the brute-force optimum
    rng = np.random.default_rng(9)
    n = 6
    C = rng.random((n, n))
    a = b = np.full(n, 1.0 / n)
    perm, opt = brute_force_assignment(C)
    X = np.zeros((n, n))
    X[np.arange(n), perm] = 1.0 / n
    X += 1e-12 * rng.random((n, n))
    cert = lc.certify(C, a, b, X, tau=0.0)
    assert cert["dual_obj"] <= opt + 1e-14
    assert cert["dual_inf"] <= 1e-15


def test_component_gauges_make_a_disconnected_support_exact():
    # two balanced blocks with expensive cross costs: the optimal plan has no flow
    # between them, so the support (and the forest) has two components whose tree
    # duals carry arbitrary relative gauges; the shortest-path shifts (step 3) make
    # them feasible and the bound exact
    rng = np.random.default_rng(31)
    C = 1.0 + rng.random((6, 6))
    C[:3, :3] = rng.random((3, 3))
    C[3:, 3:] = rng.random((3, 3))
    a = norm(np.array([1.0, 2.0, 3.0, 1.5, 2.5, 2.0]))
    b = norm(np.array([2.0, 1.0, 3.0, 2.0, 2.0, 2.0]))
    assert abs(a[:3].sum() - b[:3].sum()) < 1e-15        # balanced blocks
    ex = solve_exact(C, a, b)
    X = ex["X"]
    assert np.all(X[:3, 3:] == 0) and np.all(X[3:, :3] == 0)
    cert = lc.certify(C, a, b, X, tau=1e-300)
    assert cert["components"] >= 2
    assert cert["dual_obj"] == pytest.approx(ex["obj"], rel=1e-13)
    assert cert["dual_inf"] <= 1e-15
    # the shifts alone restore feasibility of the tree duals (before any c-transform)
    forest = lc.max_spanning_forest(*csr(X >= 1e-300, X), 6, 6)
    u0, v0 = lc.tree_duals(C, forest, 6, 6)
    us, vs = lc.component_shift(C, u0, v0, lc.components(forest, 6, 6))
    assert (us[:, None] + vs[None, :] - C).max() <= 1e-15


def test_repair_forces_violated_support_edges_into_the_forest():
    # a plan whose heaviest spanning forest is not the optimal basis: the tree duals
    # violate a support edge; forcing it in (step 5) recovers the optimal basis
    rng = np.random.default_rng(5)
    m, n = 7, 8
    C = rng.random((m, n))
    a, b = norm(rng.random(m) + 0.1), norm(rng.random(n) + 0.1)
    ex = solve_exact(C, a, b)
    X = ex["X"].copy()
    basis = np.argwhere(X > 0)
    i, j = basis[np.argmin(X[X > 0])]                   # shrink the smallest basic flow ...
    X[i, j] = 1e-12
    nb = np.argwhere(ex["X"] == 0)
    k = nb[0]
    X[k[0], k[1]] = 1e-6                                # ... below a non-basic entry
    one = lc.certify(C, a, b, X, tau=1e-300, repairs=1)
    rep = lc.certify(C, a, b, X, tau=1e-300, repairs=3)
    assert rep["dual_obj"] >= one["dual_obj"] - 1e-15
    assert rep["dual_obj"] <= ex["obj"] + 1e-14
    assert rep["dual_inf"] <= 1e-15
