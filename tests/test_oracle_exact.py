"""Pins of the exact LP oracle (network simplex) -- PAPER.md Eq. (1), Thm 4.3 proof."""
import itertools

import numpy as np
import pytest

from oracle.exact_lp import brute_force_assignment, solve_exact


def test_brute_force_trivial():
    assert brute_force_assignment(np.array([[0.3]])) == ((0,), 0.3)
    p, v = brute_force_assignment(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert p == (0, 1) and v == 0.0


def test_network_simplex_equals_brute_force_on_uniform_square():
    # Thm 4.3 proof: Birkhoff polytope, vertices = permutations
    rng = np.random.default_rng(0)
    for _ in range(25):
        n = int(rng.integers(1, 8))
        C = rng.random((n, n))
        a = np.full(n, 1.0 / n)
        r = solve_exact(C, a, a.copy())
        _, bf = brute_force_assignment(C)
        assert abs(r["obj"] - bf) <= 1e-12
        # Birkhoff invariant: the optimal vertex is a scaled permutation matrix
        X = r["X"] * n
        assert np.allclose(np.sort(X, axis=1)[:, -1], 1.0, atol=1e-12)
        assert (np.abs(X) > 1e-12).sum() == n


def test_network_simplex_vertex_and_certificate_on_rectangles():
    rng = np.random.default_rng(1)
    for _ in range(25):
        m, n = int(rng.integers(1, 25)), int(rng.integers(1, 25))
        C = rng.random((m, n))
        a = rng.random(m) + 0.05; a /= a.sum()
        b = rng.random(n) + 0.05; b /= b.sum()
        r = solve_exact(C, a, b)
        X = r["X"]
        assert (X > 0).sum() <= m + n - 1                  # vertex (basic) solution
        assert X.min() >= 0.0
        assert np.abs(X.sum(1) - a).sum() + np.abs(X.sum(0) - b).sum() <= 1e-13
        assert r["min_rc"] >= -1e-12                        # dual feasible
        assert abs(r["obj"] - (a @ r["u"] + b @ r["v"])) <= 1e-13   # zero gap


def test_network_simplex_below_random_feasible_plans():
    rng = np.random.default_rng(2)
    m, n = 7, 9
    C = rng.random((m, n)); a = np.full(m, 1 / m); b = np.full(n, 1 / n)
    opt = solve_exact(C, a, b)["obj"]
    for _ in range(100):
        K = rng.random((m, n)) + 1e-3
        for _ in range(300):                                   # rescale to the polytope
            K *= (a / K.sum(1))[:, None]
            K *= (b / K.sum(0))[None, :]
        assert (C * K).sum() >= opt - 1e-12


def test_row_shift_invariance():
    # adding t to row i changes the optimum by t * a_i (every feasible plan has row mass a_i)
    rng = np.random.default_rng(3)
    C = rng.random((5, 6)); a = rng.random(5) + .1; a /= a.sum(); b = np.full(6, 1 / 6)
    o1 = solve_exact(C, a, b)["obj"]
    C2 = C.copy(); C2[2] += 0.3
    o2 = solve_exact(C2, a, b)["obj"]
    assert abs(o2 - o1 - 0.3 * a[2]) <= 1e-13


@pytest.mark.parametrize("n", [3, 5, 8, 10])
def test_theorem_4_3_reference_hessian_sparsity(n):
    # Thm 4.3: tau(H^k) <= (3n-1)/(2n^2) for m = n, with
    # H^k's off block = an optimal vertex plan and exact diagonals.
    rng = np.random.default_rng(100 + n)
    for _ in range(5):
        C = rng.random((n, n)); a = np.full(n, 1.0 / n)
        X = solve_exact(C, a, a.copy())["X"]
        nnz = 2 * int((X > 0).sum()) + 2 * n
        assert nnz / (2 * n) ** 2 <= (3 * n - 1) / (2 * n * n) + 1e-15
