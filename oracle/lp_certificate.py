"""LP optimality certificate for a PINS plan -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It shares no code with the CUDA path.

What it computes (reading R11): certified LP duals and the LP
KKT residuals of a plan X~ produced by PINS, for the transport LP Eq. (1)


    min <C,X>  s.t.  X e = a,  X^T e = b,  X >= 0,
    dual:  max <a,u> + <b,v>  s.t.  u_i + v_j <= C_ij.

Any dual-feasible (u, v) gives the lower bound <a,u> + <b,v> <= LP* (weak
duality), so  gap = <C,X> - <a,u> - <b,v>  bounds the objective error of X from
above (up to X's own marginal residual).  The duals are built in three steps,
each a plain definition:

1. basis: a maximum-weight spanning forest T of the sparsified support graph
   of X~ (rows and columns are nodes, kept entries X~_ij >= tau are edges;
   the GPU uses tau = 1e-12/(m n), far below the Newton threshold, so basic
   edges with tiny flows stay in the graph).
   PAPER.md Thm 4.3 proof (lines 362): the LP optimum is a vertex of the
   transport polytope; a vertex's support is a forest of the bipartite graph
   (a spanning tree when non-degenerate), and PINS' plans concentrate on it
   as k grows.  Ties are broken by the strict order (fl32(X~_ij), CSR
   position), so the forest is unique (Kruskal here; the GPU builds the same
   forest by Boruvka).
2. tree duals: the unique (per component, gauge z_root = 0) solution of
   u_i + v_j = C_ij on the edges of T -- the complementary-slackness
   equations of the basis (network-simplex duals of that basis).
3. component gauges: a disconnected support leaves one free gauge (u + d_A,
   v - d_A) per component A; the shifts must satisfy d_A - d_B <= R_AB =
   min_{i in A, j in B} (C_ij - u_i - v_j), a system of difference
   constraints solved by shortest paths (Bellman-Ford from a virtual source).
   With balanced components (no optimal flow between them) every feasible
   choice gives the same bound.
4. c-transforms: u'_i = min_j (C_ij - v_j), then v'_j = min_i (C_ij - u'_i).
   (u', v') is dual feasible by construction; if T is an optimal basis, its
   duals already are, and the c-transforms change nothing (each row / column
   has a tight tree edge), so <a,u'> + <b,v'> = LP*.
5. repair (up to 3 forests): support edges that the tree duals violate
   (C_ij - u_i - v_j < -1e-13 (1 + |<C,X>|)) are forced into the next forest
   (weight 4 > any plan entry, so the forest drops the lightest edge of the
   cycle each closes); every forest's bound is valid, the best is kept.
Finally the entropic duals, c-transformed, are a second candidate.
"""
from __future__ import annotations

from collections import deque
from typing import Dict, List, Tuple

import numpy as np


def max_spanning_forest(rowptr: np.ndarray, colidx: np.ndarray, val: np.ndarray, m: int, n: int) -> List[Tuple[int, int, int]]:
    """Kruskal on the bipartite support graph (row i = node i, column j = node m + j):
    edges in decreasing (float32(value), CSR position) order, union-find.  Returns the
    forest edges as (row, column, CSR position), in insertion order."""
    nnz = len(colidx)
    rows = np.repeat(np.arange(m), np.diff(rowptr))
    w32 = val.astype(np.float32)
    order = np.lexsort((-np.arange(nnz), -w32.astype(np.float64)))   # value desc, then position desc
    parent = list(range(m + n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    out = []
    for e in order:
        i, j = int(rows[e]), int(colidx[e])
        ri, rj = find(i), find(m + j)
        if ri != rj:
            parent[ri] = rj
            out.append((i, j, int(e)))
    return out


def tree_duals(C: np.ndarray, edges, m: int, n: int) -> Tuple[np.ndarray, np.ndarray]:
    """Solve u_i + v_j = C_ij on the forest edges (complementary slackness of the basis).

    Per component: the node of smallest index (rows 0..m-1, then columns m..m+n-1) is
    the root with z = 0, where z = (u, -v); breadth-first, an edge (i, j) gives
    z_col = z_row - C_ij and z_row = z_col + C_ij.  Nodes on no edge get 0."""
    adj = [[] for _ in range(m + n)]
    for i, j, _ in edges:
        adj[i].append(m + j)
        adj[m + j].append(i)
    z = np.zeros(m + n)
    seen = np.zeros(m + n, dtype=bool)
    for r in range(m + n):
        if seen[r]:
            continue
        seen[r] = True
        q = deque([r])
        while q:
            x = q.popleft()
            for y in adj[x]:
                if seen[y]:
                    continue
                seen[y] = True
                if x < m:                 # x row i, y column j:  z_j = z_i - C_ij
                    z[y] = z[x] - C[x, y - m]
                else:                     # x column j, y row i:  z_i = z_j + C_ij
                    z[y] = z[x] + C[y, x - m]
                q.append(y)
    return z[:m].copy(), -z[m:]


def components(edges, m: int, n: int) -> np.ndarray:
    """Component label (smallest node index) of every node of the forest."""
    parent = list(range(m + n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    for i, j, _ in edges:
        a, b = find(i), find(m + j)
        if a != b:
            parent[max(a, b)] = min(a, b)
    return np.array([find(x) for x in range(m + n)])


def component_shift(C: np.ndarray, u: np.ndarray, v: np.ndarray, comp: np.ndarray):
    """Shortest-path gauge shifts of the components (step 3): constraints d_A - d_B <= R_AB
    for rows of A and columns of B; Bellman-Ford from a virtual source (d = 0 for all);
    returns the shifted (u + d_A(i), v - d_B(j)), or (u, v) unchanged if there is one
    component or a negative cycle."""
    m, n = C.shape
    labels = sorted(set(comp.tolist()))
    K = len(labels)
    if K <= 1:
        return u, v
    idx = {c: k for k, c in enumerate(labels)}
    A = np.array([idx[c] for c in comp[:m]])
    B = np.array([idx[c] for c in comp[m:]])
    r = C - u[:, None] - v[None, :]
    R = np.full((K, K), np.inf)
    for a_ in range(K):
        for b_ in range(K):
            if a_ != b_:
                blk = r[np.ix_(A == a_, B == b_)]
                if blk.size:
                    R[a_, b_] = blk.min()
    d = np.zeros(K)
    for _ in range(K + 1):
        changed = False
        for a_ in range(K):
            for b_ in range(K):
                if a_ != b_ and np.isfinite(R[a_, b_]) and d[b_] + R[a_, b_] < d[a_]:
                    d[a_] = d[b_] + R[a_, b_]
                    changed = True
        if not changed:
            return u + d[A], v - d[B]
    return u, v


def ctransform_rows(C: np.ndarray, v: np.ndarray) -> np.ndarray:
    """u_i = min_j (C_ij - v_j): the largest u with u_i + v_j <= C_ij for all j."""
    return (C - v[None, :]).min(axis=1)


def ctransform_cols(C: np.ndarray, u: np.ndarray) -> np.ndarray:
    """v_j = min_i (C_ij - u_i)."""
    return (C - u[:, None]).min(axis=0)


def certify(C: np.ndarray, a: np.ndarray, b: np.ndarray, X: np.ndarray, tau: float, duals0=None,
            repairs: int = 3) -> Dict:
    """LP KKT of the plan X (reading R11): basis forests of {X >= tau} (with up to
    `repairs` forests, step 5), tree duals, component gauges, row then column
    c-transforms, and the entropic candidate duals0 = (u0, v0) if given; the largest
    certified bound wins.  Returns u, v (dual feasible), dual_obj = <a,u>+<b,v> (<= LP*),
    primal = ||Xe-a||_1 + ||X^Te-b||_1, pobj = <C,X>, gap = pobj - dual_obj,
    dual_inf = max(0, max_ij u_i + v_j - C_ij), the first forest, the tree duals of the
    best forest (u_tree, v_tree), the number of forests tried and of components, and
    how many rows / columns the winning c-transform changed."""
    m, n = C.shape
    mask = X >= tau
    rows, cols = np.nonzero(mask)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    val = X[rows, cols]
    pobj = float((C * X).sum())
    primal = float(np.abs(X.sum(1) - a).sum() + np.abs(X.sum(0) - b).sum())
    best = None
    first_forest = None
    forced = np.zeros(len(val), dtype=bool)
    tol_rc = 1e-13 * (1.0 + abs(pobj))
    rounds = 0
    ncomp = 0
    for rnd in range(repairs):
        w = np.where(forced, 4.0, val)
        forest = max_spanning_forest(rowptr, cols, w, m, n)
        if first_forest is None:
            first_forest = forest
        u0, v0 = tree_duals(C, forest, m, n)
        comp = components(forest, m, n)
        ncomp = len(set(comp.tolist()))
        u0, v0 = component_shift(C, u0, v0, comp)
        u = ctransform_rows(C, v0)
        v = ctransform_cols(C, u)
        D = float(a @ u + b @ v)
        rounds = rnd + 1
        if best is None or D > best[0]:
            best = (D, u, v, u0, v0, 1)
        if rnd + 1 == repairs:
            break
        viol = (C[rows, cols] - u0[rows] - v0[cols]) < -tol_rc
        if not viol.any():
            break
        forced |= viol
    if duals0 is not None:
        u = ctransform_rows(C, duals0[1])
        v = ctransform_cols(C, u)
        D = float(a @ u + b @ v)
        if D > best[0]:
            best = (D, u, v, duals0[0], duals0[1], 0)
    dual_obj, u, v, u0, v0, used_tree = best
    dual_inf = float(max(0.0, (u[:, None] + v[None, :] - C).max()))
    tol = 1e-12 * (1.0 + float(np.abs(C).max()))          # "changed" beyond rounding
    return dict(u=u, v=v, u_tree=u0, v_tree=v0, forest=first_forest, dual_obj=dual_obj, pobj=pobj,
                primal=primal, gap=pobj - dual_obj, dual_inf=dual_inf, used_tree=used_tree,
                forests=rounds, components=ncomp,
                rows_changed=int(np.count_nonzero(np.abs(u - u0) > tol)),
                cols_changed=int(np.count_nonzero(np.abs(v - v0) > tol)))
