"""Seeded generators for the five BASELINE.json configurations.

Each generator returns a :class:`Workload`. Recipes (also in DESIGN.md):

* ``c0_pts64``   m=n=64, 2-D points uniform in [0,1]^2 quantised to 2^-16,
  squared Euclidean cost, uniform marginals, eta=1e-2.
* ``c1_rand1k``  m=n=1024, dense cost i.i.d. U[0,1], marginals U(0.1,1)
  normalised, eta=1e-2.
* ``c2_img4k``   m=n=4096, two 64x64 synthetic grey histograms (3-8 Gaussian
  blobs + 1e-6 floor, normalised), squared grid distance, eta=5e-3.
  (Stands in for the paper's MNIST / augmented-MNIST images, §5.1.)
* ``c3_gmm10k``  m=n=10000, points from an 8-component Gaussian mixture in
  R^10 quantised to 1/64, squared Euclidean cost, marginals U(0.1,1)
  normalised, eta=1e-3.
* ``c4_l1rect``  m=8192, n=16384, 3-D points uniform in [0,1]^3 quantised to
  2^-20, L1 cost, marginals Dirichlet(1), eta=1e-3.

The point sets of c0, c3 and c4 are quantised onto integer lattices (so that
distances are exact in fp32 and fp16, which the fast cost paths exploit); the
``*_r`` variants are the same configurations with REAL-valued coordinates as
BASELINE.json writes them (no rounding), which exercise the fp64 cost paths:

* ``c0_pts64_r``   as c0 with points uniform in [0,1]^2 (plain floats).
* ``c3_gmm10k_r``  as c3 with the Gaussian-mixture points unrounded.
* ``c4_l1rect_r``  as c4 with points uniform in [0,1]^3 (plain floats).

``scale`` (default 1.0) shrinks m and n proportionally for small parity cases;
the *structure* (value distribution, cost kind) is unchanged.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, Optional

import numpy as np

COST_DENSE = 0
COST_SQEUCLID = 1
COST_L1 = 2


@dataclass
class Workload:
    name: str
    m: int
    n: int
    kind: int                      # COST_DENSE / COST_SQEUCLID / COST_L1
    a: np.ndarray                  # (m,) float64, sums to 1, > 0
    b: np.ndarray                  # (n,) float64, sums to 1, > 0
    eta: float
    C: Optional[np.ndarray] = None  # (m,n) float64 for COST_DENSE
    X: Optional[np.ndarray] = None  # (m,d) float64 integer-valued coordinates
    Y: Optional[np.ndarray] = None  # (n,d) float64 integer-valued coordinates
    cost_scale: float = 1.0         # C_ij = D_ij * cost_scale
    meta: Dict = field(default_factory=dict)

    @property
    def d(self) -> int:
        return 0 if self.X is None else int(self.X.shape[1])


def _normalise(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    return v / v.sum()


def _max_pair_distance(X: np.ndarray, Y: np.ndarray, kind: int) -> float:
    """max_ij D_ij over all pairs (blocked): exact integer arithmetic for lattice
    points, fp64 for real-valued points."""
    integral = bool(np.all(X == np.rint(X)) and np.all(Y == np.rint(Y)))
    Xi = X.astype(np.int64) if integral else np.asarray(X, dtype=np.float64)
    Yi = Y.astype(np.int64) if integral else np.asarray(Y, dtype=np.float64)
    best = 0
    bs = max(1, 2_000_000 // max(1, Yi.shape[0]))
    for s in range(0, Xi.shape[0], bs):
        diff = Xi[s:s + bs, None, :] - Yi[None, :, :]
        if kind == COST_SQEUCLID:
            D = (diff * diff).sum(-1)
        else:
            D = np.abs(diff).sum(-1)
        best = max(best, D.max())
    return float(best)


def _points_workload(name, X, Y, kind, a, b, eta, meta=None) -> Workload:
    dmax = _max_pair_distance(X, Y, kind)
    scale = 1.0 / dmax if dmax > 0 else 1.0
    return Workload(name=name, m=X.shape[0], n=Y.shape[0], kind=kind, a=a, b=b,
                    eta=eta, X=X.astype(np.float64), Y=Y.astype(np.float64),
                    cost_scale=scale, meta=meta or {})


def c0_pts64(seed: int = 0, scale: float = 1.0, lattice: bool = True) -> Workload:
    rng = np.random.default_rng(seed)
    n = max(2, int(round(64 * scale)))
    q = float(2 ** 16) if lattice else 1.0
    X = rng.random((n, 2)) * q
    Y = rng.random((n, 2)) * q
    if lattice:
        X, Y = np.floor(X), np.floor(Y)
    a = np.full(n, 1.0 / n)
    b = np.full(n, 1.0 / n)
    return _points_workload("c0_pts64" if lattice else "c0_pts64_r", X, Y, COST_SQEUCLID, a, b, 1e-2,
                            meta={"lattice": lattice})


def c1_rand1k(seed: int = 1, scale: float = 1.0) -> Workload:
    rng = np.random.default_rng(seed)
    n = max(2, int(round(1024 * scale)))
    C = rng.random((n, n))
    a = _normalise(rng.uniform(0.1, 1.0, n))
    b = _normalise(rng.uniform(0.1, 1.0, n))
    return Workload(name="c1_rand1k", m=n, n=n, kind=COST_DENSE, a=a, b=b,
                    eta=1e-2, C=C)


def _blob_image(rng, side: int) -> np.ndarray:
    yy, xx = np.mgrid[0:side, 0:side].astype(np.float64)
    img = np.zeros((side, side))
    for _ in range(int(rng.integers(3, 9))):
        cx, cy = rng.uniform(0, side - 1, 2)
        sx, sy = rng.uniform(side / 32, side / 6, 2)
        w = rng.uniform(0.2, 1.0)
        img += w * np.exp(-0.5 * (((xx - cx) / sx) ** 2 + ((yy - cy) / sy) ** 2))
    img += 1e-6
    return img.ravel()


def c2_img4k(seed: int = 2, scale: float = 1.0) -> Workload:
    rng = np.random.default_rng(seed)
    side = max(2, int(round(64 * np.sqrt(scale))))
    a = _normalise(_blob_image(rng, side))
    b = _normalise(_blob_image(rng, side))
    idx = np.arange(side * side)
    P = np.stack([idx % side, idx // side], axis=1).astype(np.float64)
    return _points_workload("c2_img4k", P, P.copy(), COST_SQEUCLID, a, b, 5e-3,
                            meta={"side": side})


def c3_gmm10k(seed: int = 3, scale: float = 1.0, lattice: bool = True) -> Workload:
    rng = np.random.default_rng(seed)
    n = max(2, int(round(10000 * scale)))
    d, K = 10, 8
    means = rng.normal(0.0, 2.0, (K, d))
    stds = rng.uniform(0.3, 1.0, K)
    w = _normalise(rng.uniform(0.5, 1.5, K))

    def draw(cnt):
        comp = rng.choice(K, size=cnt, p=w)
        pts = means[comp] + stds[comp, None] * rng.normal(size=(cnt, d))
        return np.rint(pts * 64.0) if lattice else pts   # lattice 1/64 -> integer coordinates

    X = draw(n)
    Y = draw(n)
    a = _normalise(rng.uniform(0.1, 1.0, n))
    b = _normalise(rng.uniform(0.1, 1.0, n))
    return _points_workload("c3_gmm10k" if lattice else "c3_gmm10k_r", X, Y, COST_SQEUCLID, a, b, 1e-3,
                            meta={"lattice": lattice})


def c4_l1rect(seed: int = 4, scale: float = 1.0, lattice: bool = True) -> Workload:
    rng = np.random.default_rng(seed)
    m = max(2, int(round(8192 * scale)))
    n = max(2, int(round(16384 * scale)))
    q = float(2 ** 20) if lattice else 1.0
    X = rng.random((m, 3)) * q
    Y = rng.random((n, 3)) * q
    if lattice:
        X, Y = np.floor(X), np.floor(Y)
    a = rng.dirichlet(np.ones(m))
    b = rng.dirichlet(np.ones(n))
    return _points_workload("c4_l1rect" if lattice else "c4_l1rect_r", X, Y, COST_L1, _normalise(a),
                            _normalise(b), 1e-3, meta={"lattice": lattice})


CONFIGS: Dict[str, Callable[..., Workload]] = {
    "c0_pts64": c0_pts64,
    "c1_rand1k": c1_rand1k,
    "c2_img4k": c2_img4k,
    "c3_gmm10k": c3_gmm10k,
    "c4_l1rect": c4_l1rect,
    # real-valued (non-lattice) variants of the point configurations
    "c0_pts64_r": lambda seed=0, scale=1.0: c0_pts64(seed, scale, lattice=False),
    "c3_gmm10k_r": lambda seed=3, scale=1.0: c3_gmm10k(seed, scale, lattice=False),
    "c4_l1rect_r": lambda seed=4, scale=1.0: c4_l1rect(seed, scale, lattice=False),
}


def config_names():
    return list(CONFIGS)


def make(name: str, seed: Optional[int] = None, scale: float = 1.0) -> Workload:
    fn = CONFIGS[name]
    return fn(scale=scale) if seed is None else fn(seed=seed, scale=scale)


def random_potentials(m: int, n: int, seed: int, spread: float = 1.0):
    """Seeded (f, g) test vectors (not PINS arithmetic, just random inputs)."""
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, spread, m), rng.normal(0.0, spread, n)
