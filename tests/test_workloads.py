"""Input recipes: determinism, shapes, marginals, exact lattice costs."""
import numpy as np
import pytest

from workloads import make, config_names
from workloads.gen import COST_DENSE


@pytest.mark.parametrize("name", config_names())
def test_small_scale_recipe(name):
    sc = 0.25 if name.startswith("c0") else 0.01
    w = make(name, scale=sc)
    w2 = make(name, scale=sc)
    assert w.a.shape == (w.m,) and w.b.shape == (w.n,)
    assert (w.a > 0).all() and (w.b > 0).all()
    assert abs(w.a.sum() - 1) < 1e-12 and abs(w.b.sum() - 1) < 1e-12
    assert np.array_equal(w.a, w2.a) and np.array_equal(w.b, w2.b)
    if w.kind == COST_DENSE:
        assert np.array_equal(w.C, w2.C) and 0 <= w.C.min() and w.C.max() < 1
    else:
        assert np.array_equal(w.X, w2.X) and np.array_equal(w.Y, w2.Y)
        if w.meta.get("lattice", True):
            assert np.array_equal(w.X, np.rint(w.X)) and np.array_equal(w.Y, np.rint(w.Y))
            assert 0 < w.cost_scale <= 1
        else:   # real-valued variants (BASELINE.json as written): not on any lattice
            assert not np.array_equal(w.X, np.rint(w.X))
            assert w.name.endswith("_r") and 0 < w.cost_scale


def test_full_size_shapes():
    assert (make("c0_pts64").m, make("c0_pts64").n) == (64, 64)
    w = make("c2_img4k")
    assert (w.m, w.n) == (4096, 4096) and w.eta == 5e-3
    assert abs(w.cost_scale * 2 * 63 ** 2 - 1.0) < 1e-15
