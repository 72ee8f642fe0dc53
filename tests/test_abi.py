"""The C ABI library loads and exports every symbol include/pins.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "pins.h")


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(pins_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("pins_solve", "pins_sinkhorn_sweep", "pins_newton_step", "pins_evaluate",
                 "pins_cg", "pins_center_update", "pins_residuals", "pins_sparsify_dense"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2502_03749_b200 import build as b
    lib_path = b.build()              # nvcc cross-compiles sm_100a without a GPU
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2502_03749_b200 import pins
    assert set(pins.EXPORTS) == set(declared_symbols())


def test_struct_layouts_match_header():
    from paper_2502_03749_b200 import pins
    # pins_problem: 2 int64 (16) + 2 int32 (8) + 8 pointer/double/int64 fields (64) = 88 bytes
    assert ctypes.sizeof(pins.Problem) == 88
    assert pins.Params.outer_tol.offset == 8 and pins.Params.sink_tol.offset == 24
    assert ctypes.sizeof(pins.Params) == 112


def test_default_params_follow_appendix_a2():
    from paper_2502_03749_b200 import build as b
    b.build()
    from paper_2502_03749_b200 import pins
    p = pins.default_params()
    assert (p.K, p.T1, p.T2) == (500, 50000, 20)
    assert p.outer_tol == 1e-4 and p.newton_tol == 1e-8 and p.sink_tol == 6.3e-4


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2502_03749_b200 import pins
    with pytest.raises(RuntimeError):
        pins.center_init(None)
