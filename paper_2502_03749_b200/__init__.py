"""paper_2502_03749_b200 -- PINS (arXiv 2502.03749) hot path on B200.

The product is ``libpins_b200.so`` (C ABI in include/pins.h); ``pins`` is its
thin Python binding.
"""
from . import pins  # noqa: F401

__all__ = ["pins"]
