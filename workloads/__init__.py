"""Seeded synthetic OT instances shaped like the paper's workloads.

This module is shared by the oracle tests and the CUDA path. It only *draws*
inputs (points, dense costs, marginals, the cost normalisation constant); it
holds none of the PINS arithmetic (no plans, potentials, sweeps, Newton steps).

Cost model: point coordinates are quantised onto an
integer lattice so that every pairwise distance D_ij is an exact integer in
both fp64 and fp32; the cost is C_ij = D_ij * cost_scale with
cost_scale = fl(1 / max_ij D_ij) ("scaled to max 1", BASELINE.json configs).
Because D_ij is exact, C_ij is bit-identical wherever it is evaluated.
"""
from .gen import Workload, make, CONFIGS, config_names

__all__ = ["Workload", "make", "CONFIGS", "config_names"]
