"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no chase, no reflector application):
only a counter-based splitmix64 stream and the recipes that turn it into inputs
(DESIGN.md §3 "Input recipe").  Both a numpy and a torch implementation of the same
counter-based generator are provided so device-side generation for the bench is
bitwise identical to host-side generation for the oracle (tests/test_inputs.py).
"""
from .synth import (  # noqa: F401
    GAMMA, splitmix64_np, uniform_pm1_np, uniform_pm1_torch,
    band_matrix, dense_symmetric, synthetic_reflectors, synthetic_reflectors_torch, synthetic_q_np, synthetic_q_torch,
    config_seed, CONFIGS, spd_matrix, lower_triangular_cm_np, lower_triangular_cm_torch,
    band_matrix_c, synthetic_reflectors_c, synthetic_q_c_np,
)
