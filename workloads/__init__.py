"""Seeded synthetic workload generators shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no quantisation, no
products, no thresholding): it only draws the measurement matrix Phi, the
sparse ground truth x and the noisy observations y = Phi x + e with the shapes
and distributions of BASELINE.json's configs (recipe in DESIGN.md "Input
recipe").  Both ``oracle`` and ``paper_1802_04907_b200`` may import it.
"""
from .gen import (  # noqa: F401
    mix64, counter_hash, gauss_int, gauss_scale32, gaussian_block, ProblemSpec,
    gaussian_problem, radio_problem, config_problem, CONFIGS,
)
