"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This package holds NONE of the gamma-EigenGame arithmetic (no products, Gram
tables, updates or normalisations of the method): it only draws the random
numbers the method consumes (problem matrices, paired data views, the Gaussian
draws of the initial strategies) following the recipes of BASELINE.json's
configs.  Neither `oracle/` nor `paper_2206_04993_b200/` is imported here.
"""
from .workloads import (  # noqa: F401
    CONFIGS,
    WorkloadConfig,
    haar_orthogonal,
    dense_gep_small,
    dense_gep_large,
    cca_views,
    gaussian_init,
    appendix_b_example,
    planted_cca_views,
)
