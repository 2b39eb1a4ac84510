"""Seeded synthetic input generators shared by the tests, the bench and smoke().

This module holds NONE of the method's arithmetic (no embedding, sketch,
pivoting, coefficient or residual code); it only builds test matrices A with the
shapes and spectra of BASELINE.json's configs C1-C5 (recipes in DESIGN.md §6).
"""
from .gen import (  # noqa: F401
    CONFIGS,
    haar,
    make_c1,
    make_c2,
    make_c3,
    make_c4,
    make_lowrank,
    make_config,
    kahan_witness,
)
