"""Seeded synthetic workload shared by the CUDA path's tests/bench and the CPU oracle.

This package holds NONE of the method's arithmetic: only parameter values quoted from the
paper's tables (``presets``) and seeded input generators (``gen``) with the shapes of the
Shadow-hand workload.  Both bindings -- ``paper_1906_11633_b200.dr`` and
``oracle.oracle`` -- translate the same preset dict into their own parameter structs.
"""
from . import presets, gen  # noqa: F401
