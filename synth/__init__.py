"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no operator, no right-hand side,
no solver step).  It only draws the problem parameters and data maps with the
recipe of SURVEY.md section 8(d), which stands in for the paper's Planck maps
(n = 9 maps, 12 base faces, N = 4^10, m = 4).
"""

from .problems import CONFIGS, PatchProblem, make_patch, make_config, config_patches

__all__ = ["CONFIGS", "PatchProblem", "make_patch", "make_config", "config_patches"]
