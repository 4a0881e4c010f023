"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no cost model, no DP, no
objective).  It only draws integer inputs:

* ``gen.tables``   -- level-1 integer cost tables (A, M, R, Rskip, O per
  candidate config), e.g. the frozen toy instance and random tiny instances.
* ``gen.profiles`` -- level-2 synthetic *profiling results* (PAPER.md:87-90,
  Sec. 3.1): per-layer forward time / parameter bytes / activation bytes per
  TP size, edges, and an alpha-beta cluster record, shaped like the paper's
  evaluated models (Table 5).

Both the oracle (``oracle/``) and the product binding consume the plain
Python dicts these functions return; each side marshals them itself.
"""
from . import tables, profiles  # noqa: F401
