"""Strategy-space ablation of UniAP (Sec. 4.4; SURVEY.md
Sec. 8f NEXT-3): the unified space against inter-layer-only and
intra-layer-only spaces.

The paper constrains "the strategy space to inter-layer-only and
intra-layer-only strategies" without listing them (its Fig. 6 is lost,
reading A-21).  Readings (A-25):

  unified     every Algorithm-1 candidate (deg, c), every (t, f, d) strategy
  intra-only  no pipeline: the deg = 1 candidate only
  inter-dp    pipelines of every degree, each stage replicated by plain data
              parallelism only (strategy index 0 = (1, 1, g), App. D)
  inter-pp    pure pipeline: deg = n (one device per stage, |S| = 1)

Each variant is a restriction of the unified problem expressed on the level-1
tables (candidates dropped, or strategies forbidden through M = cap + 1, the
ABI's "forbidden" encoding), so the same solver -- GPU or oracle -- solves it,
and unified <= every variant by construction.  This module only selects
table entries; it holds none of the method's arithmetic.
"""
from __future__ import annotations

import copy

import numpy as np

VARIANTS = ("unified", "intra-only", "inter-dp", "inter-pp")


def restrict(t, variant, n_dev):
    """The level-1 tables of one ablation variant (a new dict)."""
    if variant == "unified":
        return t
    out = copy.copy(t)
    cap = t["cap"]
    if variant == "intra-only":
        out["cfgs"] = [c for c in t["cfgs"] if c["deg"] == 1]
    elif variant == "inter-pp":
        out["cfgs"] = [c for c in t["cfgs"] if c["deg"] == n_dev]
    elif variant == "inter-dp":
        cfgs = []
        for c in t["cfgs"]:
            c = dict(c)
            M = np.array(c["M"], dtype=np.int32, copy=True)
            M[:, 1:] = cap + 1  # every strategy but pure data parallelism is forbidden
            c["M"] = M
            cfgs.append(c)
        out["cfgs"] = cfgs
    else:
        raise ValueError(variant)
    return out
