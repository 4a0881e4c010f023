"""Seeded level-1 inputs: integer cost tables per candidate config.

A *tables* dict (consumed by both ``oracle.oracle`` and the product binding):

    {"L": int, "cap": int, "skip_src": int (-1 = none),
     "cfgs": [{"deg": int, "c": int, "n_strat": int,
               "A": int32[L, S], "M": int32[L, S],
               "R": int32[L-1, S, S],          # R[u][k][l]: edge u->u+1
               "Rskip": int32[L, S, S] | None, # Rskip[v][k_s][k_v]: edge skip_src->v
               "O": int32[L-1] | None}, ...]}

Entries are drawn, never computed from the method.  ``M[u][k] > cap`` marks a
forbidden (layer, strategy) pair.
"""
from __future__ import annotations

import numpy as np

__all__ = ["toy_tables", "random_tables", "large_random_tables", "with_1f1b", "with_skip_sources", "TOY_GRID"]

TOY_GRID = [(1, 1), (1, 2), (2, 1), (2, 2)]


def toy_tables(cands=TOY_GRID):
    """The frozen toy instance of SURVEY.md Sec. 8c-P: L=4, |S|=3, cap=7 (Q=8).

    A(c=1) = [[6,4,5],[6,3,4],[5,3,4],[6,4,5]], A(c=2) = ceil(a/2)+1 elementwise,
    M = [[1,3,2],[1,3,2],[1,3,2],[2,4,3]], R = [[0,2,1],[2,0,1],[1,1,0]] on every
    chain edge, O = [2,2,2], no skip edge.  The table values are data (the
    survey's), independent of deg.
    """
    A1 = np.array([[6, 4, 5], [6, 3, 4], [5, 3, 4], [6, 4, 5]], dtype=np.int32)
    A2 = (A1 + 1) // 2 + 1
    M = np.array([[1, 3, 2], [1, 3, 2], [1, 3, 2], [2, 4, 3]], dtype=np.int32)
    R1 = np.array([[0, 2, 1], [2, 0, 1], [1, 1, 0]], dtype=np.int32)
    R = np.stack([R1, R1, R1]).astype(np.int32)
    O = np.array([2, 2, 2], dtype=np.int32)
    cfgs = []
    for deg, c in cands:
        cfgs.append({"deg": deg, "c": c, "n_strat": 3,
                     "A": (A1 if c == 1 else A2).copy(), "M": M.copy(),
                     "R": R.copy(), "Rskip": None, "O": O.copy()})
    return {"L": 4, "cap": 7, "skip_src": -1, "cfgs": cfgs}


def _draw_cfg(rng, L, S, cap, skip_src, dist, forbid_p, with_O):
    if dist == "ties":
        A = rng.integers(0, 3, size=(L, S))
        R = rng.integers(0, 2, size=(max(L - 1, 0), S, S))
        O = rng.integers(0, 2, size=max(L - 1, 0))
        Rs = rng.integers(0, 2, size=(L, S, S))
    else:
        A = rng.integers(0, 10, size=(L, S))
        R = rng.integers(0, 6, size=(max(L - 1, 0), S, S))
        O = rng.integers(0, 4, size=max(L - 1, 0))
        Rs = rng.integers(0, 6, size=(L, S, S))
    # zero diagonal with probability 1/2 (identical layouts reshard for free)
    if L > 1 and rng.random() < 0.5:
        for u in range(L - 1):
            np.fill_diagonal(R[u], 0)
    M = rng.integers(0, min(cap, 4) + 1, size=(L, S)) if cap >= 0 else np.zeros((L, S))
    if forbid_p > 0:
        M = np.where(rng.random((L, S)) < forbid_p, cap + 1, M)
    Rskip = None
    if skip_src >= 0:
        Rskip = np.zeros((L, S, S), dtype=np.int64)
        Rskip[skip_src + 2:] = Rs[skip_src + 2:]
    return {"A": A.astype(np.int32), "M": M.astype(np.int32),
            "R": R.astype(np.int32).reshape(max(L - 1, 0), S, S),
            "Rskip": None if Rskip is None else Rskip.astype(np.int32),
            "O": O.astype(np.int32) if with_O else None}


def random_tables(seed, L=None, S_max=3, cap=None, n_cfg=None, dist=None,
                  skip_p=0.4, forbid_p=None, deg_max=None, stage_caps=False, rcut=False):
    """Random tiny instance for brute-force checks (SURVEY.md Sec. 4 tier T0).

    L <= 6, |S| <= 3, cap <= 7 by default; skip edges in ``skip_p`` of the
    instances; cut costs O != 0; 'uniform' or tie-heavy ('ties') values;
    forbidden entries (M = cap+1).  ``stage_caps``: every config also gets a
    per-stage memory cap (``stage_cap``, drawn in [0, cap]; heterogeneous
    devices).  ``rcut``: every config also gets a strategy-dependent cut cost
    ``Rcut[e][k][l]`` (Eq. 4 with R' per strategy pair), values like O's.
    """
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 7)) if L is None else L
    cap = int(rng.integers(0, 8)) if cap is None else cap
    dist = ("ties" if rng.random() < 0.4 else "uniform") if dist is None else dist
    forbid_p = (0.15 if rng.random() < 0.5 else 0.0) if forbid_p is None else forbid_p
    skip_src = -1
    if L >= 3 and rng.random() < skip_p:
        skip_src = int(rng.integers(0, L - 2))
    n_cfg = int(rng.integers(1, 5)) if n_cfg is None else n_cfg
    deg_max = L + 1 if deg_max is None else deg_max
    pairs = set()
    while len(pairs) < n_cfg:
        pairs.add((int(rng.integers(1, deg_max + 1)), int(rng.integers(1, 5))))
    cfgs = []
    for deg, c in sorted(pairs, key=lambda p: rng.random()):
        S = int(rng.integers(1, S_max + 1))
        d = _draw_cfg(rng, L, S, cap, skip_src, dist, forbid_p, with_O=rng.random() < 0.8)
        d.update({"deg": deg, "c": c, "n_strat": S})
        cfgs.append(d)
    if stage_caps:
        crng = np.random.default_rng(seed + 12_345_678)  # separate stream: the tables above are unchanged
        for d in cfgs:
            d["stage_cap"] = crng.integers(max(cap - 3, 0), cap + 1, size=d["deg"]).astype(np.int32)
    if rcut:
        rrng = np.random.default_rng(seed + 23_456_789)
        for d in cfgs:
            S = d["n_strat"]
            hi = 2 if dist == "ties" else 5
            d["Rcut"] = rrng.integers(0, hi, size=(max(L - 1, 0), S, S)).astype(np.int32)
    return {"L": L, "cap": cap, "skip_src": skip_src, "cfgs": cfgs}


def large_random_tables(seed, L, S_list, cap, cands, skip_src=-1, dist="uniform",
                        forbid_p=0.05, vmax=1 << 20, mem_max=None, stage_caps=False):
    """Random instance at GPU-parity sizes (several tiles and a ragged tail).

    ``S_list[i]`` strategies for candidate ``cands[i] = (deg, c)``; entries of
    A, R, Rskip, O in [0, vmax] (so the per-config sum bound of
    SURVEY.md Sec. 8c A-9 holds for L <= 64 when vmax <= 2^20); memory entries
    in [0, mem_max] (default: about cap / (L/2) so that memory binds).
    """
    rng = np.random.default_rng(seed)
    if mem_max is None:
        mem_max = max(1, (2 * cap) // max(L, 1))
    cfgs = []
    for (deg, c), S in zip(cands, S_list):
        if dist == "ties":
            A = rng.integers(0, 3, size=(L, S)) * (vmax // 4)
            R = rng.integers(0, 2, size=(L - 1, S, S)) * (vmax // 4)
        else:
            A = rng.integers(0, vmax + 1, size=(L, S))
            R = rng.integers(0, vmax + 1, size=(L - 1, S, S))
        for u in range(L - 1):
            np.fill_diagonal(R[u], 0)
        M = rng.integers(0, mem_max + 1, size=(L, S))
        M = np.where(rng.random((L, S)) < forbid_p, cap + 1, M)
        Rskip = None
        if skip_src >= 0:
            Rskip = np.zeros((L, S, S), dtype=np.int64)
            Rskip[skip_src + 2:] = rng.integers(0, vmax + 1, size=(L - skip_src - 2, S, S))
        O = rng.integers(0, vmax + 1, size=L - 1)
        cfgs.append({"deg": deg, "c": c, "n_strat": S,
                     "A": A.astype(np.int32), "M": M.astype(np.int32),
                     "R": R.astype(np.int32),
                     "Rskip": None if Rskip is None else Rskip.astype(np.int32),
                     "O": O.astype(np.int32)})
    if stage_caps:  # per-stage caps from at most 3 distinct device sizes (heterogeneous devices)
        crng = np.random.default_rng(seed + 12_345_678)
        for d in cfgs:
            d["stage_cap"] = crng.choice([cap, cap - cap // 4, cap // 2], size=d["deg"]).astype(np.int32)
    return {"L": L, "cap": cap, "skip_src": skip_src, "cfgs": cfgs}


def with_1f1b(t, seed, act_max=None):
    """The same tables with 1F1B-shaped per-stage memory (reading A-32).

    Every config gets a weight part Mw and a per-micro-batch activation part
    Ma (drawn, [L, S]); stage i of deg holds min(c, deg - i) micro-batches,
    so ``M_stage[i] = Mw + min(c, deg - i) * Ma``, and ``M`` becomes GPipe's
    ``Mw + c * Ma`` (all c in flight).  Entries forbidden in the input (M >
    cap) stay forbidden in every stage.  Returns a new dict; ``t`` is untouched.
    """
    rng = np.random.default_rng(seed + 34_567_890)
    L, cap = t["L"], t["cap"]
    out = dict(t, cfgs=[])
    for d in t["cfgs"]:
        S, deg, c = d["n_strat"], d["deg"], d["c"]
        amax = max(1, cap // (2 * max(L, 1) * max(c, 1))) if act_max is None else act_max
        wmax = max(1, cap // max(L, 1))
        Mw = rng.integers(0, wmax + 1, size=(L, S))
        Ma = rng.integers(0, amax + 1, size=(L, S))
        bad = np.asarray(d["M"]) > cap
        M = np.where(bad, cap + 1, np.minimum(Mw + c * Ma, cap + 1))
        MS = np.stack([np.where(bad, cap + 1, np.minimum(Mw + min(c, deg - i) * Ma, cap + 1)) for i in range(deg)])
        out["cfgs"].append(dict(d, M=M.astype(np.int32), M_stage=MS.astype(np.int32)))
    return out


def with_skip_sources(t, seed, n_src, vmax=None):
    """The same tables on a DAG with ``n_src`` skip sources (NEXT-4, reading
    A-33): the chain edges plus edges from each source s_j to every later
    layer v >= s_j + 2, costs ``Rskips[j][v][k_s][k_v]`` drawn like R's
    (rows v < s_j + 2 zero).  Sources distinct and ascending in [0, L - 3]
    (fewer when L is small).  Replaces any single skip source of ``t``."""
    rng = np.random.default_rng(seed + 45_678_901)
    L = t["L"]
    cand = list(range(0, max(L - 2, 0)))
    k = min(n_src, len(cand))
    srcs = sorted(int(x) for x in rng.choice(cand, size=k, replace=False)) if k else []
    out = dict(t, skip_src=-1, skip_srcs=srcs, cfgs=[])
    for d in t["cfgs"]:
        S = d["n_strat"]
        hi = vmax if vmax is not None else int(max(2, np.max(d["R"]) + 1 if d["R"].size else 2))
        Rss = np.zeros((len(srcs), L, S, S), dtype=np.int64)
        for j, sj in enumerate(srcs):
            Rss[j, sj + 2:] = rng.integers(0, hi + 1, size=(L - sj - 2, S, S))
        out["cfgs"].append(dict(d, Rskip=None, Rskips=Rss.astype(np.int32) if srcs else None))
    return out
