"""Brute force over every stage-and-strategy assignment -- TEST INFRASTRUCTURE ONLY.

For tiny instances only.  Enumerates, for every candidate config (deg, c):
  * every placement P satisfying Eqs. (6)-(7): stages are
    ordered, contiguous, non-empty intervals (reading A-3), i.e. stage_of is
    non-decreasing from 0 to deg-1 in steps of 0 or 1;
  * every strategy vector S satisfying Eq. (8);
and evaluates literally
  p_i = sum_{u in i} A_u[k_u] + sum_{<u,v> in E, u,v in i} R_uv[k_u][k_v]   (Eq. 3)
  o_j = O[e_j] (+ Rcut[e_j][k_{e_j}][k_{e_j+1}] when the config gives the
        strategy-dependent cut cost, Eq. 4 with R'; e_j = last layer of stage j)
  mem_i = sum_{u in i} M_u[k_u] <= cap_i (the stage's cap, = cap unless the
          config gives per-stage caps: heterogeneous devices, PAPER.md:161;
          M = the stage's own table M_stage[i] when the config gives one: the
          1F1B schedule, footnote of PAPER.md:122, reading A-32)            (Eq. 5)
  tpi = sum p + sum o + (c-1) * max(P u O)                                  (Eq. 2)
and returns the minimum of the key (tpi, deg, c, stage_of, strategy_of) --
with Rcut: (tpi, deg, c, stage_of, boundary vector, strategy_of), the
boundary vector (k_{e_1}, k_{e_1+1}, k_{e_2}, k_{e_2+1}, ...) (reading A-31).
"""
from __future__ import annotations

import itertools

import numpy as np

INT64_MAX = (1 << 63) - 1


def placements(L, deg):
    """All stage_of vectors in lexicographic order."""
    if deg > L:
        return
    for cuts in itertools.combinations(range(1, L), deg - 1):  # cut before layer x
        so, st = [], 0
        cs = set(cuts)
        for u in range(L):
            if u in cs:
                st += 1
            so.append(st)
        yield so
    # itertools.combinations emits cut sets in lexicographic order of the cut
    # positions, which is the reverse-lexicographic order of stage_of; callers
    # sort explicitly.


def solve_cfg(t, cfg, guard=2_000_000):
    L, cap, s = t["L"], t["cap"], t.get("skip_src", -1)
    S, deg, c = cfg["n_strat"], cfg["deg"], cfg["c"]
    A = np.asarray(cfg["A"], dtype=np.int64).reshape(L, S)
    MS = cfg.get("M_stage")
    Ms = ([np.asarray(cfg["M"], dtype=np.int64).reshape(L, S)] * deg if MS is None
          else list(np.asarray(MS, dtype=np.int64).reshape(deg, L, S)))
    R = np.asarray(cfg["R"], dtype=np.int64).reshape(max(L - 1, 0), S, S) if L > 1 else None
    # skip edges: one source (skip_src, Rskip) or several (skip_srcs, Rskips; NEXT-4, reading A-33)
    skips = []
    if cfg.get("Rskip") is not None and s >= 0:
        skips.append((s, np.asarray(cfg["Rskip"], dtype=np.int64).reshape(L, S, S)))
    for j, sj in enumerate(t.get("skip_srcs") or []):
        if cfg.get("Rskips") is not None:
            skips.append((sj, np.asarray(cfg["Rskips"], dtype=np.int64).reshape(-1, L, S, S)[j]))
    O = np.zeros(max(L - 1, 0), dtype=np.int64) if cfg.get("O") is None else np.asarray(cfg["O"], dtype=np.int64)
    caps = [cap] * deg if cfg.get("stage_cap") is None else [int(x) for x in cfg["stage_cap"]]
    RC = None if cfg.get("Rcut") is None else np.asarray(cfg["Rcut"], dtype=np.int64).reshape(L - 1, S, S)
    places = sorted(placements(L, deg))
    if not places:
        return None
    if S ** L * len(places) > guard:
        raise ValueError("instance too large for brute force")
    # every strategy vector, lexicographic order (itertools.product order)
    K = np.array(list(itertools.product(range(S), repeat=L)), dtype=np.int64).reshape(-1, L)
    idx = np.arange(L)
    Au = A[idx, K]                      # [N, L]  A_u[k_u]
    Mu = [Mi[idx, K] for Mi in Ms]      # per stage [N, L]
    Ru = R[idx[:-1], K[:, :-1], K[:, 1:]] if L > 1 else np.zeros((len(K), 0), np.int64)  # chain edge u->u+1
    best = None
    for so in places:
        so = np.asarray(so)
        ends = [int(np.max(np.nonzero(so == i)[0])) for i in range(deg)]
        starts = [int(np.min(np.nonzero(so == i)[0])) for i in range(deg)]
        total = np.zeros(len(K), dtype=np.int64)
        mx = np.zeros(len(K), dtype=np.int64)
        feas = np.ones(len(K), dtype=bool)
        for i in range(deg):
            a, b = starts[i], ends[i]
            p = Au[:, a:b + 1].sum(axis=1) + Ru[:, a:b].sum(axis=1)
            for sj, Rs in skips:  # every skip edge <s_j, v> with both ends in the stage (Eq. 3)
                if a <= sj:
                    for v in range(sj + 2, b + 1):
                        p = p + Rs[v, K[:, sj], K[:, v]]
            mem = Mu[i][:, a:b + 1].sum(axis=1)
            feas &= mem <= caps[i]
            total += p
            mx = np.maximum(mx, p)
            if i + 1 < deg:
                o = O[b] + (RC[b, K[:, b], K[:, b + 1]] if RC is not None else 0)
                total += o
                mx = np.maximum(mx, o)
        f = total + (c - 1) * mx
        f = np.where(feas, f, INT64_MAX)
        j = int(np.argmin(f))            # first = lexicographically smallest strategy vector
        if f[j] == INT64_MAX:
            continue
        if RC is not None:               # reading A-31: the boundary vector before strategy_of
            cand = np.nonzero(f == f[j])[0]
            bidx = [x for e in ends[:-1] for x in (e, e + 1)]
            j = int(min(cand, key=lambda r: (tuple(K[r, bidx]), tuple(K[r]))))
        if best is None or f[j] < best[0]:   # placements in lexicographic order: keep first
            best = (int(f[j]), list(map(int, so)), list(map(int, K[j])))
    return best


def solve_tables(t, guard=2_000_000):
    """Minimum of the key (tpi, deg, c, stage_of, strategy_of) over all configs."""
    per = []
    win = None
    for i, cfg in enumerate(t["cfgs"]):
        b = solve_cfg(t, cfg, guard)
        per.append(INT64_MAX if b is None else b[0])
        if b is None:
            continue
        key = (b[0], cfg["deg"], cfg["c"], b[1], b[2])
        if win is None or key < win[0]:
            win = (key, i)
    if win is None:
        return {"objective": INT64_MAX, "cfg_index": -1, "cfg_objective": per}
    (f, deg, c, so, sk), i = win
    return {"objective": f, "cfg_index": i, "deg": deg, "c": c, "stage_of": so, "strategy_of": sk,
            "cfg_objective": per}
