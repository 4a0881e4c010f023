"""Pins of the oracle against closed forms, textbook routines and invariants
(CPU only).  Each test names the property it checks and
the passage that fixes it."""
import itertools

import numpy as np
import pytest

from gen import tables
from oracle import brute

INF = brute.INT64_MAX


def _one(L, S, A, M, R, cap, deg=1, c=1, O=None, Rskip=None, skip=-1):
    cfg = {"deg": deg, "c": c, "n_strat": S, "A": np.asarray(A, np.int32).reshape(L, S),
           "M": np.asarray(M, np.int32).reshape(L, S),
           "R": np.asarray(R, np.int32).reshape(L - 1, S, S),
           "Rskip": None if Rskip is None else np.asarray(Rskip, np.int32), "O": None if O is None else np.asarray(O, np.int32)}
    return {"L": L, "cap": cap, "skip_src": skip, "cfgs": [cfg]}


def _minplus_chain(A, R, a, b, allowed, Rskip=None, s=-1, ks=-1):
    """Textbook tropical product a_a (x) T_{a+1} (x) ... (x) T_b, T_u[k'][k] = R[u-1][k'][k] + A'[u][k]."""
    S = A.shape[1]
    big = np.int64(1) << 50

    def Ap(u):
        x = A[u].astype(np.int64).copy()
        if ks >= 0 and u >= s + 2:
            x += Rskip[u, ks]
        x[~allowed[u]] = big
        if ks >= 0 and u == s:
            x[np.arange(S) != ks] = big
        return x
    v = Ap(a)
    for u in range(a + 1, b + 1):
        T = R[u - 1].astype(np.int64) + Ap(u)[None, :]
        v = np.min(v[:, None] + T, axis=0)
    m = int(v.min())
    return m if m < big else INF


def test_interval_table_is_tropical_chain_product_when_memory_slack(orc):
    """With cap >= sum_u max_k M, P[a][b] = min over the min-plus chain product
    (Eq. 3 with Eq. 5 inactive), including the skip-source conditioning."""
    for seed in range(60):
        rng = np.random.default_rng(seed)
        L, S = int(rng.integers(2, 9)), int(rng.integers(1, 6))
        t = tables.random_tables(seed, L=L, S_max=S, cap=200, n_cfg=1, skip_p=0.5, forbid_p=0.1)
        cfg = t["cfgs"][0]
        P = orc.interval_table(t, 0)
        A, R, M = cfg["A"], cfg["R"], cfg["M"]
        allowed = M <= t["cap"]
        s = t["skip_src"]
        for a in range(L):
            for b in range(a, L):
                if s >= 0 and cfg["Rskip"] is not None and a <= s and s + 2 <= b:
                    want = min(_minplus_chain(A, R, a, b, allowed, cfg["Rskip"], s, ks) for ks in range(cfg["n_strat"]))
                else:
                    want = _minplus_chain(A, R, a, b, allowed)
                assert P[a, b] == want, (seed, a, b)


def test_memory_dimension_is_multiple_choice_knapsack(orc):
    """A = R = 0: P[a][b] is 0 iff some choice of one strategy per layer has
    sum M <= cap (multiple-choice knapsack feasibility), else infeasible."""
    for seed in range(80):
        rng = np.random.default_rng(seed)
        L, S, cap = int(rng.integers(1, 6)), int(rng.integers(1, 4)), int(rng.integers(0, 12))
        M = rng.integers(0, 6, size=(L, S))
        t = _one(L, S, np.zeros((L, S)), M, np.zeros((max(L - 1, 1), S, S))[:L - 1], cap) if L > 1 else \
            {"L": 1, "cap": cap, "skip_src": -1, "cfgs": [{"deg": 1, "c": 1, "n_strat": S, "A": np.zeros((1, S), np.int32),
                                                          "M": M.astype(np.int32), "R": np.zeros((0, S, S), np.int32), "Rskip": None, "O": None}]}
        P = orc.interval_table(t, 0)
        for a in range(L):
            for b in range(a, L):
                ok = any(sum(M[u, k[u - a]] for u in range(a, b + 1)) <= cap
                         for k in itertools.product(range(S), repeat=b - a + 1))
                assert P[a, b] == (0 if ok else INF)


def test_deg1_is_appendix_c_qip(orc):
    """pp = 1 reduces to pure intra-layer search (App. C, Eqs. 9-11,
    PAPER.md:587-607): OPT = P[0][L-1] = an independent chain DP over
    (strategy, exact memory used) states."""
    for seed in range(100):
        rng = np.random.default_rng(seed)
        L, S, cap = int(rng.integers(1, 8)), int(rng.integers(1, 5)), int(rng.integers(0, 15))
        t = tables.random_tables(seed, L=L, S_max=S, cap=cap, n_cfg=1, skip_p=0.0)
        cfg = t["cfgs"][0]
        cfg["deg"], cfg["c"] = 1, 1
        A, M, R = cfg["A"], cfg["M"], cfg["R"]
        states = {(k, int(M[0, k])): int(A[0, k]) for k in range(cfg["n_strat"]) if M[0, k] <= cap}
        for u in range(1, L):
            nxt = {}
            for (kp, mem), cost in states.items():
                for k in range(cfg["n_strat"]):
                    m2 = mem + int(M[u, k])
                    if m2 > cap:
                        continue
                    v = cost + int(R[u - 1, kp, k]) + int(A[u, k])
                    if v < nxt.get((k, m2), INF):
                        nxt[(k, m2)] = v
            states = nxt
        want = min(states.values()) if states else INF
        assert orc.solve_tables(t)["objective"] == want


def test_closed_form_zero_resharding(orc):
    """R = 0 and slack memory: P[a][b] = sum_u min_k A[u][k]; the
    strategies are the smallest argmins (lexicographic tie-break, A-11)."""
    for seed in range(40):
        rng = np.random.default_rng(seed)
        L, S = int(rng.integers(1, 10)), int(rng.integers(1, 7))
        A = rng.integers(0, 5, size=(L, S))
        t = _one(L, S, A, np.zeros((L, S)), np.zeros((L - 1, S, S)), cap=0) if L > 1 else None
        if t is None:
            continue
        P = orc.interval_table(t, 0)
        cs = np.concatenate([[0], np.cumsum(A.min(axis=1))])
        for a in range(L):
            for b in range(a, L):
                assert P[a, b] == cs[b + 1] - cs[a]
        r = orc.solve_tables(t)
        assert r["strategy_of"] == [int(np.argmin(A[u])) for u in range(L)]


def test_closed_form_single_strategy_prefix_sums(orc):
    """|S| = 1 (deg = n): P[a][b] = sum_{a..b} A + sum_{a..b-1} R (prefix sums)."""
    rng = np.random.default_rng(7)
    L = 12
    A = rng.integers(0, 100, size=(L, 1))
    R = rng.integers(0, 100, size=(L - 1, 1, 1))
    t = _one(L, 1, A, np.zeros((L, 1)), R, cap=0)
    P = orc.interval_table(t, 0)
    for a in range(L):
        for b in range(a, L):
            assert P[a, b] == A[a:b + 1].sum() + R[a:b].sum()


def test_c1_O0_tie_break_gives_long_early_stages(orc):
    """c = 1, O = 0, R = 0, slack memory: tpi is placement-independent, so the
    lexicographically smallest stage_of is [0,...,0,1,2,...,deg-1] (A-11)."""
    for deg in range(1, 7):
        L, S = 8, 3
        A = np.random.default_rng(deg).integers(0, 9, size=(L, S))
        t = _one(L, S, A, np.zeros((L, S)), np.zeros((L - 1, S, S)), cap=5, deg=deg, c=1)
        r = orc.solve_tables(t)
        assert r["stage_of"] == [0] * (L - deg + 1) + list(range(1, deg))
        assert r["objective"] == A.min(axis=1).sum()


def test_large_c_is_min_max_linear_partition(orc):
    """|S| = 1, R = O = 0: tpi = total + (c-1) * max stage, so OPT equals
    total + (c-1) * (textbook min-max linear partition, binary search + greedy)."""
    rng = np.random.default_rng(3)
    for trial in range(40):
        L = int(rng.integers(2, 20))
        deg = int(rng.integers(1, L + 1))
        c = int(rng.integers(2, 50))
        w = rng.integers(0, 1000, size=L)

        def feasible(x):
            parts, cur = 1, 0
            for v in w:
                if v > x:
                    return False
                if cur + v > x:
                    parts, cur = parts + 1, v
                else:
                    cur += v
            return parts <= deg
        lo, hi = 0, int(w.sum())
        while lo < hi:
            mid = (lo + hi) // 2
            if feasible(mid):
                hi = mid
            else:
                lo = mid + 1
        t = _one(L, 1, w.reshape(L, 1), np.zeros((L, 1)), np.zeros((L - 1, 1, 1)), cap=0, deg=deg, c=c)
        assert orc.solve_tables(t)["objective"] == w.sum() + (c - 1) * lo


def test_eq2_worked_example(orc):
    """Eq. (2): deg=2, c=4, p=(3,3), o=(1) -> 3+3+1+3*3 = 16;
    c = 1 -> sum p + sum o = 7."""
    for c, want in ((4, 16), (1, 7)):
        t = _one(2, 1, [[3], [3]], [[0], [0]], [[[0]]], cap=0, deg=2, c=c, O=[1])
        r = orc.solve_tables(t)
        assert r["objective"] == want and r["stage_cost"] == [3, 3] and r["cut_cost"] == [1]


def test_algorithm1_candidate_counts(orc):
    """Algorithm 1: 1 QIP + |F| x |B| MIQPs:
    n=8, B=32 -> 1 + 3*5; n=4, B=6 -> 1 + 2*3; the factor
    loops are O(sqrt(Bn)) (Sec. 3.5)."""
    assert len(orc.candidates(8, 32)) == 16
    assert len(orc.candidates(4, 6)) == 7
    assert orc.candidates(2, 2) == [(1, 1), (2, 2)]
    assert orc.candidates(1, 7) == [(1, 1)]
    assert orc.candidates(8, 32)[1:4] == [(2, 2), (2, 4), (2, 8)]


def test_strategy_catalogue(orc):
    """Reading A-6: all (t,f,d) with t*f*d = g, t a power of two, ordered
    (t asc, f asc); |S(2^k)| = C(k+2, 2); index 0 = pure DP (App. D)."""
    for k in range(6):
        cat = orc.catalogue(2 ** k)
        assert len(cat) == (k + 2) * (k + 1) // 2
        assert cat[0] == (1, 1, 2 ** k)
        assert all(t * f * d == 2 ** k for t, f, d in cat)
        assert cat == sorted(cat, key=lambda x: (x[0], x[1]))
    assert orc.catalogue(2) == [(1, 1, 2), (1, 2, 1), (2, 1, 1)]


def test_appendix_d_encoding(orc):
    """App. D: a 3-layer, 2-stage solution with P =
    [[1,0],[1,0],[0,1]]; our stage_of maps to that one-hot P."""
    A = [[1, 5], [1, 5], [1, 5]]
    t = _one(3, 2, A, np.zeros((3, 2)), np.zeros((2, 2, 2)), cap=0, deg=2, c=1)
    r = orc.solve_tables(t)
    P = np.eye(2, dtype=int)[r["stage_of"]]
    assert P.tolist() == [[1, 0], [1, 0], [0, 1]]
    S = np.eye(2, dtype=int)[r["strategy_of"]].T
    assert S[:, 0].tolist() == [1, 0]


def test_contiguity_definition_equals_intervals_on_chain_plus_skip():
    """Reading A-3: on chain (+ one skip source) graphs, Definition 1
     holds exactly for the intervals of the layer order."""
    for L in range(1, 8):
        for s in [-1] + list(range(max(L - 2, 0))):
            edges = [(u, u + 1) for u in range(L - 1)] + ([(s, v) for v in range(s + 2, L)] if s >= 0 else [])
            reach = np.eye(L, dtype=bool)
            for _ in range(L):
                for (u, v) in edges:
                    reach[:, v] |= reach[:, u]
            for mask in range(1, 2 ** L):
                W = [u for u in range(L) if mask >> u & 1]
                contiguous = not any(reach[u, v] and reach[v, w] for u in W for w in W
                                     for v in range(L) if v not in W)
                interval = W == list(range(W[0], W[-1] + 1))
                assert contiguous == interval


def test_invariants_on_random(orc):
    """Memory <= cap per stage, ordered non-empty stages, one strategy per
    layer, re-evaluated Eq. (2) == objective; more candidates never raise
    OPT; scaling every time entry by kappa scales OPT by kappa with the same
    argmin; OPT is non-increasing in cap."""
    for seed in range(120):
        t = tables.random_tables(seed)
        r = orc.solve_tables(t)
        if r["objective"] == INF:
            continue
        cfg = t["cfgs"][r["cfg_index"]]
        so, sk = r["stage_of"], r["strategy_of"]
        assert so[0] == 0 and so[-1] == r["deg"] - 1 and all(0 <= so[u + 1] - so[u] <= 1 for u in range(t["L"] - 1))
        assert all(0 <= k < cfg["n_strat"] for k in sk)
        assert all(m <= t["cap"] for m in r["stage_mem"])
        p, o = r["stage_cost"], r["cut_cost"]
        assert sum(p) + sum(o) + (r["c"] - 1) * max(p + o) == r["objective"]
        # more candidates never raise OPT
        sub = dict(t, cfgs=t["cfgs"][:1])
        assert orc.solve_tables(sub)["objective"] >= r["objective"]
        # kappa scaling
        kap = 3
        t3 = dict(t, cfgs=[dict(c, A=c["A"] * kap, R=c["R"] * kap,
                                Rskip=None if c["Rskip"] is None else c["Rskip"] * kap,
                                O=None if c["O"] is None else c["O"] * kap) for c in t["cfgs"]])
        r3 = orc.solve_tables(t3)
        assert r3["objective"] == kap * r["objective"]
        assert (r3["deg"], r3["c"], r3["stage_of"], r3["strategy_of"]) == (r["deg"], r["c"], so, sk)
        # cap monotonicity
        t2 = dict(t, cap=t["cap"] + 2)
        assert orc.solve_tables(t2)["objective"] <= r["objective"]


def test_infeasible_and_degenerate(orc):
    """deg > L is infeasible (A-22); deg = L gives one placement; every
    config infeasible -> INFEASIBLE status with per-config INT64_MAX."""
    L, S = 3, 2
    A = np.arange(6).reshape(3, 2)
    t = _one(L, S, A, np.zeros((L, S)), np.zeros((L - 1, S, S)), cap=0, deg=4)
    r = orc.solve_tables(t)
    assert r["status"] == 2 and r["objective"] == INF and r["cfg_objective"] == [INF]
    t = _one(L, S, A, np.zeros((L, S)), np.zeros((L - 1, S, S)), cap=0, deg=3, c=2)
    r = orc.solve_tables(t)
    assert r["stage_of"] == [0, 1, 2] and r["objective"] == 0 + 2 + 4 + 4
    t = _one(L, S, A, np.full((L, S), 5), np.zeros((L - 1, S, S)), cap=4)
    assert orc.solve_tables(t)["status"] == 2


def test_rejects_bad_tables(orc):
    t = tables.toy_tables()
    bad = dict(t, cfgs=[dict(t["cfgs"][0]), dict(t["cfgs"][0])])
    with pytest.raises(orc.OracleError):
        orc.solve_tables(bad)
    big = dict(t, cfgs=[dict(t["cfgs"][0], A=t["cfgs"][0]["A"] + (1 << 22))])
    with pytest.raises(orc.OracleError):
        orc.solve_tables(big)
