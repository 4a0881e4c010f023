"""Pins of the oracle on DAGs with several skip sources (NEXT-4, reading A-33;
CPU only).

Definition 1 on a DAG whose layers are given in
topological order with every chain edge u -> u+1: a set is contiguous iff it
is an interval of that order (checked here by brute force over every subset
of random such DAGs), so the ordered interval partitions stay exact.  Eq. 3
then charges every edge with both ends in a stage: a stage
conditions on the strategy of each skip source it holds together with an
edge of it.

Pins: brute force over every placement and strategy vector (every skip edge
evaluated literally) on tiny instances with 2-3 sources; one source given
through the multi-source tables = the single-source tables; all-zero skip
costs = no skip edges (every field); a source whose edges all leave the
stage costs nothing (the literal re-check)."""
import numpy as np
import pytest

from gen import tables
from oracle import brute

KEYS = ("objective", "cfg_index", "deg", "c", "stage_of", "strategy_of", "cfg_objective")


def test_contiguity_equals_intervals_on_random_chain_dags():
    rng = np.random.default_rng(33)
    for _ in range(300):
        L = int(rng.integers(2, 9))
        edges = [(u, u + 1) for u in range(L - 1)]
        edges += [(u, v) for u in range(L) for v in range(u + 2, L) if rng.random() < 0.3]
        reach = np.eye(L, dtype=bool)
        for _ in range(L):
            for (u, v) in edges:
                reach[:, v] |= reach[:, u]
        for mask in range(1, 2 ** L):
            W = [u for u in range(L) if mask >> u & 1]
            contiguous = not any(reach[u, v] and reach[v, w] for u in W for w in W for v in range(L) if v not in W)
            assert contiguous == (W == list(range(W[0], W[-1] + 1)))


@pytest.mark.parametrize("chunk", range(3))
def test_brute_force_several_skip_sources(orc, chunk):
    multi = 0
    for seed in range(chunk * 500, (chunk + 1) * 500):
        t = tables.with_skip_sources(tables.random_tables(110_000 + seed, skip_p=0.0), seed, 2 + seed % 2)
        multi += len(t["skip_srcs"]) >= 2
        want = brute.solve_tables(t)
        got = orc.solve_tables(t)
        for k in KEYS:
            if k in want:
                assert got[k] == want[k], (seed, k, got[k], want[k])
    assert multi >= 200


def test_one_source_through_the_multi_source_tables(orc):
    for seed in range(300):
        t = tables.random_tables(120_000 + seed, skip_p=1.0)
        if t["skip_src"] < 0:
            continue
        m = dict(t, skip_src=-1, skip_srcs=[t["skip_src"]],
                 cfgs=[dict(c, Rskip=None, Rskips=None if c["Rskip"] is None else c["Rskip"][None]) for c in t["cfgs"]])
        assert orc.solve_tables(m) == orc.solve_tables(t), seed


def test_zero_skip_costs_equal_no_skip_edges(orc):
    for seed in range(300):
        t = tables.with_skip_sources(tables.random_tables(130_000 + seed, skip_p=0.0), seed, 3, vmax=0)
        plain = dict(t, skip_srcs=[], cfgs=[dict(c, Rskips=None) for c in t["cfgs"]])
        assert orc.solve_tables(t) == orc.solve_tables(plain), seed


def test_bad_skip_sources_rejected(orc):
    t = tables.with_skip_sources(tables.random_tables(7, L=6, skip_p=0.0), 7, 2)
    for srcs in ([3, 1], [2, 2], [-1, 2], [0, 1, 2, 3, 4]):
        bad = dict(t, skip_srcs=srcs, cfgs=[dict(c, Rskips=np.zeros((len(srcs), 6, c["n_strat"], c["n_strat"]),
                                                                    np.int32)) for c in t["cfgs"]])
        with pytest.raises(orc.OracleError):
            orc.solve_tables(bad)
    both = dict(t, skip_src=1)
    with pytest.raises(orc.OracleError):
        orc.solve_tables(both)


def test_builder_several_sources_match_single_source_builds(orc):
    """Level 2 (builder'): with two skip sources, each source's table equals
    the Rskip table of the same profile keeping only that source's edges
    (the same formula per edge, PAPER.md:134 / reading A-15); the cut costs
    count every edge crossing the cut (reading A-16), so they equal the
    all-edges profile's."""
    from gen import profiles
    checked = 0
    for seed in range(40):
        p = profiles.random_profile(6000 + seed, L=6, Q=64, n_skip=2)
        p = dict(p, options=dict(p["options"], quantum_ns=1 << 10))  # one quantum for every variant
        t, _, _ = orc.build_tables(p)
        if "skip_srcs" not in t:
            continue
        for j, s in enumerate(t["skip_srcs"]):
            edges = [e for e in p["model"]["edges"] if e["dst"] == e["src"] + 1 or e["src"] == s]
            pj = dict(p, model=dict(p["model"], edges=edges))
            tj, _, _ = orc.build_tables(pj)
            assert tj["skip_src"] == s
            for c, cj in zip(t["cfgs"], tj["cfgs"]):
                assert np.array_equal(c["Rskips"][j], cj["Rskip"]), (seed, j)
                assert np.array_equal(c["A"], cj["A"]) and np.array_equal(c["M"], cj["M"])
        checked += 1
    assert checked >= 20


def test_builder_several_sources_brute_force(orc):
    from gen import profiles
    n = 0
    for seed in range(60):
        p = profiles.random_profile(5000 + seed, L=5, Q=16, n_skip=2 + seed % 2)
        t, _, _ = orc.build_tables(p)
        if max(c["n_strat"] for c in t["cfgs"]) ** t["L"] * 16 > 2_000_000:
            continue
        want, got = brute.solve_tables(t), orc.solve_tables(t)
        for k in KEYS:
            if k in want:
                assert got[k] == want[k], (seed, k)
        n += "skip_srcs" in t
    assert n >= 20


def test_brute_force_several_sources_with_1f1b(orc):
    """Several skip sources together with 1F1B's per-stage memory tables."""
    for seed in range(500):
        t = tables.with_skip_sources(tables.with_1f1b(tables.random_tables(140_000 + seed, skip_p=0.0), seed), seed, 2)
        want = brute.solve_tables(t)
        got = orc.solve_tables(t)
        for k in KEYS:
            if k in want:
                assert got[k] == want[k], (seed, k, got[k], want[k])
