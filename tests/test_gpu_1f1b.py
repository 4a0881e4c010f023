"""GPU parity of the 1F1B memory constraint (NEXT-2, reading A-32): stage i
of deg keeps min(c, deg - i) micro-batches in flight, so each stage reads its
own memory table (uniap_config.M_stage at level 1, uniap_options.schedule = 1
at level 2).  Bit-exact against the oracle: the whole result, the production
plan's interval tables per level (one per distinct (cap, table) pair), and the
builder's per-stage tables."""
import numpy as np
import pytest

from gen import profiles, tables

pytestmark = pytest.mark.gpu

KEYS = ("objective", "cfg_index", "deg", "c", "cfg_objective")
ASSIGN = ("stage_of", "strategy_of", "stage_cost", "cut_cost", "stage_mem")


@pytest.fixture(scope="module")
def h():
    import paper_2307_16375_b200 as pkg
    hd = pkg.Handle(0)
    yield hd
    hd.close()


def _same(g, o, what=""):
    for k in KEYS:
        assert g[k] == o[k], (what, k, g[k], o[k])
    if o["objective"] != (1 << 63) - 1:
        for k in ASSIGN:
            assert g[k] == o[k], (what, k, g[k], o[k])


@pytest.mark.parametrize("chunk", range(3))
def test_1f1b_tiny_brute_checked(h, orc, chunk):
    """The oracle is pinned to brute force on these instances (test_oracle_1f1b)."""
    for seed in range(chunk * 500, (chunk + 1) * 500):
        t = tables.with_1f1b(tables.random_tables(70_000 + seed), seed)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)


@pytest.mark.parametrize("seed", range(8))
def test_1f1b_large_tables_and_intervals(h, orc, seed):
    """Several configs, up to 6 stage tables each, ragged Q up to 4096, a skip
    source, per-stage caps on some: the solve and every level's interval
    table element by element."""
    from test_gpu_plan_parity import check
    rng = np.random.default_rng(300 + seed)
    L = int(rng.integers(6, 20))
    Q = int(rng.choice([64, 300, 1025, 4096]))
    cands = [(2, 4), (3, 2), (4, 8), (6, 6), (1, 3)]
    S = [int(rng.choice([2, 3, 6, 10])) for _ in cands]
    skip = int(rng.integers(0, L - 3)) if seed % 2 else -1
    t = tables.large_random_tables(500 + seed, L, S, Q - 1, cands, skip_src=skip, stage_caps=seed % 3 == 0,
                                   dist="ties" if seed % 4 == 1 else "uniform")
    t = tables.with_1f1b(t, seed, act_max=max(1, (Q - 1) // (3 * L)))
    got = h.solve_tables(t)
    check(h, orc, t, h.fetch_intervals(), ("1f1b", seed))
    _same(got, orc.solve_tables(t, n_threads=0), seed)


def test_1f1b_many_levels_k4_global_tables(h, orc):
    """L = 64, deg = 16 and 24 with c = 64: 16 / 24 levels, whose interval
    tables exceed K4's shared memory (read in place from global memory)."""
    from test_gpu_plan_parity import check
    cands = [(16, 64), (24, 64), (8, 2)]
    t = tables.large_random_tables(77, 64, [3, 2, 4], 255, cands, mem_max=12)
    t = tables.with_1f1b(t, 5, act_max=3)
    got = h.solve_tables(t)
    check(h, orc, t, h.fetch_intervals(), "many levels")
    _same(got, orc.solve_tables(t, n_threads=0), "many levels")


@pytest.mark.parametrize("name", ["llama", "t5", "bert"])
def test_1f1b_profiles_full_size(h, orc, name):
    """schedule = 1 on the BASELINE.json workloads: the builder's tables
    (with every stage's memory table) bit-equal to builder', and the plan
    equal to the oracle's, never worse than GPipe's."""
    p = profiles.make_profile(name)
    p1 = dict(p, options=dict(p["options"], schedule=1))
    t, qn, buf = orc.build_tables(p1)
    gt, gq, gbuf = h.build_tables(p1)
    assert gq == qn and np.array_equal(gbuf, buf), name
    want = orc.solve_tables(t, n_threads=0)
    got = h.plan(p1)
    _same(got, want, name)
    gpipe = h.plan(p)
    assert got["objective"] <= gpipe["objective"]
    assert all(a <= b for a, b in zip(got["cfg_objective"], gpipe["cfg_objective"]))


def test_1f1b_random_profiles(h, orc):
    for seed in range(12):
        p = profiles.random_profile(4000 + seed, Q=int(np.random.default_rng(seed).choice([16, 64, 256])))
        p = dict(p, options=dict(p["options"], schedule=1))
        t, qn, buf = orc.build_tables(p)
        gt, gq, gbuf = h.build_tables(p)
        assert gq == qn and np.array_equal(gbuf, buf), seed
        _same(h.plan(p), orc.solve_tables(t, n_threads=0), seed)


def test_1f1b_bad_tables_rejected(h):
    t = tables.with_1f1b(tables.random_tables(3), 3)
    bad = dict(t, cfgs=[dict(c, Rcut=np.zeros((max(t["L"] - 1, 1), c["n_strat"], c["n_strat"]), np.int32))
                        for c in t["cfgs"]])
    if t["L"] > 1:
        with pytest.raises(Exception):
            h.solve_tables(bad)
    neg = dict(t, cfgs=[dict(c, M_stage=-np.ones_like(c["M_stage"])) for c in t["cfgs"]])
    with pytest.raises(Exception):
        h.solve_tables(neg)
