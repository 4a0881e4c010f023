"""GPU parity on DAGs with several skip sources (NEXT-4, reading A-33):
layers in topological order with every chain edge plus edges from up to four
sources to later layers; a stage conditions on each source it holds with an
edge.  The library runs every conditioning copy as a plain chain sweep over
its own A' / M' tables (uniap_tables.skip_srcs, uniap_config.Rskips).
Bit-exact against the oracle (itself pinned by brute force in
test_oracle_dag.py): the whole result, the production plan's interval tables,
tracebacks over more copies than a CTA has warps."""
import numpy as np
import pytest

from gen import tables

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
def test_dag_tiny_brute_checked(h, orc, chunk):
    for seed in range(chunk * 500, (chunk + 1) * 500):
        t = tables.with_skip_sources(tables.random_tables(110_000 + seed, skip_p=0.0), seed, 2 + seed % 2)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)


@pytest.mark.parametrize("seed", range(8))
def test_dag_large_tables_and_intervals(h, orc, seed):
    """2-4 sources, |S| up to 6, ragged Q up to 4096 (cluster sweeps too),
    per-stage caps on some: the solve and every interval table entry the
    production plan emits."""
    from test_gpu_plan_parity import check
    rng = np.random.default_rng(700 + seed)
    L = int(rng.integers(8, 22))
    Q = int(rng.choice([64, 300, 1025, 2048, 4096]))
    cands = [(1, 2), (2, 4), (3, 2), (4, 8), (5, 3)]
    S = [int(rng.choice([2, 3, 4, 6])) for _ in cands]
    t = tables.large_random_tables(800 + seed, L, S, Q - 1, cands, stage_caps=seed % 3 == 0,
                                   dist="ties" if seed % 4 == 1 else "uniform")
    t = tables.with_skip_sources(t, seed, 2 + seed % 3, vmax=1 << 19)
    got = h.solve_tables(t)
    check(h, orc, t, h.fetch_intervals(), ("dag", seed))
    _same(got, orc.solve_tables(t, n_threads=0), seed)


@pytest.mark.parametrize("S,n_src", [(6, 3), (5, 4), (32, 2)])
def test_dag_deg1_traceback_over_many_copies(h, orc, S, n_src):
    """deg = 1 winners holding every source: up to 6^3 = 216 / 5^4 = 625 /
    32^2 = 1024 copies in the traceback (more than a CTA's 32 warps)."""
    L = 12 if S < 32 else 6
    t = tables.large_random_tables(S * 10 + n_src, L, [S, S], 255, [(1, 1), (1, 3)], mem_max=20)
    t = tables.with_skip_sources(t, S, n_src, vmax=1 << 19)
    assert len(t["skip_srcs"]) == n_src
    _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), (S, n_src))


def test_one_source_list_equals_single_source_tables(h, orc):
    for seed in range(200):
        t = tables.random_tables(120_000 + seed, skip_p=1.0)
        if t["skip_src"] < 0:
            continue
        m = dict(t, skip_src=-1, skip_srcs=[t["skip_src"]],
                 cfgs=[dict(c, Rskip=None, Rskips=None if c["Rskip"] is None else c["Rskip"][None]) for c in t["cfgs"]])
        _same(h.solve_tables(m), h.solve_tables(t), seed)


def test_dag_limits_rejected(h):
    t = tables.with_skip_sources(tables.random_tables(9, L=7, S_max=3, skip_p=0.0), 9, 2)
    bad = dict(t, skip_srcs=list(reversed(t["skip_srcs"])))
    with pytest.raises(Exception):
        h.solve_tables(bad)
    with pytest.raises(Exception):
        h.solve_tables(dict(t, skip_src=1))
    # |S| = 32 with 3 sources: 32^3 copies exceed UNIAP_MAX_COPIES
    big = tables.large_random_tables(3, 10, [32], 63, [(2, 2)], mem_max=4)
    big = tables.with_skip_sources(big, 3, 3, vmax=100)
    with pytest.raises(Exception):
        h.solve_tables(big)


def test_dag_profiles_builder_and_plan(h, orc):
    """Level 2: random profiles with 2-4 skip sources -- K1's per-source skip
    tables and K1g's conditioning copies: builder tables bit-equal to
    builder', plan = the oracle's."""
    from gen import profiles
    n = 0
    for seed in range(30):
        rng = np.random.default_rng(seed)
        p = profiles.random_profile(7000 + seed, L=int(rng.integers(5, 12)), Q=int(rng.choice([16, 64, 256])),
                                    n_skip=2 + seed % 3)
        try:
            t, qn, buf = orc.build_tables(p)
        except orc.OracleError:
            with pytest.raises(Exception):
                h.build_tables(p)
            continue
        ns = len(t.get("skip_srcs") or [])
        copies = max(sum(c["n_strat"] ** (j1 - j0 + 1) for j0 in range(ns) for j1 in range(j0, ns))
                     for c in t["cfgs"]) if ns >= 2 else 0
        if copies > 4096:  # beyond UNIAP_MAX_COPIES: the library refuses (documented limit)
            with pytest.raises(Exception, match="skip-conditioning copies"):
                h.build_tables(p)
            continue
        gt, gq, gbuf = h.build_tables(p)
        assert gq == qn and np.array_equal(gbuf, buf), seed
        _same(h.plan(p), orc.solve_tables(t, n_threads=0), seed)
        n += ns >= 2
    assert n >= 12


def test_t5_with_a_second_source_profile(h, orc):
    """The T5-like profile plus edges from a second source (an extra encoder
    tap 11 -> 13..23): two skip sources at full size."""
    from gen import profiles
    p = profiles.make_profile("t5")
    edges = list(p["model"]["edges"]) + [{"src": 11, "dst": v, "tensor_bytes_per_sample": 512 * 1024 * 4}
                                         for v in range(13, 24)]
    p = dict(p, model=dict(p["model"], edges=edges))
    t, qn, buf = orc.build_tables(p)
    assert t.get("skip_srcs") == [11, 23]
    gt, gq, gbuf = h.build_tables(p)
    assert gq == qn and np.array_equal(gbuf, buf)
    _same(h.plan(p), orc.solve_tables(t, n_threads=0), "t5 two sources")


def test_dag_profile_unsupported_combinations_rejected(h):
    """Several skip sources with cut matrices are refused (UNIAP_ERR_ARG),
    not solved wrongly."""
    from gen import profiles
    p = None
    for seed in range(40):
        q = profiles.random_profile(7100 + seed, L=8, Q=64, n_skip=2)
        if len({e["src"] for e in q["model"]["edges"] if e["dst"] != e["src"] + 1}) >= 2:
            p = q
            break
    assert p is not None
    import paper_2307_16375_b200 as pkg
    ncat = sum(len(pkg.catalogue(g)) for g in range(1, p["cluster"]["n_dev"] + 1) if p["cluster"]["n_dev"] % g == 0)
    edges = [dict(e, cut_ns_per_sample=np.zeros((ncat, ncat), np.int64)) if e["dst"] == e["src"] + 1 else e
             for e in p["model"]["edges"]]
    with pytest.raises(Exception, match="cut matrices"):
        h.plan(dict(p, model=dict(p["model"], edges=edges)))


def test_dag_with_1f1b_tables_and_profiles(h, orc):
    """Several skip sources with 1F1B's per-stage memory tables: each copy
    keeps one M' per memory table (level 1: brute-pinned tiny instances and
    larger tables with the interval tables; level 2: schedule = 1 profiles)."""
    from test_gpu_plan_parity import check
    from gen import profiles
    for seed in range(500):
        t = tables.with_skip_sources(tables.with_1f1b(tables.random_tables(140_000 + seed, skip_p=0.0), seed), seed, 2)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)
    for seed in range(4):
        t = tables.large_random_tables(900 + seed, 14, [3, 4, 6], 1023, [(4, 8), (3, 2), (6, 12)], mem_max=60)
        t = tables.with_skip_sources(tables.with_1f1b(t, seed, act_max=8), seed, 2 + seed % 2, vmax=1 << 18)
        got = h.solve_tables(t)
        check(h, orc, t, h.fetch_intervals(), ("dag 1f1b", seed))
        _same(got, orc.solve_tables(t, n_threads=0), seed)
    n = 0
    for seed in range(20):
        p = profiles.random_profile(7200 + seed, L=7, Q=64, n_skip=2)
        p = dict(p, options=dict(p["options"], schedule=1))
        t, qn, buf = orc.build_tables(p)
        ns = len(t.get("skip_srcs") or [])
        if ns < 2 or max(sum(c["n_strat"] ** (j1 - j0 + 1) for j0 in range(ns) for j1 in range(j0, ns))
                         for c in t["cfgs"]) > 4096:
            continue
        gt, gq, gbuf = h.build_tables(p)
        assert gq == qn and np.array_equal(gbuf, buf), seed
        _same(h.plan(p), orc.solve_tables(t, n_threads=0), seed)
        n += 1
    assert n >= 8
