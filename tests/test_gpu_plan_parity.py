"""GPU parity of the plan that actually runs, element by element.

uniap_interval_table checks the canonical all-intervals forward plan; the
solver runs a different one (prefix sweeps from layer 0, ONE backward
suffix sweep per config, middle sweeps only for deg >= 3, skip-conditioned
copies split at the skip source, the deg = 1 chain as a G-keeping backward
sweep, every P sweep trimmed on the device at its feasible prefix).  Here the
interval optima the solver's own run left in its P arena
(uniap_fetch_intervals) are compared with the oracle's interval table on
every entry some placement of the config can use -- and every other entry
must be untouched (UNIAP_INF) or exact as well.  An over-estimated P entry off the optimal
path cannot hide: it is compared directly.
"""
import numpy as np
import pytest

from gen import profiles, tables

pytestmark = pytest.mark.gpu
INF = 0x40000000
BIG = (1 << 63) - 1


@pytest.fixture(scope="module")
def h():
    import paper_2307_16375_b200 as pkg
    hd = pkg.Handle(0)
    yield hd
    hd.close()


def stage_intervals(L, deg, i):
    """Intervals [a, b] stage i (0-based) of a deg-stage ordered placement can
    be: i layers before it, deg-1-i after it."""
    m = np.zeros((L, L), dtype=bool)
    if deg > L:
        return m
    for a in range(i, L):
        for b in range(a, L - (deg - 1 - i)):
            if (i == 0 and a != 0) or (i == deg - 1 and b != L - 1):
                continue
            m[a, b] = True
    return m


def levels(t, cfg):
    """The config's distinct (stage cap, stage memory table) pairs in order of
    first appearance (the library's levels: per-stage caps, NEXT-2, and the
    per-stage tables of 1F1B, reading A-32) as (cap, M) and each stage's
    level."""
    deg = cfg["deg"]
    caps = [t["cap"]] * deg if cfg.get("stage_cap") is None else [int(x) for x in cfg["stage_cap"]]
    MS = cfg.get("M_stage")
    tabs = [np.asarray(cfg["M"]) if MS is None else np.asarray(MS[i]) for i in range(min(deg, t["L"]))]
    tabs += [tabs[0] if tabs else None] * (deg - len(tabs))
    lv, of = [], []
    for c, m in zip(caps, tabs):
        j = next((i for i, (c2, m2) in enumerate(lv) if c2 == c and np.array_equal(m2, m)), None)
        if j is None:
            lv.append((c, m))
            j = len(lv) - 1
        of.append(j)
    return lv, of


def check(h, orc, t, P, what):
    """P: the flat fetch_intervals array (per config, one L*L block per cap level)."""
    import concurrent.futures as cf
    L = t["L"]
    jobs, off = [], 0
    for i, cfg in enumerate(t["cfgs"]):
        lv_list, lev_of = levels(t, cfg)
        for lv, (cap, m) in enumerate(lv_list):
            jobs.append((i, lv, cap, off, m))
            off += L * L
    assert off == P.size, (what, off, P.size)

    def table(j):  # the level's interval table: the config with that cap and memory table
        i, _, cap, _, m = j
        cfgs = [{k: v for k, v in c.items() if k not in ("stage_cap", "M_stage")} for c in t["cfgs"]]
        cfgs[i]["M"] = m
        return orc.interval_table(dict(t, cap=cap, cfgs=cfgs), i)

    with cf.ThreadPoolExecutor() as ex:  # ctypes releases the GIL: one oracle call per table in parallel
        tabs = list(ex.map(table, jobs))
    for (i, lv, cap, o, _), want in zip(jobs, tabs):
        cfg = t["cfgs"][i]
        want = np.where(want == BIG, INF, want)
        _, lev_of = levels(t, cfg)
        m = np.zeros((L, L), dtype=bool)
        for st, l in enumerate(lev_of if cfg["deg"] <= L else []):
            if l == lv:
                m |= stage_intervals(L, cfg["deg"], st)
        got = P[o:o + L * L].reshape(L, L).astype(np.int64)
        bad = np.argwhere(m & (got != want))
        assert bad.size == 0, (what, i, lv, cfg["deg"], cfg["c"], bad[:5].tolist(),
                               [(int(got[a, b]), int(want[a, b])) for a, b in bad[:5]])
        # entries no placement needs may still be computed by a sweep (e.g. a
        # deg = 1 chain with the skip source inside runs as a forward sweep
        # and emits every prefix): each is either untouched or exact
        extra = ~m & (got != INF)
        assert np.array_equal(got[extra], want[extra]), (what, i, lv, "an extra entry is wrong")


@pytest.mark.parametrize("name", ["bert", "t5", "vit", "swin", "llama"])
def test_production_plan_intervals_full_size(h, orc, name):
    p = profiles.make_profile(name)
    t, qn, _ = orc.build_tables(p)
    h.plan(p)                                   # level 2: K1 + the production solve
    check(h, orc, t, h.fetch_intervals(), name + " plan")
    h.solve_tables(t)                           # level 1: the same tables
    check(h, orc, t, h.fetch_intervals(), name + " tables")


def test_production_plan_intervals_random_skip_tables(h, orc):
    """Random tables with a skip source at every position, every deg up to L,
    memory binding (the device trim acts), |S| across the kernel classes."""
    rng = np.random.default_rng(31)
    for seed in range(24):
        L = int(rng.integers(3, 16))
        Q = int(rng.choice([7, 64, 300, 1025, 4096]))
        cands = sorted({(int(d), int(c)) for d, c in zip(rng.integers(1, L + 2, 4), rng.integers(1, 5, 4))})
        S = [int(rng.choice([1, 2, 3, 6, 10, 15, 21])) for _ in cands]
        skip = int(rng.integers(-1, L - 2))
        t = tables.large_random_tables(40_000 + seed, L, S, Q - 1, cands, skip_src=skip,
                                       mem_max=max(1, (4 * Q) // L))
        h.solve_tables(t)
        check(h, orc, t, h.fetch_intervals(), ("random", seed, L, Q, skip))


def test_level2_swin50_llama_envc_llama13b(h, orc):
    """The profiles gen/ defines beyond the five bench workloads, solved on the GPU."""
    for name in ("swin50", "llama-envc", "llama13b"):
        p = profiles.make_profile(name)
        want, t = orc.plan(p, n_threads=0)
        got = h.plan(p)
        for k in ("objective", "deg", "c", "cfg_objective", "quantum_ns"):
            assert got[k] == want[k], (name, k)
        if want["objective"] != BIG:
            for k in ("stage_of", "strategy_of", "stage_cost", "cut_cost", "stage_mem"):
                assert got[k] == want[k], (name, k)
        check(h, orc, t, h.fetch_intervals(), name)


# ---------------------------------------------------------------------------
# NEXT-2: per-stage memory limits (heterogeneous devices)
# ---------------------------------------------------------------------------

KEYS = ("objective", "cfg_index", "deg", "c", "cfg_objective")
ASSIGN = ("stage_of", "strategy_of", "stage_cost", "cut_cost", "stage_mem")


def _same(g, o, what=""):
    for k in KEYS:
        assert g[k] == o[k], (what, k, g[k], o[k])
    if o["objective"] != BIG:
        for k in ASSIGN:
            assert g[k] == o[k], (what, k, g[k], o[k])


def test_stage_caps_tiny_brute_checked(h, orc):
    """The brute-force-pinned tiny instances with per-stage caps, GPU = oracle."""
    for seed in range(1500):
        t = tables.random_tables(700_000 + seed, stage_caps=True)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)


def test_stage_caps_large_tables_and_intervals(h, orc):
    rng = np.random.default_rng(77)
    for seed in range(16):
        L = int(rng.integers(4, 20))
        Q = int(rng.choice([64, 300, 1025, 4096]))
        cands = sorted({(int(d), int(c)) for d, c in zip(rng.integers(1, 9, 4), rng.integers(1, 5, 4))})
        S = [int(rng.choice([1, 3, 6, 10, 15])) for _ in cands]
        skip = int(rng.integers(-1, L - 2))
        t = tables.large_random_tables(60_000 + seed, L, S, Q - 1, cands, skip_src=skip,
                                       mem_max=max(1, (3 * Q) // L), stage_caps=True)
        _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), ("large", seed))
        check(h, orc, t, h.fetch_intervals(), ("large", seed))


@pytest.mark.parametrize("name", ["llama", "t5"])
def test_heterogeneous_device_memory_profiles(h, orc, name):
    """Level 2 with per-device memory: half of the devices with 60 % of the
    memory (alternating blocks of 4), K1 tables incl. stage caps bit-equal,
    plan = oracle plan, interval tables element by element."""
    p = profiles.make_profile(name)
    cl = p["cluster"]
    n = cl["n_dev"]
    small = cl["mem_reserve_bytes"] + (cl["mem_bytes"] - cl["mem_reserve_bytes"]) * 6 // 10
    cl["dev_mem_bytes"] = [small if (d // 4) % 2 else cl["mem_bytes"] for d in range(n)]
    t, qn, buf = orc.build_tables(p)
    gt, gq, gbuf = h.build_tables(p)
    assert gq == qn and np.array_equal(gbuf, buf)
    want = orc.solve_tables(t, n_threads=0)
    _same(h.plan(p), want, name)
    check(h, orc, t, h.fetch_intervals(), name + " hetero")
