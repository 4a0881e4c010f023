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


def covered(L, deg):
    """Intervals [a, b] a deg-stage ordered placement can use (SURVEY.md 8a,
    the solver's sweep plan): stage 1 a prefix, the last stage a suffix,
    middle stages inside."""
    m = np.zeros((L, L), dtype=bool)
    if deg > L:
        return m
    if deg == 1:
        m[0, L - 1] = True
        return m
    m[0, :L - deg + 1] = True                       # prefixes [0, b], b <= L - deg
    m[deg - 1:, L - 1] = True                       # suffixes [a, L-1], a >= deg - 1
    for a in range(1, L - 1) if deg >= 3 else ():   # middle stages i = 2..deg-1
        bmax = L - 1 - deg + min(a + 1, deg - 1)
        m[a, a:bmax + 1] = True
    return m


def check(h, orc, t, P, what):
    import concurrent.futures as cf
    L = t["L"]
    with cf.ThreadPoolExecutor() as ex:  # ctypes releases the GIL: one oracle call per config in parallel
        tabs = list(ex.map(lambda i: orc.interval_table(t, i), range(len(t["cfgs"]))))
    for i, cfg in enumerate(t["cfgs"]):
        want = np.where(tabs[i] == BIG, INF, tabs[i])
        m = covered(L, cfg["deg"])
        got = P[i].astype(np.int64)
        bad = np.argwhere(m & (got != want))
        assert bad.size == 0, (what, i, cfg["deg"], cfg["c"], bad[:5].tolist(),
                               [(int(got[a, b]), int(want[a, b])) for a, b in bad[:5]])
        # entries no placement needs may still be computed by a sweep (e.g. a
        # deg = 1 chain with the skip source inside runs as a forward sweep
        # and emits every prefix): each is either untouched or exact
        off = ~m & (got != INF)
        assert np.array_equal(got[off], want[off]), (what, i, "an extra entry is wrong")


@pytest.mark.parametrize("name", ["bert", "t5", "vit", "swin", "llama"])
def test_production_plan_intervals_full_size(h, orc, name):
    p = profiles.make_profile(name)
    t, qn, _ = orc.build_tables(p)
    h.plan(p)                                   # level 2: K1 + the production solve
    check(h, orc, t, h.fetch_intervals(t["L"]), name + " plan")
    h.solve_tables(t)                           # level 1: the same tables
    check(h, orc, t, h.fetch_intervals(t["L"]), name + " tables")


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
        check(h, orc, t, h.fetch_intervals(L), ("random", seed, L, Q, skip))
        _ = orc.solve_tables(t)


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
        check(h, orc, t, h.fetch_intervals(t["L"]), name)
