"""NEXT-1 on the GPU: the strategy-dependent cross-stage cost (Eq. 4 with R'
per strategy pair at each cut; uniap_config.Rcut) --
GPU = oracle, bit-exact, under the boundary-vector tie-break (reading A-31):
the brute-force-pinned tiny instances, larger random tables (skip edges,
ragged bucket counts, several kernel shapes) and a T5-shaped instance."""
import numpy as np
import pytest

from gen import profiles, tables

pytestmark = pytest.mark.gpu
BIG = (1 << 63) - 1
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
    if o["objective"] != BIG:
        for k in ASSIGN:
            assert g[k] == o[k], (what, k, g[k], o[k])


@pytest.mark.parametrize("chunk", range(2))
def test_cut_cost_tiny_brute_checked(h, orc, chunk):
    for seed in range(chunk * 1000, (chunk + 1) * 1000):
        t = tables.random_tables(900_000 + seed, rcut=True)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)


def test_cut_cost_larger_tables(h, orc):
    rng = np.random.default_rng(123)
    for seed in range(24):
        L = int(rng.integers(3, 14))
        Q = int(rng.choice([8, 33, 100, 256, 513, 1024]))
        cands = sorted({(int(d), int(c)) for d, c in zip(rng.integers(1, 6, 4), rng.integers(1, 5, 4))})
        S = [int(rng.choice([1, 2, 3, 5, 6, 8])) for _ in cands]
        skip = int(rng.integers(-1, L - 2))
        t = tables.large_random_tables(80_000 + seed, L, S, Q - 1, cands, skip_src=skip,
                                       mem_max=max(1, (3 * Q) // L), vmax=1 << 16)
        crng = np.random.default_rng(seed)
        for c in t["cfgs"]:
            s = c["n_strat"]
            c["Rcut"] = crng.integers(0, 1 << 16, size=(L - 1, s, s)).astype(np.int32)
        _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), ("large", seed, L, Q, S, skip))


def test_cut_cost_t5_shaped(h, orc):
    """The T5-Large-like profile's tables (48 layers, cross-attention skip
    edges 23 -> 25..47) at 256 buckets for the pipeline configs with 4 and 8
    stages, with a strategy-dependent cut cost: each cut costs its scalar
    O plus 0..1/4 of O by the pair of strategies meeting at the cut."""
    p = profiles.make_profile("t5")
    p["options"]["Q"] = 256
    p["options"]["cand"] = [(4, 2), (4, 4), (8, 2), (8, 8)]
    t, qn, _ = orc.build_tables(p)
    rng = np.random.default_rng(5)
    for c in t["cfgs"]:
        c.pop("stage_cap", None)  # (all at cap here; NEXT-1 is not combined with per-stage caps)
        s, O = c["n_strat"], np.asarray(c["O"], dtype=np.int64)
        c["Rcut"] = (rng.integers(0, 256, size=(t["L"] - 1, s, s)) * (O[:, None, None] // 1024 + 1)).astype(np.int32)
    _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), "t5 cut")


@pytest.mark.parametrize("space", [0, 1])
def test_cut_matrices_at_profile_level(h, orc, space):
    """uniap_edge.cut_ns_per_sample (R'_uv per sample on chain edges): K1's
    tables incl. Rcut bit-equal to builder''s, the plan equal to the oracle's."""
    import paper_2307_16375_b200 as pkg
    checked = 0
    for seed in range(30):
        n = [2, 4, 8][seed % 3]
        dim = sum(len(orc.catalogue(g, space)) for g in range(1, n + 1) if n % g == 0)
        p = profiles.random_profile(7000 + seed, n=n, Q=int([16, 64, 256][seed % 3]), mat_dim=dim, space=space)
        rng = np.random.default_rng(seed)
        for e in p["model"]["edges"]:
            if e["dst"] == e["src"] + 1 and rng.random() < 0.7:
                e["cut_ns_per_sample"] = rng.integers(0, 1 << 20, size=(dim, dim), dtype=np.int64)
        try:
            t, qn, buf = orc.build_tables(p)
        except orc.OracleError as e:
            with pytest.raises(pkg.UniapError) as ei:
                h.build_tables(p)
            assert ei.value.status == e.status
            continue
        gt, gq, gbuf = h.build_tables(p)
        assert gq == qn and np.array_equal(gbuf, buf), seed
        _same(h.plan(p), orc.solve_tables(t, n_threads=0), seed)
        checked += 1
    assert checked > 10
