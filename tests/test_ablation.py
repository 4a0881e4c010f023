"""Strategy-space ablation (
reading A-25): every restricted space is a subset of the unified one, so its
optimum can only be worse, and each variant's plan obeys its restriction.
Oracle on CPU; the GPU solves the same restricted tables bit-exactly
(tests marked gpu)."""
import pytest

from gen import ablation, profiles, tables

INT64_MAX = (1 << 63) - 1


def _check_variant(r, variant, n_dev):
    if r["objective"] == INT64_MAX:
        return
    if variant == "intra-only":
        assert r["deg"] == 1
    if variant == "inter-pp":
        assert r["deg"] == n_dev
    if variant == "inter-dp":
        assert all(k == 0 for k in r["strategy_of"])


def _solve(orc, t):
    if not t["cfgs"]:
        return {"objective": INT64_MAX}
    return orc.solve_tables(t, n_threads=0)


@pytest.mark.parametrize("seed", range(12))
def test_restricted_spaces_never_beat_unified(orc, seed):
    p = profiles.random_profile(seed)
    try:
        t, _, _ = orc.build_tables(p)
    except orc.OracleError:
        pytest.skip("profile out of range for the builder")
    n = p["cluster"]["n_dev"]
    best = _solve(orc, t)["objective"]
    for v in ablation.VARIANTS[1:]:
        r = _solve(orc, ablation.restrict(t, v, n))
        assert r["objective"] >= best, (seed, v)
        _check_variant(r, v, n)


def test_unified_equals_best_variant_when_a_variant_covers_the_optimum(orc):
    """The toy grid: the unified winner (deg 2, strategies [1,1,1,1]) is not
    pure DP, so inter-dp is strictly worse; intra-only is the deg = 1 optimum."""
    t = tables.toy_tables()
    uni = orc.solve_tables(t)
    intra = orc.solve_tables(ablation.restrict(t, "intra-only", 2))
    interdp = orc.solve_tables(ablation.restrict(t, "inter-dp", 2))
    assert uni["objective"] == 16
    assert intra["objective"] == min(21, 32) and intra["deg"] == 1
    assert interdp["objective"] > uni["objective"]
    assert all(k == 0 for k in interdp["strategy_of"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["t5", "vit"])
def test_ablation_gpu_matches_oracle(orc, name):
    import paper_2307_16375_b200 as pkg
    h = pkg.Handle(0)
    p = profiles.make_profile(name)
    t, _, _ = orc.build_tables(p)
    n = p["cluster"]["n_dev"]
    for v in ablation.VARIANTS:
        tv = ablation.restrict(t, v, n)
        if not tv["cfgs"]:
            continue
        want = orc.solve_tables(tv, n_threads=0)
        got = h.solve_tables(tv)
        for k in ("objective", "deg", "c", "cfg_objective"):
            assert got[k] == want[k], (name, v, k)
        if want["objective"] != INT64_MAX:
            assert got["stage_of"] == want["stage_of"] and got["strategy_of"] == want["strategy_of"], (name, v)
            _check_variant(got, v, n)
    h.close()
