"""Oracle vs brute force (tier T0) and the frozen toy golden (CPU only).

Pins the whole objective + argmin of the oracle (Eqs. 2-8, PAPER.md:122-202;
Algorithm 1; tie-break reading A-11) against the literal
enumeration of every stage-and-strategy assignment in oracle/brute.py.
"""
import json
import os

import numpy as np
import pytest

from gen import tables
from oracle import brute

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "toy.json")


def _same(r, b):
    assert r["objective"] == b["objective"]
    assert r["cfg_objective"] == b["cfg_objective"]
    if b["objective"] != brute.INT64_MAX:
        assert r["cfg_index"] == b["cfg_index"]
        assert (r["deg"], r["c"]) == (b["deg"], b["c"])
        assert r["stage_of"] == b["stage_of"]
        assert r["strategy_of"] == b["strategy_of"]


def test_toy_golden(orc):
    g = json.load(open(GOLDEN))
    t = tables.toy_tables()
    for i, want in enumerate(g["per_config"]):
        t1 = dict(t, cfgs=[t["cfgs"][i]])
        r = orc.solve_tables(t1)
        assert (r["objective"], r["stage_of"], r["strategy_of"]) == \
            (want["objective"], want["stage_of"], want["strategy_of"])
    r = orc.solve_tables(t)
    w = g["global"]["grid"]
    assert (r["objective"], r["deg"], r["c"]) == (w["objective"], w["deg"], w["c"]) == (16, 2, 1)
    r = orc.solve_tables(tables.toy_tables([(1, 1), (2, 2)]))
    w = g["global"]["algorithm1"]
    assert (r["objective"], r["deg"], r["c"]) == (w["objective"], w["deg"], w["c"]) == (20, 2, 2)


def test_toy_hand_check(orc):
    """(deg,c)=(1,1): strategies [2,2,0,0] -> A 5+4+5+6 + R 0+1+0 = 21, M 2+2+1+2 = 7 <= cap."""
    t = tables.toy_tables([(1, 1)])
    r = orc.solve_tables(t)
    A, R, M = t["cfgs"][0]["A"], t["cfgs"][0]["R"], t["cfgs"][0]["M"]
    k = r["strategy_of"]
    p = sum(int(A[u, k[u]]) for u in range(4)) + sum(int(R[u, k[u], k[u + 1]]) for u in range(3))
    assert p == 21 == r["objective"] == r["stage_cost"][0]
    assert sum(int(M[u, k[u]]) for u in range(4)) == r["stage_mem"][0] <= 7


@pytest.mark.parametrize("chunk", range(4))
def test_random_tiny_vs_brute(orc, chunk):
    """>= 2000 random tiny instances: L <= 6, |S| <= 3, cap <= 7, skip edges, O != 0,
    tie-heavy values and forbidden entries."""
    feasible = 0
    for seed in range(chunk * 600, (chunk + 1) * 600):
        t = tables.random_tables(seed)
        r, b = orc.solve_tables(t), brute.solve_tables(t)
        _same(r, b)
        feasible += b["objective"] != brute.INT64_MAX
    assert feasible > 400


def test_random_wider_vs_brute(orc):
    """Wider strategy sets and longer chains (|S| <= 4, L <= 7), tie-heavy."""
    for seed in range(300):
        rng = np.random.default_rng(10_000 + seed)
        L = int(rng.integers(4, 8))
        S = 4 if L <= 6 else 3
        t = tables.random_tables(10_000 + seed, L=L, S_max=S, cap=int(rng.integers(3, 12)),
                                 dist="ties" if seed % 2 else "uniform")
        _same(orc.solve_tables(t), brute.solve_tables(t))


def test_threads_do_not_change_result(orc):
    for seed in range(50):
        t = tables.random_tables(seed, n_cfg=4)
        assert orc.solve_tables(t, n_threads=1) == orc.solve_tables(t, n_threads=4)


# ---------------------------------------------------------------------------
# NEXT-2: per-stage memory limits m_i (heterogeneous devices, PAPER.md:161
# "the value of m varies in the case of heterogeneous computing devices";
# PAPER.md:603).  Eq. (5) per stage with its own cap.
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("chunk", range(3))
def test_oracle_equals_brute_force_with_stage_caps(orc, chunk):
    """The whole key against the literal enumeration with mem_i <= cap_i."""
    n = 0
    for seed in range(chunk * 500, (chunk + 1) * 500):
        t = tables.random_tables(700_000 + seed, stage_caps=True)
        _same(orc.solve_tables(t), brute.solve_tables(t))
        n += 1
    assert n == 500


def test_stage_caps_equal_to_cap_change_nothing_and_lower_caps_never_help(orc):
    for seed in range(300):
        t = tables.random_tables(800_000 + seed, stage_caps=True)
        base = dict(t, cfgs=[{k: v for k, v in c.items() if k != "stage_cap"} for c in t["cfgs"]])
        full = dict(t, cfgs=[dict(c, stage_cap=np.full(c["deg"], t["cap"], np.int32)) for c in base["cfgs"]])
        r0, r1, r2 = orc.solve_tables(base), orc.solve_tables(full), orc.solve_tables(t)
        assert r0 == r1
        for a, b in zip(r0["cfg_objective"], r2["cfg_objective"]):
            assert b >= a  # restricting a stage's memory can only raise the optimum


# ---------------------------------------------------------------------------
# NEXT-1: strategy-dependent cross-stage cost (Eq. 4, S_u^T R'_uv S_v for
# the chain edge at each cut); tie-break reading A-31.
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("chunk", range(4))
def test_oracle_equals_brute_force_with_strategy_dependent_cut_cost(orc, chunk):
    for seed in range(chunk * 500, (chunk + 1) * 500):
        t = tables.random_tables(900_000 + seed, rcut=True)
        _same(orc.solve_tables(t), brute.solve_tables(t))


def test_zero_cut_matrix_keeps_the_objective_and_costs_only_add(orc):
    """Rcut = 0 is Eq. 4 with a constant R' (the scalar path): same optimum;
    Rcut >= 0 only adds to the objective."""
    for seed in range(300):
        t = tables.random_tables(950_000 + seed, rcut=True)
        base = dict(t, cfgs=[{k: v for k, v in c.items() if k != "Rcut"} for c in t["cfgs"]])
        zero = dict(t, cfgs=[dict(c, Rcut=np.zeros_like(c["Rcut"])) for c in t["cfgs"]])
        r0, rz, r1 = orc.solve_tables(base), orc.solve_tables(zero), orc.solve_tables(t)
        assert r0["cfg_objective"] == rz["cfg_objective"]
        assert all(b >= a for a, b in zip(r0["cfg_objective"], r1["cfg_objective"]))
