"""Eq. 2 against an event simulation of the GPipe schedule
(reading A-20: the objective is the formula, a
lower bound of the flush schedule, equal when bp is proportional to fp).

The simulator (tests/gpipe_sim.py) replays forward and backward micro-batches
through the chain of stages and cut links; it shares nothing with the
oracle's evaluation of Eq. 2, so the last test pins the oracle's objective
(and its reported stage / cut costs) to the schedule the paper describes.
CPU only.
"""
import os
import random
import sys

import pytest

from gen import tables

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gpipe_sim as gs  # noqa: E402


def test_simulator_forward_only_is_flow_shop():
    """Zero backward times: the makespan is the textbook flow-shop makespan of
    identical jobs, sum t + (c-1) max t."""
    rng = random.Random(7)
    for _ in range(300):
        K, c = rng.randint(1, 7), rng.randint(1, 9)
        f = [rng.randint(0, 20) for _ in range(K)]
        T, log = gs.simulate(f, [0] * K, c)
        assert T == sum(f) + (c - 1) * max(f)
        assert gs.no_overlap(log)


def test_eq2_is_a_lower_bound_and_exact_when_bp_proportional_to_fp():
    rng = random.Random(11)
    for _ in range(500):
        deg, c = rng.randint(1, 6), rng.randint(1, 8)
        sf = [rng.randint(1, 30) for _ in range(deg)]
        lf = [rng.randint(0, 30) for _ in range(deg - 1)]
        # arbitrary backward times: Eq. 2 (with p = fwd + bwd) never exceeds the schedule
        sb = [rng.randint(0, 60) for _ in range(deg)]
        lb = [rng.randint(0, 60) for _ in range(deg - 1)]
        f, b = gs.servers(sf, sb, lf, lb)
        T, log = gs.simulate(f, b, c)
        assert gs.no_overlap(log)
        p = [x + y for x, y in zip(sf, sb)]
        o = [x + y for x, y in zip(lf, lb)]
        assert T >= gs.eq2(p, o, c)
        # bp = kappa * fp on every stage and link (bp = 2 fp): equality
        kappa = rng.randint(1, 3)
        f, b = gs.servers(sf, [kappa * x for x in sf], lf, [kappa * x for x in lf])
        T, _ = gs.simulate(f, b, c)
        assert T == gs.eq2([(1 + kappa) * x for x in sf], [(1 + kappa) * x for x in lf], c)


def test_eq2_worked_example_against_simulation():
    """deg 2, c 4, p = (3, 3), o = (1) -> 16; as a schedule
    with fp = 1, bp = 2 per stage and a 1-unit link split 0 / 1."""
    f, b = gs.servers([1, 1], [2, 2], [0], [1])
    T, _ = gs.simulate(f, b, 4)
    assert T == 16 == gs.eq2([3, 3], [1], 4)


@pytest.mark.parametrize("seed0", [0, 400])
def test_oracle_objective_is_the_gpipe_makespan(orc, seed0):
    """The oracle's optimum, replayed as a GPipe schedule with fp = p, bp = 2p
    per stage and fo = o, bo = 2o per cut (so every server's per-micro-batch
    time is 3x its Eq. 3 / Eq. 4 cost), takes exactly 3 x the objective."""
    checked = 0
    for seed in range(seed0, seed0 + 400):
        t = tables.random_tables(seed)
        r = orc.solve_tables(t)
        if r["objective"] == (1 << 63) - 1:
            continue
        p, o, c = r["stage_cost"], r["cut_cost"], r["c"]
        f, b = gs.servers(p, [2 * x for x in p], o, [2 * x for x in o])
        T, log = gs.simulate(f, b, c)
        assert gs.no_overlap(log)
        assert T == 3 * r["objective"], (seed, p, o, c, r["objective"])
        checked += 1
    assert checked > 100


def test_toy_winner_as_a_schedule(orc):
    r = orc.solve_tables(tables.toy_tables())
    f, b = gs.servers(r["stage_cost"], [2 * x for x in r["stage_cost"]], r["cut_cost"],
                      [2 * x for x in r["cut_cost"]])
    T, _ = gs.simulate(f, b, r["c"])
    assert T == 3 * r["objective"] == 3 * 16
