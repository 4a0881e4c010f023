"""Pins of the 1F1B memory constraint (NEXT-2, reading A-32; CPU only).

The footnote of PAPER.md:122: "users need to modify only the memory
constraint in Section 3.3.2 to adapt to synchronous 1F1B pipeline".  Stage i
(0-based) of deg then keeps the activations of min(c, deg - i) micro-batches
in flight instead of GPipe's c, so Eq. (5) uses a per-stage memory table
M_stage[i]; the time model (Eq. 2) is unchanged.

Pins: brute force over every placement and strategy vector (the literal
Eqs. 2, 3, 5 with the stage's own table) on tiny random instances; the
special cases that reduce to GPipe (identical stage tables; c = 1; deg = 1);
1F1B never worse than GPipe (its memory is never larger, so the feasible set
only grows); and builder' integers worked out by hand for a two-stage
profile."""
import numpy as np
import pytest

from gen import profiles, tables
from oracle import brute

INT64_MAX = (1 << 63) - 1
KEYS = ("objective", "cfg_index", "deg", "c", "stage_of", "strategy_of", "cfg_objective")


def _gpipe(t):
    return dict(t, cfgs=[{k: v for k, v in c.items() if k != "M_stage"} for c in t["cfgs"]])


@pytest.mark.parametrize("chunk", range(3))
def test_brute_force_1f1b(orc, chunk):
    """The oracle's whole key equals brute force on 500 instances per chunk."""
    differ = 0
    for seed in range(chunk * 500, (chunk + 1) * 500):
        t = tables.with_1f1b(tables.random_tables(70_000 + seed), seed)
        want = brute.solve_tables(t)
        got = orc.solve_tables(t)
        for k in KEYS:
            if k in want:
                assert got[k] == want[k], (seed, k, got[k], want[k])
        differ += got["objective"] != orc.solve_tables(_gpipe(t))["objective"]
    assert differ >= 20  # the stage tables matter in a fair share of the instances


def test_identical_stage_tables_reduce_to_gpipe(orc):
    """M_stage[i] = M for every stage: exactly the GPipe answer (all fields)."""
    for seed in range(300):
        t = tables.random_tables(80_000 + seed)
        same = dict(t, cfgs=[dict(c, M_stage=np.stack([c["M"]] * c["deg"])) for c in t["cfgs"]])
        a, b = orc.solve_tables(same), orc.solve_tables(t)
        assert a == b, seed


def test_1f1b_never_worse_than_gpipe(orc):
    """n_i = min(c, deg - i) <= c: every config's optimum is <= GPipe's."""
    for seed in range(300):
        t = tables.with_1f1b(tables.random_tables(90_000 + seed), seed, act_max=3)
        a, b = orc.solve_tables(t), orc.solve_tables(_gpipe(t))
        assert all(x <= y for x, y in zip(a["cfg_objective"], b["cfg_objective"])), seed


def _two_stage_profile(schedule):
    """n = 2 devices, one layer kind x 2 layers, fp32, B = 8; candidates
    (deg, c) = (2, 4), (2, 1), (1, 4); memory unit 1 byte (Q - 1 = mem)."""
    layer = {"fwd_ns_per_sample": [1_000, 600], "param_bytes": 1_000, "act_bytes_per_sample": [300, 170],
             "ctx_bytes": 10, "tp_comm_bytes_per_sample": 0}
    return {"name": "1f1b", "model": {"L": 2, "layers": [dict(layer), dict(layer)],
                                      "edges": [{"src": 0, "dst": 1, "tensor_bytes_per_sample": 64}]},
            "cluster": dict(n_dev=2, node_size=2, mem_bytes=8191, mem_reserve_bytes=0, bw_intra_Bps=10 ** 9,
                            bw_inter_Bps=10 ** 9, p2p_Bps=10 ** 9, lat_ns=0, ccoc_permille=0),
            "options": dict(B=8, precision=0, Q=8192, quantum_ns=0, cand=[(2, 4), (2, 1), (1, 4)],
                            schedule=schedule)}


def test_builder_1f1b_memory_by_hand(orc):
    """Eq. (1) + activations + context with n micro-batches in flight
    (footnote of PAPER.md:122), unit = 1 byte:
      deg = 2, c = 4, b = B / c = 2, one device per stage (g = 1, strategy
      (1, 1, 1), micro-batch per device 2):
        GPipe  M = 4 * 1000 + 4 * 2 * 300 + 10 = 6410
        stage 0: n = min(4, 2) = 2 -> 4000 + 2 * 2 * 300 + 10 = 5210
        stage 1: n = min(4, 1) = 1 -> 4000 + 1 * 2 * 300 + 10 = 4610
      deg = 2, c = 1, b = 8: n = min(1, .) = 1 = c -> both stages = GPipe
        = 4000 + 8 * 300 + 10 = 6410
      deg = 1, c = 4, b = 2, g = 2: strategy (1, 1, 2) (DP): micro-batch per
        device 1; GPipe 4000 + 4 * 1 * 300 + 10 = 5210, 1F1B n = min(4, 1) = 1
        -> 4000 + 300 + 10 = 4310; strategy (2, 1, 1) (TP 2): params / 2,
        activation per sample 170, micro-batch 2: GPipe 2000 + 4 * 2 * 170 + 10
        = 3370, 1F1B 2000 + 2 * 170 + 10 = 2350."""
    t, _, _ = orc.build_tables(_two_stage_profile(1))
    g = {(c["deg"], c["c"]): c for c in t["cfgs"]}
    c24 = g[(2, 4)]
    assert c24["M"][0, 0] == 6410 and c24["M"][1, 0] == 6410
    assert list(c24["M_stage"][:, 0, 0]) == [5210, 4610] and list(c24["M_stage"][:, 1, 0]) == [5210, 4610]
    c21 = g[(2, 1)]
    assert list(c21["M_stage"][:, 0, 0]) == [6410, 6410] and c21["M"][0, 0] == 6410
    c14 = g[(1, 4)]
    kdp = orc.catalogue(2).index((1, 1, 2))
    ktp = orc.catalogue(2).index((2, 1, 1))
    assert c14["M"][0, kdp] == 5210 and c14["M_stage"][0, 0, kdp] == 4310
    assert c14["M"][0, ktp] == 3370 and c14["M_stage"][0, 0, ktp] == 2350
    # GPipe schedule: no stage tables in the block
    t0, _, _ = orc.build_tables(_two_stage_profile(0))
    assert all(c["M_stage"] is None for c in t0["cfgs"])
    assert all(np.array_equal(a["M"], b["M"]) for a, b in zip(t0["cfgs"], t["cfgs"]))


@pytest.mark.parametrize("name", ["toy", "random"])
def test_builder_1f1b_stage_tables_properties(orc, name):
    """On built tables: stage tables non-increasing in the stage index; stage
    0 equals GPipe's M when c <= deg (n_0 = min(c, deg) = c); every stage
    equals M when c = 1; and the solve equals brute force."""
    ps = [profiles.toy_profile()] if name == "toy" else [profiles.random_profile(s, L=4, Q=64) for s in range(6)]
    for p in ps:
        p = dict(p, options=dict(p["options"], schedule=1))
        t, _, _ = orc.build_tables(p)
        for c in t["cfgs"]:
            MS, M = c["M_stage"], c["M"]
            assert MS.shape == (c["deg"],) + M.shape
            assert np.all(MS[1:] <= MS[:-1])
            if c["c"] <= c["deg"]:
                assert np.array_equal(MS[0], M)
            if c["c"] == 1:
                assert all(np.array_equal(m, M) for m in MS)
        if max(c["n_strat"] for c in t["cfgs"]) ** t["L"] * 16 <= 2_000_000:
            want = brute.solve_tables(t)
            got = orc.solve_tables(t)
            for k in KEYS:
                if k in want:
                    assert got[k] == want[k], (p["name"], k)
