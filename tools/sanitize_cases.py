"""Small runs of every kernel family for compute-sanitizer (racecheck /
synccheck / memcheck): toy tables, the BERT profile (level 2: K1 incl. the
K1f trim role, K2 one-CTA classes, K4, K5a, backward K2, K5c), a deg = 1
chain on a 16-CTA cluster at Q = 4096 (DSMEM fix-up, split cluster barrier,
kept G tables) and a skip-conditioned cluster case; each checked against the
oracle.  usage: python tools/sanitize_cases.py [case ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles, tables  # noqa: E402
from oracle import oracle  # noqa: E402


def same(g, o, what):
    for k in ("objective", "deg", "c", "stage_of", "strategy_of"):
        assert g.get(k) == o.get(k), (what, k, g.get(k), o.get(k))
    print("ok", what, g["objective"], flush=True)


def main(cases):
    h = pkg.Handle(0)
    if "toy" in cases:
        t = tables.toy_tables()
        same(h.solve_tables(t), oracle.solve_tables(t), "toy")
    if "bert" in cases:
        p = profiles.make_profile("bert")
        want, _ = oracle.plan(p, n_threads=0)
        same(h.plan(p), want, "bert plan")
    if "cluster" in cases:  # deg = 1, |S| = 21, Q = 4096: the 16-CTA cluster chain that keeps G
        t = tables.large_random_tables(99, 8, [21, 15], 4095, [(1, 1), (2, 2)], skip_src=-1, mem_max=900)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "cluster deg1")
    if "skip" in cases:  # skip-conditioned copies on clusters, Q = 4096
        t = tables.large_random_tables(7, 8, [10, 6], 4095, [(1, 1), (2, 2)], skip_src=2, mem_max=900)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "cluster skip")
    if "levels" in cases:  # NEXT-2: per-stage caps (cap levels, per-level launches, K4/K5a per level)
        t = tables.large_random_tables(61, 10, [6, 10, 3], 1023, [(2, 2), (3, 4), (4, 2)], skip_src=3,
                                       mem_max=300, stage_caps=True)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "stage caps")
    if "cut" in cases:  # NEXT-1: tmode K2, K4c, conditioned traceback
        import numpy as np
        t = tables.large_random_tables(62, 9, [6, 3, 5], 255, [(2, 2), (3, 4), (4, 2)], skip_src=2, mem_max=80,
                                       vmax=1 << 16)
        rng = np.random.default_rng(1)
        for c in t["cfgs"]:
            c["Rcut"] = rng.integers(0, 1 << 16, size=(8, c["n_strat"], c["n_strat"])).astype(np.int32)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "cut cost")
    if "1f1b" in cases:  # NEXT-2 1F1B: per-stage memory tables (levels, K4 from global memory at 16 levels)
        t = tables.with_1f1b(tables.large_random_tables(63, 20, [3, 4, 2], 255, [(4, 8), (16, 32), (2, 2)],
                                                        mem_max=10), 63, act_max=3)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "1f1b tables")
        p = profiles.make_profile("bert")
        p = dict(p, options=dict(p["options"], schedule=1))
        want, _ = oracle.plan(p, n_threads=0)
        same(h.plan(p), want, "bert 1f1b plan")
    if "dag" in cases:  # NEXT-4: several skip sources (copy tables, per-copy traceback over > 32 copies)
        t = tables.with_skip_sources(tables.large_random_tables(64, 12, [6, 4], 511, [(1, 1), (3, 2)], mem_max=60),
                                     64, 3, vmax=1 << 18)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "dag tables")
    if "lone" in cases:  # a lone deg = 1 chain, |S| = 16 at Q = 1024: 8 x 128-bucket cluster, one bucket per thread
        t = tables.large_random_tables(65, 10, [16, 5], 1023, [(1, 1), (2, 4)], mem_max=150)
        same(h.solve_tables(t), oracle.solve_tables(t, n_threads=0), "lone chain")
    h.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["toy", "bert", "cluster", "skip", "levels", "cut", "1f1b", "dag", "lone"])
