"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact
(objective, per-config optima, deg, c, stage_of, strategy_of, p, o, memory).

The bar is bit-exact equality: everything is integer (DESIGN.md Sec. 2,
readings A-8..A-10).  Sizes: the toy; thousands of random tiny instances
(brute-force-checked oracle); random tables spanning several tiles, ragged
bucket tails and the cluster (DSMEM) path; the five synthetic model profiles
at full size (BASELINE.json configs); builder tables; edge cases.
"""
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


def test_toy(h, orc):
    for cands in (tables.TOY_GRID, [(1, 1), (2, 2)], [(1, 2)], [(2, 1)]):
        t = tables.toy_tables(cands)
        _same(h.solve_tables(t), orc.solve_tables(t), cands)


@pytest.mark.parametrize("chunk", range(4))
def test_random_tiny(h, orc, chunk):
    for seed in range(chunk * 600, (chunk + 1) * 600):
        t = tables.random_tables(seed)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)


def test_random_wide_strategy_sets(h, orc):
    """|S| up to 32 (every kernel class), L up to 10, tie-heavy and uniform."""
    rng = np.random.default_rng(5)
    for seed in range(150):
        L = int(rng.integers(1, 11))
        t = tables.random_tables(50_000 + seed, L=L, S_max=int(rng.choice([4, 8, 12, 16, 24, 32])),
                                 cap=int(rng.integers(0, 40)), n_cfg=int(rng.integers(1, 5)))
        _same(h.solve_tables(t), orc.solve_tables(t), seed)


@pytest.mark.parametrize("Q", [1, 7, 31, 33, 64, 100, 129, 300, 513, 1024, 1025, 2047, 3000, 4096, 5000, 8192])
def test_interval_table_elementwise(h, orc, Q):
    """Every interval optimum P[a][b], element by element, across bucket
    counts that exercise each K2 shape, ragged tails and the cluster path."""
    rng = np.random.default_rng(Q)
    for S in (1, 3, 6, 10, 15, 21):
        if Q > 2048 and S > 15:
            continue
        L = 12 if Q <= 1024 else 6
        skip = int(rng.integers(0, L - 2)) if rng.random() < 0.5 else -1
        t = tables.large_random_tables(Q * 100 + S, L, [S], Q - 1, [(1, 1)], skip_src=skip,
                                       mem_max=max(1, (3 * Q) // L))
        got = h.interval_table(t, 0).astype(np.int64)
        want = orc.interval_table(t, 0)
        want = np.where(want == (1 << 63) - 1, 0x40000000, want)
        iu = np.triu_indices(L)
        assert np.array_equal(got[iu], want[iu]), (Q, S, skip)


@pytest.mark.parametrize("L,S,Q", [(64, 32, 256), (4, 32, 8192), (64, 21, 64), (3, 24, 8192)])
def test_maximum_sizes(h, orc, L, S, Q):
    """The ABI's maxima (L = 64 layers, |S| = 32 strategies, Q = 8192
    buckets: the widest cluster class) element by element, then the whole
    solve over deg 1 / 2 / L."""
    cands = [(1, 1), (2, 2), (L, 3)]
    t = tables.large_random_tables(L * 1000 + S, L, [S, S, S], Q - 1, cands, skip_src=min(5, L - 3) if L >= 3 else -1,
                                   mem_max=max(1, (2 * Q) // max(L // 2, 1)))
    got = h.interval_table(t, 0).astype(np.int64)
    want = orc.interval_table(t, 0)
    want = np.where(want == (1 << 63) - 1, 0x40000000, want)
    iu = np.triu_indices(L)
    assert np.array_equal(got[iu], want[iu]), (L, S, Q)
    _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), (L, S, Q))


@pytest.mark.parametrize("dist", ["uniform", "ties"])
def test_random_gpu_sized(h, orc, dist):
    """Several configs of mixed |S|, L = 24, Q = 1000 (ragged), skip edges."""
    rng = np.random.default_rng(11 if dist == "ties" else 12)
    cands = [(1, 1), (2, 2), (2, 4), (4, 2), (4, 8), (8, 4), (24, 2), (25, 3)]
    S = [int(rng.choice([1, 3, 6, 10, 15])) for _ in cands]
    t = tables.large_random_tables(77, 24, S, 999, cands, skip_src=9, dist=dist)
    _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), dist)


def test_cluster_path_solve(h, orc):
    """Q = 4096 with |S| = 15 and 21: the DSMEM cluster variant end to end."""
    cands = [(1, 1), (2, 2), (3, 4)]
    t = tables.large_random_tables(99, 10, [21, 15, 10], 4095, cands, skip_src=3, mem_max=900)
    _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), "cluster")


@pytest.mark.parametrize("name", ["bert", "t5", "vit", "swin", "llama"])
def test_models_full_size(h, orc, name):
    """The BASELINE.json workloads at full size: oracle tables -> GPU solve;
    GPU plan (K1 + solve) -> same answer; builder tables bit-equal."""
    p = profiles.make_profile(name)
    t, qn, buf = orc.build_tables(p)
    want = orc.solve_tables(t, n_threads=0)
    _same(h.solve_tables(t), want, name)
    gt, gq, gbuf = h.build_tables(p)
    assert gq == qn and np.array_equal(gbuf, buf), name
    got = h.plan(p)
    _same(got, want, name + " plan")
    assert got["quantum_ns"] == qn


def test_prepared_profile_object(h, orc):
    """pkg.Profile (marshalled once, reused; arrays edited in place) gives the
    oracle's answer on every call, like the dict path."""
    import paper_2307_16375_b200 as pkg
    p = profiles.make_profile("vit")
    prof = pkg.Profile(p)
    want, _ = orc.plan(p)
    for _ in range(2):
        h.prepare(prof)
        h.run()
        _same(h.fetch(), want, "vit Profile")
    # edit in place: halve every forward time; the dict path of the edited
    # profile is the reference
    prof.fwd[:] = prof.fwd // 2
    for ly, row in zip(p["model"]["layers"], prof.fwd):
        ly["fwd_ns_per_sample"] = [int(x) for x in row]
    want2, _ = orc.plan(p)
    _same(h.plan(prof), want2, "vit Profile edited")


def test_models_nojitter_ties(h, orc):
    for name in ("bert", "vit"):
        p = profiles.make_profile(name, jitter=False)
        t, qn, buf = orc.build_tables(p)
        _same(h.solve_tables(t), orc.solve_tables(t, n_threads=0), name)


def test_builder_random_profiles(h, orc):
    for seed in range(60):
        p = profiles.random_profile(seed)
        try:
            t, qn, buf = orc.build_tables(p)
        except orc.OracleError as e:
            import paper_2307_16375_b200 as pkg
            with pytest.raises(pkg.UniapError) as ei:
                h.build_tables(p)
            assert ei.value.status == e.status
            continue
        gt, gq, gbuf = h.build_tables(p)
        assert gq == qn and np.array_equal(gbuf, buf), seed
        _same(h.plan(p), orc.solve_tables(t), seed)


@pytest.mark.parametrize("L,Q", [(None, None), (24, 1024), (40, 4096)])
def test_plan_random_profiles(h, orc, L, Q):
    """Level 2 end to end (GPU builder, plan-time sweep trim from the host
    memory bound, solve) = the oracle's builder' + solve, on random profiles
    whose memory often binds; out-of-range profiles fail with the same status."""
    import paper_2307_16375_b200 as pkg
    checked = 0
    for seed in range({None: 40, 24: 12, 40: 6}[L]):
        p = profiles.random_profile(1000 * (L or 1) + seed, L=L, Q=Q)
        try:
            want, _ = orc.plan(p)
        except orc.OracleError as e:
            with pytest.raises(pkg.UniapError) as ei:
                h.plan(p)
            assert ei.value.status == e.status
            continue
        got = h.plan(p)
        for k in ("objective", "deg", "c", "quantum_ns", "cfg_objective"):
            assert got[k] == want[k], (seed, k)
        if want["objective"] != (1 << 63) - 1:
            assert got["stage_of"] == want["stage_of"] and got["strategy_of"] == want["strategy_of"], seed
        checked += 1
    assert checked > 0


def test_edge_cases(h, orc):
    # L = 1; deg = L; deg > L; cap = 0; everything infeasible
    for seed in range(40):
        t = tables.random_tables(90_000 + seed, L=1)
        _same(h.solve_tables(t), orc.solve_tables(t), seed)
    t = tables.random_tables(3, L=5, cap=0, n_cfg=3)
    _same(h.solve_tables(t), orc.solve_tables(t))
    t = tables.large_random_tables(5, 6, [2, 2], 10, [(6, 2), (7, 1)])
    _same(h.solve_tables(t), orc.solve_tables(t))
    t = tables.large_random_tables(5, 6, [3], 10, [(1, 1)], forbid_p=1.0)
    g = h.solve_tables(t)
    assert g["status"] == 2 and g["objective"] == (1 << 63) - 1


def test_bad_tables_rejected(h):
    import paper_2307_16375_b200 as pkg
    t = tables.toy_tables()
    with pytest.raises(pkg.UniapError) as e:
        h.solve_tables(dict(t, cfgs=[t["cfgs"][0], t["cfgs"][0]]))
    assert e.value.status == 1
    with pytest.raises(pkg.UniapError) as e:
        h.solve_tables(dict(t, cfgs=[dict(t["cfgs"][0], A=t["cfgs"][0]["A"] + (1 << 22))]))
    assert e.value.status == 3


@pytest.mark.parametrize("name", ["vit", "t5"])
def test_world_size_invariance(h, orc, name):
    """Shards of world 2/4/8 run one after another on one GPU ("fake world"),
    records picked on the host == the ORACLE's plan (the a-8 exchange path
    against the independent answer) and == the world-1 work counters
    (SURVEY.md T4)."""
    import torch
    import paper_2307_16375_b200 as pkg
    p = profiles.make_profile(name)
    want, _ = orc.plan(p, n_threads=0)
    ref = h.plan(p)
    for k in ("objective", "deg", "c", "cfg_index", "stage_of", "strategy_of", "stage_cost", "cut_cost", "stage_mem"):
        assert ref[k] == want[k], (1, k)
    for world in (2, 4, 8):
        h.prepare(p)
        recs = b""
        for rank in range(world):
            buf = torch.zeros(pkg.RECORD_BYTES, dtype=torch.uint8, device="cuda")
            h.run(rank, world, buf.data_ptr())
            torch.cuda.synchronize()
            recs += buf.cpu().numpy().tobytes()
        st, r = pkg.pick(recs, world)
        for k in ("objective", "deg", "c", "cfg_index", "stage_of", "strategy_of", "stage_cost", "cut_cost",
                  "stage_mem"):
            assert r[k] == want[k], (world, k)
        for k in ("dp_cells", "dp_relax", "dp_cells_canonical"):
            assert r[k] == ref[k], (world, k)


@pytest.mark.parametrize("name", ["t5", "llama", "bert"])
def test_split_run_world_sizes(h, orc, name):
    """uniap_run_phase at world 2/4/8 (phase 1 on every rank, headers
    gathered, phase 2: only the global winner's owner traces back), run one
    rank after another on one GPU: the picked records == the ORACLE's plan;
    every other rank's record carries no traceback (it loses the pick)."""
    import torch
    import paper_2307_16375_b200 as pkg
    p = profiles.make_profile(name)
    want, _ = orc.plan(p, n_threads=0)
    RB = pkg.RECORD_BYTES
    for world in (2, 4, 8):
        h.prepare(p)
        bufs = [torch.zeros(RB, dtype=torch.uint8, device="cuda") for _ in range(world)]
        hdrs = torch.zeros(world * RB, dtype=torch.uint8, device="cuda")
        for rank in range(world):
            h.run_phase(rank, world, bufs[rank].data_ptr(), 1)
            torch.cuda.synchronize()
            hdrs[rank * RB:(rank + 1) * RB].copy_(bufs[rank])
        recs = b""
        for rank in range(world):
            h.run_phase(rank, world, bufs[rank].data_ptr(), 1)
            h.run_phase(rank, world, bufs[rank].data_ptr(), 2, hdrs.data_ptr())
            torch.cuda.synchronize()
            recs += bufs[rank].cpu().numpy().tobytes()
        st, r = pkg.pick(recs, world)
        for k in ("objective", "deg", "c", "cfg_index", "stage_of", "strategy_of", "stage_cost", "cut_cost",
                  "stage_mem"):
            assert r[k] == want[k], (world, k)


def test_plan_shard_world_sizes(h, orc):
    """uniap_plan_shard (prepare + this rank's share in one
    call) for every rank of world 2 / 4, records picked on the host == the
    oracle's plan (ViT)."""
    import torch
    import paper_2307_16375_b200 as pkg
    p = profiles.make_profile("vit")
    want, _ = orc.plan(p, n_threads=0)
    for world in (2, 4):
        recs = b""
        for rank in range(world):
            buf = torch.zeros(pkg.RECORD_BYTES, dtype=torch.uint8, device="cuda")
            h.plan_shard(p, rank, world, buf.data_ptr())
            h.fetch()
            recs += buf.cpu().numpy().tobytes()
        st, r = pkg.pick(recs, world)
        for k in ("objective", "deg", "c", "cfg_index", "stage_of", "strategy_of", "stage_cost", "cut_cost",
                  "stage_mem"):
            assert r[k] == want[k], (world, k)


def test_interval_table_between_solves_keeps_the_captured_plan(h, orc):
    """solve -> interval_table -> solve on the SAME tables: the second solve
    replays the captured graph of the first, so the all-intervals call must
    not reallocate any buffer that graph uses."""
    for seed, (L, S, Q) in enumerate([(12, 6, 300), (20, 10, 1025), (6, 3, 8192)]):
        t = tables.large_random_tables(9000 + seed, L, [S, S], Q - 1, [(1, 1), (2, 2)], skip_src=2,
                                       mem_max=max(1, (3 * Q) // L))
        want = orc.solve_tables(t)
        _same(h.solve_tables(t), want, ("first", seed))
        P = h.interval_table(t, 1).astype(np.int64)
        ref = orc.interval_table(t, 1)
        ref = np.where(ref == (1 << 63) - 1, 0x40000000, ref)
        iu = np.triu_indices(L)
        assert np.array_equal(P[iu], ref[iu])
        _same(h.solve_tables(t), want, ("second", seed))


@pytest.mark.parametrize("space", [0, 1])
def test_builder_reshard_matrices_and_strategy_space(h, orc, space):
    """Per-edge resharding matrices (uniap_edge.reshard_ns_per_sample) and
    SPEC's strategy space (uniap_options.strategy_space): K1's tables are
    bit-equal to builder''s and the plan equals the oracle's."""
    import paper_2307_16375_b200 as pkg
    checked = 0
    for seed in range(40):
        n = [1, 2, 4, 6, 8, 12, 16][seed % 7]
        dim = sum(len(orc.catalogue(g, space)) for g in range(1, n + 1) if n % g == 0)
        p = profiles.random_profile(5000 + seed, n=n, mat_dim=dim, space=space)
        try:
            t, qn, buf = orc.build_tables(p)
        except orc.OracleError as e:
            with pytest.raises(pkg.UniapError) as ei:
                h.build_tables(p)
            assert ei.value.status == e.status
            continue
        gt, gq, gbuf = h.build_tables(p)
        assert gq == qn and np.array_equal(gbuf, buf), seed
        _same(h.plan(p), orc.solve_tables(t), seed)
        checked += 1
    assert checked > 10


def _recost(p, seed):
    """The same shapes (layers, edges, candidates, Q, schedule) with new cost
    values: every time, byte count and the cluster's memory and bandwidths
    drawn again -- what a re-profiled model looks like to uniap_prepare."""
    rng = np.random.default_rng(seed)
    q = {"name": p["name"] + "'", "options": dict(p["options"]), "cluster": dict(p["cluster"])}
    layers = []
    for ly in p["model"]["layers"]:
        f = int(rng.integers(10_000, 5_000_000))
        layers.append(dict(ly, fwd_ns_per_sample=[max(1, f // (i + 1) + int(rng.integers(0, 999)))
                                                  for i in range(len(ly["fwd_ns_per_sample"]))],
                           param_bytes=int(rng.integers(0, 1 << 31)),
                           act_bytes_per_sample=sorted((int(rng.integers(0, 1 << 28))
                                                        for _ in ly["act_bytes_per_sample"]), reverse=True),
                           ctx_bytes=int(rng.integers(0, 1 << 24))))
    edges = [dict(e, tensor_bytes_per_sample=int(rng.integers(0, 1 << 24))) for e in p["model"]["edges"]]
    q["model"] = dict(p["model"], layers=layers, edges=edges)
    q["cluster"].update(mem_bytes=int(rng.integers(1 << 30, 1 << 36)), bw_intra_Bps=int(rng.integers(1 << 30, 1 << 38)),
                        p2p_Bps=int(rng.integers(1 << 27, 1 << 36)))
    return q


@pytest.mark.parametrize("kind", ["chain", "dag", "1f1b"])
def test_layout_cache_sequences(h, orc, kind):
    """uniap_prepare keeps the level-2 layout (arena offsets, classes, levels,
    copies) and the captured graph when the shapes repeat: alternate
    same-shape re-costed profiles with a different-shape one, every plan equal
    to the oracle's (or failing with the oracle's status)."""
    import paper_2307_16375_b200 as pkg
    checked = 0
    for seed in range(8):
        rng = np.random.default_rng(seed)
        L = int(rng.integers(5, 11))
        p = profiles.random_profile(9100 + seed, L=L, Q=int(rng.choice([64, 256])), n_skip=2 if kind == "dag" else 0)
        if kind == "1f1b":
            p = dict(p, options=dict(p["options"], schedule=1))
        other = profiles.random_profile(9200 + seed, L=L + 1, Q=p["options"]["Q"])
        seq = [p, _recost(p, seed), p, other, _recost(p, seed + 50), _recost(p, seed)]
        for i, x in enumerate(seq):
            try:
                want, _ = orc.plan(x)
            except orc.OracleError as e:
                with pytest.raises(pkg.UniapError) as ei:
                    h.plan(x)
                assert ei.value.status == e.status, (seed, i)
                continue
            got = h.plan(x)
            for k in ("objective", "deg", "c", "quantum_ns", "cfg_objective"):
                assert got[k] == want[k], (kind, seed, i, k)
            if want["objective"] != (1 << 63) - 1:
                assert got["stage_of"] == want["stage_of"] and got["strategy_of"] == want["strategy_of"], (seed, i)
            checked += 1
    assert checked >= 24


@pytest.mark.parametrize("S,Q", [(11, 129), (16, 300), (24, 777), (32, 1024), (12, 1025)])
def test_lone_chain_cluster_shapes(h, orc, S, Q):
    """A lone deg = 1 chain (no skip source) with |S| > 10: at Q <= 1024 it
    runs on a cluster of 128-bucket CTAs, one bucket per thread (2 .. 8 CTAs,
    ragged tails); Q = 1025 keeps the 256-bucket shape.  The solve and every
    interval-table entry against the oracle, with a deg = 2 config beside it."""
    from test_gpu_plan_parity import check
    t = tables.large_random_tables(60_000 + S * 7 + Q, 20, [S, max(2, S // 3)], Q - 1, [(1, 4), (2, 2)],
                                   dist="ties" if S % 2 else "uniform")
    got = h.solve_tables(t)
    check(h, orc, t, h.fetch_intervals(), ("lone chain", S, Q))
    _same(got, orc.solve_tables(t, n_threads=0), (S, Q))
