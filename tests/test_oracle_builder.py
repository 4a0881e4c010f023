"""Pins of the oracle's builder' (the cost model) against the
paper's Eq. (1) anchors and SPEC.md's worked examples rescaled to integer ns
and bytes (CPU only).  Absolute builder values are otherwise "parity
unpinned" against the paper (it prints no per-layer tables)."""
import numpy as np

from gen import profiles

GB = 10 ** 9


def _profile(L=1, n=1, B=4, fwd=None, ps=0, act=None, tpcomm=0, ctx=0, edges=(), Q=1024, mem=None,
             precision=0, quantum=100, cand=None, bw=GB, p2p=GB, lat=0, ccoc=0, node=64):
    tps = profiles.tp_sizes(n)
    fwd = fwd or [10_000_000 // t for t in tps]
    act = act or [0 for _ in tps]
    layers = [{"fwd_ns_per_sample": list(fwd), "param_bytes": ps, "act_bytes_per_sample": list(act),
               "ctx_bytes": ctx, "tp_comm_bytes_per_sample": tpcomm} for _ in range(L)]
    return {"name": "unit", "model": {"L": L, "layers": layers,
                                      "edges": [dict(src=a, dst=b, tensor_bytes_per_sample=v) for a, b, v in edges]},
            "cluster": dict(n_dev=n, node_size=node, mem_bytes=mem or (Q - 1), mem_reserve_bytes=0,
                            bw_intra_Bps=bw, bw_inter_Bps=bw, p2p_Bps=p2p, lat_ns=lat, ccoc_permille=ccoc),
            "options": dict(B=B, precision=precision, Q=Q, quantum_ns=quantum, cand=cand)}


def _strat(orc, g, tfd):
    return orc.catalogue(g).index(tfd)


def test_spec_allreduce_p2p_overlap_examples(orc):
    """SPEC.md:149-151 (ring all-reduce 1.0 s / 1.5 s), 159-161 (p2p
    0.50001 s), 169-171 (overlap 5/3/4), in ns."""
    assert orc.allreduce_ns(10 ** 9, 1, GB, 0) == 0
    assert orc.allreduce_ns(10 ** 9, 2, GB, 0) == 1_000_000_000
    assert orc.allreduce_ns(10 ** 9, 4, GB, 0) == 1_500_000_000
    assert orc.p2p_ns(0, GB, 0) == 0
    assert orc.p2p_ns(10 ** 9, GB, 0) == 1_000_000_000
    assert orc.p2p_ns(5 * 10 ** 8, GB, 10_000) == 500_010_000
    assert orc.overlap_ns(3, 2, 0) == 5
    assert orc.overlap_ns(3, 2, 1000) == 3
    assert orc.overlap_ns(3, 2, 500) == 4
    # monotone in volume and (lat = 0) in group size
    vals = [orc.allreduce_ns(v, g, GB, 0) for g in (2, 4, 8) for v in (1, 10 ** 6, 10 ** 9)]
    assert vals == sorted(vals) or all(orc.allreduce_ns(v, 2, GB, 0) <= orc.allreduce_ns(v, 4, GB, 0) for v in (1, 10 ** 6))


def test_layer_exec_cost_examples(orc):
    """(dp=1,tp=1), b=4, 0.01 s/sample -> 0.12 s (fp 0.04 +
    bp 0.08); (dp=2), b=4 -> 0.06 s; b=3 with dp=2 -> forbidden."""
    t, qn, _ = orc.build_tables(_profile(n=1, B=4))
    assert qn == 100 and t["cfgs"][0]["A"][0, 0] == 120_000_000 // 100
    t, qn, _ = orc.build_tables(_profile(n=2, B=4, cand=[(1, 1)]))
    k = _strat(orc, 2, (1, 1, 2))
    assert t["cfgs"][0]["A"][0, k] == 60_000_000 // 100
    t, qn, _ = orc.build_tables(_profile(n=2, B=3, cand=[(1, 1)]))
    assert t["cfgs"][0]["M"][0, k] == t["cap"] + 1


def test_eq1_memory_anchors(orc):
    """Eq. (1): m_s = c_dtype * ps / (ts * fs) with c_dtype
    = 4 (FP32) and 8 (FP16 mixed); ps=16, FP32, ts=2, fs=2 -> 16 B.
    Memory unit = 1 byte here (mem = Q-1), so M is in bytes."""
    t, _, _ = orc.build_tables(_profile(n=4, B=4, ps=16, cand=[(1, 1)]))
    assert t["cfgs"][0]["M"][0, _strat(orc, 4, (2, 2, 1))] == 16
    for prec, cd in ((0, 4), (1, 8)):
        ps = 100
        t, _, _ = orc.build_tables(_profile(n=1, B=1, ps=ps, precision=prec))
        assert t["cfgs"][0]["M"][0, 0] == cd * ps
        for ts in (1, 2, 4):
            for fs in (1, 2, 4):
                n = ts * fs
                t, _, _ = orc.build_tables(_profile(n=n, B=n, ps=ps * 8, precision=prec, cand=[(1, 1)], Q=8192))
                assert t["cfgs"][0]["M"][0, _strat(orc, n, (ts, fs, 1))] == -(-cd * ps * 8 // (ts * fs))


def test_activation_memory_gpipe_inflight(orc):
    """Reading A-12: GPipe keeps all c micro-batches in flight, m_a =
    c * (b/r) * act[t] = (B/r) * act[t], independent of c."""
    for cand in ([(2, 2)], [(2, 4)]):
        t, _, _ = orc.build_tables(_profile(L=2, n=4, B=8, act=[10, 6, 4], cand=cand))
        cfg = t["cfgs"][0]  # g = 2
        assert cfg["M"][0, _strat(orc, 2, (1, 1, 2))] == 8 // 2 * 10
        assert cfg["M"][0, _strat(orc, 2, (2, 1, 1))] == 8 * 6


def test_resharding_examples(orc):
    """SPEC.md:238-240 (one direction): same-stage (dp=1,tp=2)->(dp=2,tp=1),
    b=2, 1e6 B/sample, 1e9 B/s -> 0.002 s; cross-stage (1,1)->(1,1), b=4 ->
    0.004 s.  Ours charges forward + backward (x2, reading A-15)."""
    prof = _profile(L=2, n=2, B=2, edges=[(0, 1, 10 ** 6)], cand=[(1, 1)], quantum=1000)
    t, qn, _ = orc.build_tables(prof)
    R = t["cfgs"][0]["R"][0]
    k_tp, k_dp = _strat(orc, 2, (2, 1, 1)), _strat(orc, 2, (1, 1, 2))
    assert R[k_tp, k_dp] == 2 * 2_000_000 // 1000
    assert all(R[k, k] == 0 for k in range(3))          # R diagonal = 0
    prof = _profile(L=2, n=2, B=4, edges=[(0, 1, 10 ** 6)], cand=[(2, 1)], quantum=1000)
    t, qn, _ = orc.build_tables(prof)
    assert t["cfgs"][0]["O"][0] == 2 * 4_000_000 // 1000


def test_cut_cost_counts_every_crossing_edge(orc):
    """Reading A-16: an edge skipping stages is charged at every cut it crosses."""
    prof = _profile(L=4, n=1, B=1, edges=[(0, 1, 10), (1, 2, 10), (2, 3, 10), (0, 2, 1000), (0, 3, 1000)],
                    cand=[(1, 1)], quantum=1, p2p=10 ** 9, lat=0, fwd=[1000])
    t, _, _ = orc.build_tables(prof)
    O = t["cfgs"][0]["O"]
    assert list(O) == [2 * (10 + 1000 + 1000), 2 * (10 + 1000 + 1000), 2 * (10 + 1000)]
    assert t["skip_src"] == 0


def test_bp_is_twice_fp_and_linear_in_b(orc):
    """PAPER.md:95 bp = 2 fp; doubling the micro-batch doubles the compute term."""
    a = [orc.build_tables(_profile(n=1, B=B, quantum=1, fwd=[1000]))[0]["cfgs"][0]["A"][0, 0] for B in (1, 2, 4)]
    assert a == [3000, 6000, 12000]


def test_auto_quantum_is_smallest_power_of_two(orc):
    """Reading A-9: auto quantum = smallest power of two with entries <= 2^22
    and per-config sums <= 2^28."""
    p = profiles.make_profile("bert")
    t, qn, _ = orc.build_tables(p)
    assert qn & (qn - 1) == 0
    for cfg in t["cfgs"]:
        assert cfg["A"].max() <= 1 << 22 and cfg["R"].max() <= 1 << 22
    p["options"]["quantum_ns"] = qn // 2
    try:
        orc.build_tables(p)
        ok_half = True
    except orc.OracleError:
        ok_half = False
    assert not ok_half


def test_all_models_build_and_solve(orc):
    for name in ("bert", "vit", "swin", "llama"):
        p = profiles.make_profile(name)
        t, qn, buf = orc.build_tables(p)
        assert len(t["cfgs"]) == {"bert": 16, "vit": 29, "swin": 25, "llama": 31}[name]
        assert buf.dtype == np.int32
