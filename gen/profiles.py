"""Seeded level-2 inputs: synthetic profiling results (Sec. 3.1).

The paper profiles real models on real clusters; we have neither, so each
workload is a synthetic integer profile shaped like one of the paper's
evaluated models (Table 5) on an alpha-beta cluster record
shaped like its environments.  The recipe is SURVEY.md
Sec. 8d and is restated in DESIGN.md Sec. 3.  These are INPUTS: the numbers
here stand in for measurements; the cost model that turns them into tables
 lives separately in the oracle and in the CUDA builder.

A *profile* dict:

    {"name": str,
     "model": {"L": int,
               "layers": [{"fwd_ns_per_sample": [int per TP size 1,2,4,..],
                           "param_bytes": int,
                           "act_bytes_per_sample": [int per TP size],
                           "ctx_bytes": int,
                           "tp_comm_bytes_per_sample": int}, ...],
               "edges": [{"src": int, "dst": int,
                          "tensor_bytes_per_sample": int}, ...]},
     "cluster": {"n_dev", "node_size", "mem_bytes", "mem_reserve_bytes",
                 "bw_intra_Bps", "bw_inter_Bps", "p2p_Bps", "lat_ns",
                 "ccoc_permille"},
     "options": {"B", "precision" (0 FP32, 1 FP16-mixed), "Q",
                 "quantum_ns" (0 = auto), "cand": None | [(deg, c), ...]}}
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["MODELS", "make_profile", "toy_profile", "random_profile", "tp_sizes"]

GiB = 1 << 30


def tp_sizes(n):
    """TP sizes profiled: powers of two dividing n (1, 2, 4, ...)."""
    out, t = [], 1
    while n % t == 0:
        out.append(t)
        t *= 2
    return out


def _fwd_ns(flops, tps, peak, eff, jitter=1.0):
    # fwd_ns[t] = ceil(FLOPs * 1e9 * jitter / (t * peak * eff * (1 - 0.06 log2 t)))
    return [int(math.ceil(flops * 1e9 * jitter / (t * peak * eff * (1.0 - 0.06 * math.log2(t)))))
            for t in tps]


def _act(bytes_, s, h, heads, skv, tps):
    # Korthikanti et al. activation bytes/sample without recompute (the paper
    # turns recompute off): s*h*(10 + 24/t) + 5*heads*s*skv/t
    # bytes at FP16, scaled by bytes_/2 for the training dtype.
    return [(bytes_ * (s * h * 10 + (s * h * 24) // t + (5 * heads * s * skv) // t)) // 2
            for t in tps]


ENV_A = dict(n_dev=8, node_size=8, mem_bytes=32 * GiB, mem_reserve_bytes=1 * GiB,
             bw_intra_Bps=100_000_000_000, bw_inter_Bps=100_000_000_000,
             p2p_Bps=40_000_000_000, lat_ns=10_000, ccoc_permille=300)
ENV_B = dict(n_dev=16, node_size=4, mem_bytes=12 * GiB, mem_reserve_bytes=GiB // 2,
             bw_intra_Bps=10_000_000_000, bw_inter_Bps=1_250_000_000,
             p2p_Bps=1_250_000_000, lat_ns=20_000, ccoc_permille=300)
ENV_LLAMA = dict(n_dev=32, node_size=8, mem_bytes=180_000_000_000, mem_reserve_bytes=4_000_000_000,
                 bw_intra_Bps=700_000_000_000, bw_inter_Bps=50_000_000_000,
                 p2p_Bps=50_000_000_000, lat_ns=5_000, ccoc_permille=500)
ENV_C = dict(n_dev=8, node_size=8, mem_bytes=40 * GiB, mem_reserve_bytes=2 * GiB,
             bw_intra_Bps=24_000_000_000, bw_inter_Bps=24_000_000_000,
             p2p_Bps=24_000_000_000, lat_ns=10_000, ccoc_permille=300)

PEAK = {"A": (15.7e12, 0.45), "B": (12.1e12, 0.45), "LLAMA": (2.25e15, 0.45), "C": (312e12, 0.45)}


def _layer(params, flops, bytes_, s, h, heads, skv, tps, peak, eff, jit=1.0):
    return {"fwd_ns_per_sample": _fwd_ns(flops, tps, peak, eff, jit),
            "param_bytes": int(params * bytes_),
            "act_bytes_per_sample": _act(bytes_, s, h, heads, skv, tps),
            "ctx_bytes": 0,
            "tp_comm_bytes_per_sample": 2 * s * h * bytes_}


def _chain_edges(out_bytes):
    return [{"src": u, "dst": u + 1, "tensor_bytes_per_sample": int(out_bytes[u])}
            for u in range(len(out_bytes) - 1)]


def _bert(jitter):
    h, s, heads, L = 1280, 512, 16, 32
    tps = tp_sizes(ENV_A["n_dev"])
    peak, eff = PEAK["A"]
    rng = np.random.default_rng(2307 + 1)
    layers = []
    for _ in range(L):
        p = 12 * h * h
        jit = 1.0 + (rng.uniform(-0.03, 0.03) if jitter else 0.0)
        layers.append(_layer(p, 2 * p * s + 4 * s * s * h, 4, s, h, heads, s, tps, peak, eff, jit))
    return {"L": L, "layers": layers, "edges": _chain_edges([s * h * 4] * L)}, ENV_A, dict(B=32, precision=0, Q=1024)


def _t5(jitter):
    h, s, heads, ffn, Le, Ld = 1024, 512, 16, 4096, 24, 24
    tps = tp_sizes(ENV_B["n_dev"])
    peak, eff = PEAK["B"]
    rng = np.random.default_rng(2307 + 2)
    layers = []
    for _ in range(Le):
        p = 4 * h * h + 2 * h * ffn
        jit = 1.0 + (rng.uniform(-0.03, 0.03) if jitter else 0.0)
        layers.append(_layer(p, 2 * p * s + 4 * s * s * h, 4, s, h, heads, s, tps, peak, eff, jit))
    for _ in range(Ld):
        p = 4 * h * h + 2 * h * ffn + 4 * h * h  # + cross-attention
        jit = 1.0 + (rng.uniform(-0.03, 0.03) if jitter else 0.0)
        fl = 2 * p * s + 4 * s * s * h + 4 * s * 512 * h
        layers.append(_layer(p, fl, 4, s, h, heads, s + 512, tps, peak, eff, jit))
    L = Le + Ld
    edges = _chain_edges([s * h * 4] * L)
    enc_out = 512 * 1024 * 4
    edges += [{"src": Le - 1, "dst": v, "tensor_bytes_per_sample": enc_out} for v in range(Le + 1, L)]
    return {"L": L, "layers": layers, "edges": edges}, ENV_B, dict(B=16, precision=0, Q=1024)


def _vit(jitter):
    h, s, heads, ffn, L = 1280, 197, 16, 5120, 32
    tps = tp_sizes(ENV_B["n_dev"])
    peak, eff = PEAK["B"]
    rng = np.random.default_rng(2307 + 3)
    layers = []
    for _ in range(L):
        p = 4 * h * h + 2 * h * ffn
        jit = 1.0 + (rng.uniform(-0.03, 0.03) if jitter else 0.0)
        layers.append(_layer(p, 2 * p * s + 4 * s * s * h, 4, s, h, heads, s, tps, peak, eff, jit))
    return {"L": L, "layers": layers, "edges": _chain_edges([s * h * 4] * L)}, ENV_B, dict(B=128, precision=0, Q=1024)


def _swin(jitter, with_embed_head=False):
    depths, dims, toks, win = (2, 2, 42, 2), (320, 640, 1280, 2560), (3136, 784, 196, 49), 49
    tps = tp_sizes(ENV_B["n_dev"])
    peak, eff = PEAK["B"]
    rng = np.random.default_rng(2307 + 4)
    layers, outb = [], []
    if with_embed_head:  # patch embedding 4x4x3 -> C0
        p = 48 * dims[0]
        layers.append(_layer(p, 2 * p * toks[0], 4, toks[0], dims[0], 1, 1, tps, peak, eff))
        outb.append(toks[0] * dims[0] * 4)
    for st, (dpt, C, T) in enumerate(zip(depths, dims, toks)):
        for i in range(dpt):
            p = 12 * C * C
            fl = 2 * p * T + 4 * T * win * C
            if st > 0 and i == 0:  # patch merging folded into the first block
                Cp = dims[st - 1]
                p += 8 * Cp * Cp
                fl += 2 * 8 * Cp * Cp * T
            jit = 1.0 + (rng.uniform(-0.03, 0.03) if jitter else 0.0)
            layers.append(_layer(p, fl, 4, T, C, C // 32, win, tps, peak, eff, jit))
            outb.append(T * C * 4)
    if with_embed_head:  # pooling + classifier head (1000 classes)
        p = dims[-1] * 1000
        layers.append(_layer(p, 2 * p, 4, 1, dims[-1], 1, 1, tps, peak, eff))
        outb.append(1000 * 4)
    L = len(layers)
    return {"L": L, "layers": layers, "edges": _chain_edges(outb)}, ENV_B, dict(B=64, precision=0, Q=1024)


def _llama(jitter, env=ENV_LLAMA, B=64, h=4096, L=32, ffn=11008, heads=32, Q=4096, peak_key="LLAMA"):
    s = 2048
    tps = tp_sizes(env["n_dev"])
    peak, eff = PEAK[peak_key]
    rng = np.random.default_rng(2307 + 5)
    layers = []
    for _ in range(L):
        p = 4 * h * h + 3 * h * ffn
        jit = 1.0 + (rng.uniform(-0.03, 0.03) if jitter else 0.0)
        layers.append(_layer(p, 2 * p * s + 4 * s * s * h, 2, s, h, heads, s, tps, peak, eff, jit))
    return {"L": L, "layers": layers, "edges": _chain_edges([s * h * 2] * L)}, env, dict(B=B, precision=1, Q=Q)


MODELS = {
    "bert": lambda j: _bert(j),
    "t5": lambda j: _t5(j),
    "vit": lambda j: _vit(True if j is None else j),
    "swin": lambda j: _swin(j),
    "swin50": lambda j: _swin(j, with_embed_head=True),
    "llama": lambda j: _llama(j),
    "llama-envc": lambda j: _llama(j, env=ENV_C, B=8, peak_key="C"),
    "llama13b": lambda j: _llama(j, env=dict(ENV_LLAMA, n_dev=64), B=128, h=5120, L=40,
                                 ffn=13824, heads=40),
}


def make_profile(name, jitter=None, Q=None, cand=None):
    """Synthetic profile of one of the paper's evaluated models (Table 5).

    jitter=None uses the survey default (ViT +-3 %, others exact); True/False
    forces it ('nojitter' variants stress ties).
    """
    model, cluster, opts = MODELS[name](jitter if jitter is not None else (None if name == "vit" else False))
    opts = dict(opts)
    if Q is not None:
        opts["Q"] = Q
    opts.setdefault("quantum_ns", 0)
    opts["cand"] = cand
    return {"name": name, "model": model, "cluster": dict(cluster), "options": opts}


def toy_profile():
    """Profile-level toy: 4 layers, n=2 devices, B=2."""
    tps = tp_sizes(2)
    layers = []
    for u in range(4):
        layers.append({"fwd_ns_per_sample": [1_000_000 + 100_000 * u, 560_000 + 50_000 * u],
                       "param_bytes": 4_000_000 * (1 + (u % 2)),
                       "act_bytes_per_sample": [2_000_000, 1_200_000][:len(tps)],
                       "ctx_bytes": 0, "tp_comm_bytes_per_sample": 1_000_000})
    edges = [{"src": u, "dst": u + 1, "tensor_bytes_per_sample": 500_000} for u in range(3)]
    cluster = dict(n_dev=2, node_size=2, mem_bytes=64_000_000, mem_reserve_bytes=0,
                   bw_intra_Bps=10_000_000_000, bw_inter_Bps=10_000_000_000,
                   p2p_Bps=5_000_000_000, lat_ns=10_000, ccoc_permille=300)
    return {"name": "toy", "model": {"L": 4, "layers": layers, "edges": edges},
            "cluster": cluster, "options": dict(B=2, precision=0, Q=8, quantum_ns=0, cand=None)}


def random_profile(seed, L=None, n=None, B=None, Q=None, skip=None, mat_dim=None, space=0, n_skip=0):
    """Random small profile for builder / end-to-end parity tests.

    ``mat_dim``: if given, about half of the edges carry a random resharding
    matrix of that order (``reshard_ns_per_sample``, ns per sample in
    [0, 2^20]; the caller passes |Cat| of the strategy space); ``space``: the
    options' strategy space."""
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 9)) if L is None else L
    n = int(rng.choice([1, 2, 4, 6, 8, 12, 16])) if n is None else n
    B = int(rng.choice([1, 2, 4, 6, 8, 16])) if B is None else B
    Q = int(rng.choice([2, 8, 16, 64, 256])) if Q is None else Q
    tps = tp_sizes(n)
    layers = []
    for _ in range(L):
        f1 = int(rng.integers(10_000, 5_000_000))
        layers.append({"fwd_ns_per_sample": [max(1, f1 // t + int(rng.integers(0, 1000))) for t in tps],
                       "param_bytes": int(rng.integers(0, 1 << 31)),
                       "act_bytes_per_sample": sorted([int(rng.integers(0, 1 << 28)) for _ in tps], reverse=True),
                       "ctx_bytes": int(rng.integers(0, 1 << 24)),
                       "tp_comm_bytes_per_sample": int(rng.integers(0, 1 << 24))})
    edges = [{"src": u, "dst": u + 1, "tensor_bytes_per_sample": int(rng.integers(0, 1 << 24))}
             for u in range(L - 1)]
    if (skip if skip is not None else rng.random() < 0.3) and L >= 4:
        s = int(rng.integers(0, L - 3))
        for v in range(s + 2, L):
            if rng.random() < 0.7:
                edges.append({"src": s, "dst": v, "tensor_bytes_per_sample": int(rng.integers(0, 1 << 24))})
    if n_skip:  # NEXT-4: a DAG with several skip sources (separate stream: the rest is unchanged)
        drng = np.random.default_rng(seed + 9_000_000)
        edges = [e for e in edges if e["dst"] == e["src"] + 1]
        cand = list(range(0, max(L - 2, 0)))
        srcs = sorted(int(x) for x in drng.choice(cand, size=min(n_skip, len(cand)), replace=False)) if cand else []
        for s in srcs:
            for v in range(s + 2, L):
                if drng.random() < 0.6:
                    edges.append({"src": s, "dst": v, "tensor_bytes_per_sample": int(drng.integers(0, 1 << 22))})
    node = int(rng.choice([d for d in (1, 2, 4, 8) if n % d == 0] or [1]))
    cluster = dict(n_dev=n, node_size=node, mem_bytes=int(rng.integers(1 << 30, 1 << 36)),
                   mem_reserve_bytes=int(rng.integers(0, 1 << 29)),
                   bw_intra_Bps=int(rng.integers(1 << 30, 1 << 38)),
                   bw_inter_Bps=int(rng.integers(1 << 27, 1 << 34)),
                   p2p_Bps=int(rng.integers(1 << 27, 1 << 36)),
                   lat_ns=int(rng.integers(0, 50_000)), ccoc_permille=int(rng.integers(0, 1001)))
    if mat_dim:
        mrng = np.random.default_rng(seed + 7_000_000)  # separate stream: the rest of the profile is unchanged
        for e in edges:
            if mrng.random() < 0.5:
                e["reshard_ns_per_sample"] = mrng.integers(0, 1 << 20, size=(mat_dim, mat_dim), dtype=np.int64)
    opts = dict(B=B, precision=int(rng.integers(0, 2)), Q=Q, quantum_ns=0, cand=None, strategy_space=space)
    return {"name": f"rand{seed}", "model": {"L": L, "layers": layers, "edges": edges},
            "cluster": cluster, "options": opts}
