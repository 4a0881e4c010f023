"""ctypes wrapper of the C oracle (oracle.c) -- TEST INFRASTRUCTURE ONLY.

Marshals the plain dicts of ``gen.tables`` / ``gen.profiles`` into the oracle's
own C structs (declared again here; nothing is shared with the product
binding).  ``build_oracle()`` compiles ``liboracle.so`` with gcc.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
INT64_MAX = (1 << 63) - 1

ORC_OK, ORC_ERR_ARG, ORC_ERR_INFEASIBLE, ORC_ERR_RANGE = 0, 1, 2, 3
MAX_L = 64


def build_oracle(force=False):
    src = os.path.join(HERE, "oracle.c")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src),
                                                  os.path.getmtime(os.path.join(HERE, "oracle.h")))):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-march=native", "-std=c11", "-fPIC", "-shared", "-Wall", "-Wextra",
           "-Wno-unused-parameter", "-o", LIB_PATH, src, "-lpthread"]
    subprocess.run(cmd, check=True)
    return LIB_PATH


class _Cfg(C.Structure):
    _fields_ = [("deg", C.c_int32), ("c", C.c_int32), ("n_strat", C.c_int32),
                ("A", C.POINTER(C.c_int32)), ("M", C.POINTER(C.c_int32)), ("R", C.POINTER(C.c_int32)),
                ("Rskip", C.POINTER(C.c_int32)), ("O", C.POINTER(C.c_int32)),
                ("stage_cap", C.POINTER(C.c_int32)), ("Rcut", C.POINTER(C.c_int32)),
                ("M_stage", C.POINTER(C.c_int32)), ("Rskips", C.POINTER(C.c_int32))]


class _Tables(C.Structure):
    _fields_ = [("L", C.c_int32), ("cap", C.c_int32), ("skip_src", C.c_int32), ("n_cfg", C.c_int32),
                ("cfg", C.POINTER(_Cfg)), ("n_skip", C.c_int32), ("skip_srcs", C.POINTER(C.c_int32))]


class _Result(C.Structure):
    _fields_ = [("objective", C.c_int64), ("cfg_index", C.c_int32), ("deg", C.c_int32), ("c", C.c_int32),
                ("L", C.c_int32), ("stage_of", C.c_int32 * MAX_L), ("strategy_of", C.c_int32 * MAX_L),
                ("stage_cost", C.c_int64 * MAX_L), ("cut_cost", C.c_int64 * MAX_L),
                ("stage_mem", C.c_int32 * MAX_L)]


class _Layer(C.Structure):
    _fields_ = [("fwd_ns", C.POINTER(C.c_int64)), ("param_bytes", C.c_int64),
                ("act_bytes", C.POINTER(C.c_int64)), ("ctx_bytes", C.c_int64), ("tpcomm_bytes", C.c_int64)]


class _Edge(C.Structure):
    _fields_ = [("src", C.c_int32), ("dst", C.c_int32), ("tensor_bytes", C.c_int64),
                ("reshard_ns", C.POINTER(C.c_int64)), ("cut_ns", C.POINTER(C.c_int64))]


class _Cluster(C.Structure):
    _fields_ = [("n_dev", C.c_int32), ("node_size", C.c_int32), ("mem_bytes", C.c_int64),
                ("mem_reserve", C.c_int64), ("bw_intra", C.c_int64), ("bw_inter", C.c_int64),
                ("p2p_bw", C.c_int64), ("lat_ns", C.c_int64), ("ccoc_permille", C.c_int32),
                ("dev_mem", C.POINTER(C.c_int64))]


class _Model(C.Structure):
    _fields_ = [("L", C.c_int32), ("layers", C.POINTER(_Layer)), ("n_edges", C.c_int32),
                ("edges", C.POINTER(_Edge))]


class _Options(C.Structure):
    _fields_ = [("B", C.c_int32), ("precision", C.c_int32), ("Q", C.c_int32), ("quantum_ns", C.c_int64),
                ("cand", C.POINTER(C.c_int32)), ("n_cand", C.c_int32), ("strategy_space", C.c_int32),
                ("schedule", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_solve.argtypes = [C.POINTER(_Tables), C.c_int, C.POINTER(_Result), C.POINTER(C.c_int64)]
        _lib.orc_interval_table.argtypes = [C.POINTER(_Tables), C.c_int, C.POINTER(C.c_int64)]
        _lib.orc_build.argtypes = [C.POINTER(_Model), C.POINTER(_Cluster), C.POINTER(_Options),
                                   C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        _lib.orc_catalogue.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32]
        _lib.orc_candidates.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32]
        for f in ("orc_allreduce_ns", "orc_allgather_ns"):
            getattr(_lib, f).argtypes = [C.c_int64] * 4
            getattr(_lib, f).restype = C.c_int64
        _lib.orc_p2p_ns.argtypes = [C.c_int64] * 3
        _lib.orc_p2p_ns.restype = C.c_int64
        _lib.orc_overlap_ns.argtypes = [C.c_int64, C.c_int64, C.c_int32]
        _lib.orc_overlap_ns.restype = C.c_int64
    return _lib


def _i32(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _ptr32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32)) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def _marshal_tables(t):
    keep = []
    cfgs = (_Cfg * len(t["cfgs"]))()
    L = t["L"]
    for i, c in enumerate(t["cfgs"]):
        S = c["n_strat"]
        A = _i32(c["A"]).reshape(L, S)
        M = _i32(c["M"]).reshape(L, S) if c.get("M") is not None else None
        R = _i32(c["R"]).reshape(max(L - 1, 0), S, S) if L > 1 else np.zeros((1, S, S), np.int32)
        Rs = _i32(c["Rskip"]).reshape(L, S, S) if c.get("Rskip") is not None else None
        O = _i32(c["O"]).reshape(max(L - 1, 0)) if c.get("O") is not None else None
        if O is not None and O.size == 0:
            O = np.zeros(1, np.int32)
        SC = _i32(c["stage_cap"]).reshape(c["deg"]) if c.get("stage_cap") is not None else None
        RC = _i32(c["Rcut"]).reshape(L - 1, S, S) if c.get("Rcut") is not None and L > 1 else None
        MS = _i32(c["M_stage"]).reshape(c["deg"], L, S) if c.get("M_stage") is not None else None
        srcs = t.get("skip_srcs") or []
        RSS = _i32(c["Rskips"]).reshape(len(srcs), L, S, S) if c.get("Rskips") is not None and srcs else None
        keep += [A, M, R, Rs, O, SC, RC, MS, RSS]
        cfgs[i] = _Cfg(c["deg"], c["c"], S, _ptr32(A), _ptr32(M), _ptr32(R), _ptr32(Rs), _ptr32(O), _ptr32(SC),
                       _ptr32(RC), _ptr32(MS), _ptr32(RSS))
    srcs = _i32(t.get("skip_srcs") or [0])
    keep.append(srcs)
    tb = _Tables(L, t["cap"], t.get("skip_src", -1), len(t["cfgs"]), cfgs, len(t.get("skip_srcs") or []),
                 _ptr32(srcs))
    keep.append(cfgs)
    return tb, keep


def solve_tables(t, n_threads=1):
    """Solve level-1 tables.  Returns a dict (objective INT64_MAX if infeasible)."""
    tb, keep = _marshal_tables(t)
    res = _Result()
    cfg_obj = (C.c_int64 * len(t["cfgs"]))()
    st = lib().orc_solve(C.byref(tb), n_threads, C.byref(res), cfg_obj)
    if st not in (ORC_OK, ORC_ERR_INFEASIBLE):
        raise OracleError(st, "solve")
    L = t["L"]
    deg = res.deg
    out = {"status": st, "objective": res.objective, "cfg_index": res.cfg_index, "deg": deg, "c": res.c,
           "cfg_objective": list(cfg_obj)}
    if st == ORC_OK:
        out.update({"stage_of": list(res.stage_of[:L]), "strategy_of": list(res.strategy_of[:L]),
                    "stage_cost": list(res.stage_cost[:deg]), "cut_cost": list(res.cut_cost[:max(deg - 1, 0)]),
                    "stage_mem": list(res.stage_mem[:deg])})
    return out


def interval_table(t, cfg):
    tb, keep = _marshal_tables(t)
    L = t["L"]
    P = np.zeros(L * L, dtype=np.int64)
    st = lib().orc_interval_table(C.byref(tb), cfg, P.ctypes.data_as(C.POINTER(C.c_int64)))
    if st != ORC_OK:
        raise OracleError(st, "interval_table")
    return P.reshape(L, L)


def allreduce_ns(V, G, bw, lat):
    return lib().orc_allreduce_ns(V, G, bw, lat)


def allgather_ns(V, G, bw, lat):
    return lib().orc_allgather_ns(V, G, bw, lat)


def p2p_ns(V, bw, lat):
    return lib().orc_p2p_ns(V, bw, lat)


def overlap_ns(comp, comm, ccoc_permille):
    return lib().orc_overlap_ns(comp, comm, ccoc_permille)


def catalogue(g, space=0):
    buf = (C.c_int32 * (3 * 64))()
    n = lib().orc_catalogue(g, space, buf, 64)
    return [tuple(buf[3 * i:3 * i + 3]) for i in range(min(n, 64))]


def candidates(n, B):
    buf = (C.c_int32 * 8192)()
    k = lib().orc_candidates(n, B, buf, 4096)
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(k)]


def _marshal_profile(p):
    keep = []
    m = p["model"]
    L = m["L"]
    layers = (_Layer * L)()
    for u, ly in enumerate(m["layers"]):
        f = np.ascontiguousarray(ly["fwd_ns_per_sample"], dtype=np.int64)
        a = np.ascontiguousarray(ly["act_bytes_per_sample"], dtype=np.int64)
        keep += [f, a]
        layers[u] = _Layer(f.ctypes.data_as(C.POINTER(C.c_int64)), ly["param_bytes"],
                           a.ctypes.data_as(C.POINTER(C.c_int64)), ly["ctx_bytes"],
                           ly["tp_comm_bytes_per_sample"])
    E = len(m["edges"])
    edges = (_Edge * max(E, 1))()
    def _mat(x):
        if x is None:
            return None
        x = np.ascontiguousarray(x, dtype=np.int64).reshape(-1)
        keep.append(x)
        return x.ctypes.data_as(C.POINTER(C.c_int64))
    for i, e in enumerate(m["edges"]):
        edges[i] = _Edge(e["src"], e["dst"], e["tensor_bytes_per_sample"], _mat(e.get("reshard_ns_per_sample")),
                         _mat(e.get("cut_ns_per_sample")))
    model = _Model(L, layers, E, edges)
    cl = p["cluster"]
    dm = None
    if cl.get("dev_mem_bytes") is not None:
        dm = np.ascontiguousarray(cl["dev_mem_bytes"], dtype=np.int64)
        keep.append(dm)
    cluster = _Cluster(cl["n_dev"], cl["node_size"], cl["mem_bytes"], cl["mem_reserve_bytes"],
                       cl["bw_intra_Bps"], cl["bw_inter_Bps"], cl["p2p_Bps"], cl["lat_ns"], cl["ccoc_permille"],
                       None if dm is None else dm.ctypes.data_as(C.POINTER(C.c_int64)))
    o = p["options"]
    cand = None
    if o.get("cand"):
        cand = np.ascontiguousarray(np.array(o["cand"], dtype=np.int32).reshape(-1))
        keep.append(cand)
    opts = _Options(o["B"], o["precision"], o["Q"], o.get("quantum_ns", 0),
                    _ptr32(cand), 0 if cand is None else len(cand) // 2, o.get("strategy_space", 0),
                    o.get("schedule", 0))
    keep += [layers, edges]
    return model, cluster, opts, keep


def build_tables(p):
    """Builder': profile -> (tables dict, quantum_ns, flat int32 buffer)."""
    model, cluster, opts, keep = _marshal_profile(p)
    n_cfg, skip, qn, words, nsk = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
    srcs = (C.c_int32 * 8)()
    st = lib().orc_build(C.byref(model), C.byref(cluster), C.byref(opts), None, 0, C.byref(n_cfg),
                         C.byref(skip), C.byref(qn), C.byref(words), C.byref(nsk), srcs)
    if st != ORC_OK:
        raise OracleError(st, "build(size)")
    buf = np.zeros(words.value, dtype=np.int32)
    st = lib().orc_build(C.byref(model), C.byref(cluster), C.byref(opts), _ptr32(buf), words.value,
                         C.byref(n_cfg), C.byref(skip), C.byref(qn), C.byref(words), C.byref(nsk), srcs)
    if st != ORC_OK:
        raise OracleError(st, "build")
    return unpack_buffer(buf, p["model"]["L"], p["options"]["Q"] - 1, skip.value, n_cfg.value,
                         list(srcs[:nsk.value])), qn.value, buf


def unpack_buffer(buf, L, cap, skip_src, n_cfg, skip_srcs=()):
    """Split the builder block layout into a tables dict (``skip_srcs``:
    several skip sources, their tables at each block's tail)."""
    cfgs, off = [], 0
    for _ in range(n_cfg):
        deg, c, S, g = (int(x) for x in buf[off:off + 4])
        off += 4
        A = buf[off:off + L * S].reshape(L, S); off += L * S
        M = buf[off:off + L * S].reshape(L, S); off += L * S
        R = buf[off:off + (L - 1) * S * S].reshape(L - 1, S, S); off += (L - 1) * S * S
        Rs = buf[off:off + L * S * S].reshape(L, S, S); off += L * S * S
        O = buf[off:off + L - 1]; off += L - 1
        SC = buf[off:off + deg]; off += deg
        has_rcut = int(buf[off]); off += 1
        RC = None
        if has_rcut:
            RC = buf[off:off + (L - 1) * S * S].reshape(L - 1, S, S); off += (L - 1) * S * S
        has_ms = int(buf[off]); off += 1
        MS = None
        if has_ms:
            MS = buf[off:off + deg * L * S].reshape(deg, L, S); off += deg * L * S
        RSS = None
        if len(skip_srcs) >= 2:
            n = len(skip_srcs)
            RSS = buf[off:off + n * L * S * S].reshape(n, L, S, S); off += n * L * S * S
        cfgs.append({"deg": deg, "c": c, "n_strat": S, "g": g, "A": A, "M": M, "R": R,
                     "Rskip": Rs if skip_src >= 0 else None, "O": O, "stage_cap": SC, "Rcut": RC,
                     "M_stage": MS, "Rskips": RSS})
    t = {"L": L, "cap": cap, "skip_src": skip_src, "cfgs": cfgs}
    if len(skip_srcs) >= 2:
        t["skip_srcs"] = list(skip_srcs)
    return t


def plan(p, n_threads=1):
    """Whole oracle pipeline on a profile: builder' + solve."""
    t, qn, _ = build_tables(p)
    r = solve_tables(t, n_threads)
    r["quantum_ns"] = qn
    return r, t
