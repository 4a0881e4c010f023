"""Thin ctypes binding of libuniap.so (include/uniap.h) -- marshalling only.

Every step of the method runs inside the library's CUDA kernels; this module
only converts the plain dicts of ``gen`` (tables / profiles) into the C
structs of the ABI and the results back into dicts.  It raises if the
library is missing (no CPU fallback exists).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libuniap.so")
INT64_MAX = (1 << 63) - 1
MAX_L = 64

UNIAP_OK, UNIAP_ERR_ARG, UNIAP_ERR_INFEASIBLE, UNIAP_ERR_RANGE = 0, 1, 2, 3
UNIAP_ERR_CUDA, UNIAP_ERR_COMM, UNIAP_ERR_OOM, UNIAP_ERR_INTERNAL = 4, 5, 6, 99
UNIAP_INF = 0x40000000

_P32 = C.POINTER(C.c_int32)
_P64 = C.POINTER(C.c_int64)


class uniap_config(C.Structure):
    _fields_ = [("deg", C.c_int32), ("c", C.c_int32), ("n_strat", C.c_int32), ("A", _P32), ("M", _P32),
                ("R", _P32), ("Rskip", _P32), ("O", _P32), ("stage_cap", _P32), ("Rcut", _P32),
                ("M_stage", _P32), ("Rskips", _P32)]


class uniap_tables(C.Structure):
    _fields_ = [("L", C.c_int32), ("cap", C.c_int32), ("skip_src", C.c_int32), ("n_cfg", C.c_int32),
                ("cfg", C.POINTER(uniap_config)), ("n_skip", C.c_int32), ("skip_srcs", _P32)]


class uniap_result(C.Structure):
    _fields_ = [("objective", C.c_int64), ("cfg_index", C.c_int32), ("deg", C.c_int32), ("c", C.c_int32),
                ("L", C.c_int32), ("stage_of", C.c_int32 * MAX_L), ("strategy_of", C.c_int32 * MAX_L),
                ("stage_cost", C.c_int64 * MAX_L), ("cut_cost", C.c_int64 * MAX_L),
                ("stage_mem", C.c_int32 * MAX_L), ("cfg_objective", _P64), ("quantum_ns", C.c_int64),
                ("dp_cells", C.c_uint64), ("dp_relax", C.c_uint64), ("dp_cells_canonical", C.c_uint64),
                ("ms_gpu_dp", C.c_double),
                ("ms_gpu_total", C.c_double), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("n_launches", C.c_uint32), ("n_k2_launches", C.c_uint32)]


class uniap_layer(C.Structure):
    _fields_ = [("fwd_ns_per_sample", _P64), ("param_bytes", C.c_int64), ("act_bytes_per_sample", _P64),
                ("ctx_bytes", C.c_int64), ("tp_comm_bytes_per_sample", C.c_int64)]


class uniap_edge(C.Structure):
    _fields_ = [("src", C.c_int32), ("dst", C.c_int32), ("tensor_bytes_per_sample", C.c_int64),
                ("reshard_ns_per_sample", _P64), ("cut_ns_per_sample", _P64)]


class uniap_cluster(C.Structure):
    _fields_ = [("n_dev", C.c_int32), ("node_size", C.c_int32), ("mem_bytes", C.c_int64),
                ("mem_reserve_bytes", C.c_int64), ("bw_intra_Bps", C.c_int64), ("bw_inter_Bps", C.c_int64),
                ("p2p_Bps", C.c_int64), ("lat_ns", C.c_int64), ("ccoc_permille", C.c_int32),
                ("dev_mem_bytes", _P64)]


class uniap_model(C.Structure):
    _fields_ = [("L", C.c_int32), ("layers", C.POINTER(uniap_layer)), ("n_edges", C.c_int32),
                ("edges", C.POINTER(uniap_edge))]


class uniap_options(C.Structure):
    _fields_ = [("B", C.c_int32), ("precision", C.c_int32), ("Q", C.c_int32), ("quantum_ns", C.c_int64),
                ("cand", _P32), ("n_cand", C.c_int32), ("strategy_space", C.c_int32), ("schedule", C.c_int32)]


class uniap_record(C.Structure):
    _fields_ = [("objective", C.c_int64), ("cfg_index", C.c_int32), ("deg", C.c_int32), ("c", C.c_int32),
                ("L", C.c_int32), ("status", C.c_int32), ("n_cfg_local", C.c_int32),
                ("stage_of", C.c_int32 * MAX_L), ("strategy_of", C.c_int32 * MAX_L),
                ("stage_cost", C.c_int64 * MAX_L), ("cut_cost", C.c_int64 * MAX_L),
                ("stage_mem", C.c_int32 * MAX_L), ("dp_cells", C.c_uint64), ("dp_relax", C.c_uint64),
                ("dp_cells_canonical", C.c_uint64)]


RECORD_BYTES = C.sizeof(uniap_record)

EXPORTS = ("uniap_create", "uniap_destroy", "uniap_last_error", "uniap_status_string", "uniap_version",
           "uniap_solve_tables", "uniap_interval_table", "uniap_plan", "uniap_build_tables", "uniap_prepare",
           "uniap_prepare_tables", "uniap_run", "uniap_run_phase", "uniap_plan_shard", "uniap_fetch", "uniap_shard_assign", "uniap_shard_tables",
           "uniap_pick", "uniap_selftest", "uniap_fetch_intervals",
           "uniap_candidates", "uniap_catalogue")

_lib = None


def lib():
    """Load libuniap.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python build.py` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        H = C.c_void_p
        L.uniap_create.argtypes = [C.POINTER(H), C.c_int, C.c_void_p]
        L.uniap_destroy.argtypes = [H]
        L.uniap_destroy.restype = None
        L.uniap_last_error.argtypes = [H]
        L.uniap_last_error.restype = C.c_char_p
        L.uniap_status_string.argtypes = [C.c_int]
        L.uniap_status_string.restype = C.c_char_p
        L.uniap_version.restype = C.c_char_p
        L.uniap_solve_tables.argtypes = [H, C.POINTER(uniap_tables), C.POINTER(uniap_result)]
        L.uniap_interval_table.argtypes = [H, C.POINTER(uniap_tables), C.c_int32, _P32]
        L.uniap_plan.argtypes = [H, C.POINTER(uniap_model), C.POINTER(uniap_cluster), C.POINTER(uniap_options),
                                 C.POINTER(uniap_result)]
        L.uniap_build_tables.argtypes = [H, C.POINTER(uniap_model), C.POINTER(uniap_cluster),
                                         C.POINTER(uniap_options), _P32, C.c_int64, _P64, _P32, _P32, _P64]
        L.uniap_prepare.argtypes = [H, C.POINTER(uniap_model), C.POINTER(uniap_cluster), C.POINTER(uniap_options)]
        L.uniap_prepare_tables.argtypes = [H, C.POINTER(uniap_tables)]
        L.uniap_run.argtypes = [H, C.c_int32, C.c_int32, C.c_void_p]
        L.uniap_run_phase.argtypes = [H, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]
        L.uniap_plan_shard.argtypes = [H, C.POINTER(uniap_model), C.POINTER(uniap_cluster), C.POINTER(uniap_options),
                                       C.c_int32, C.c_int32, C.c_void_p]
        L.uniap_fetch.argtypes = [H, C.POINTER(uniap_result)]
        L.uniap_fetch_intervals.argtypes = [H, _P32, C.c_int64, _P64]
        L.uniap_shard_assign.argtypes = [H, C.c_int32, _P32]
        L.uniap_shard_tables.argtypes = [C.POINTER(uniap_tables), C.c_int32, _P32]
        L.uniap_pick.argtypes = [C.POINTER(uniap_record), C.c_int32, C.POINTER(uniap_result)]
        L.uniap_candidates.argtypes = [C.c_int32, C.c_int32, _P32, C.c_int32]
        L.uniap_catalogue.argtypes = [C.c_int32, C.c_int32, _P32, C.c_int32]
        L.uniap_selftest.argtypes = [_P32, _P32, _P32]
        for f in EXPORTS:
            if f not in ("uniap_destroy", "uniap_last_error", "uniap_status_string", "uniap_version"):
                getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


class UniapError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"uniap status {status}: {msg}")
        self.status = status


def _i32(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _p32(a):
    return None if a is None else a.ctypes.data_as(_P32)


def _tables(t):
    keep = []
    L = t["L"]
    cfgs = (uniap_config * len(t["cfgs"]))()
    for i, c in enumerate(t["cfgs"]):
        S = c["n_strat"]
        A = _i32(c["A"]).reshape(L, S)
        M = _i32(c["M"]).reshape(L, S) if c.get("M") is not None else None
        R = _i32(c["R"]).reshape(L - 1, S, S) if L > 1 else np.zeros((1, S, S), np.int32)
        Rs = _i32(c["Rskip"]).reshape(L, S, S) if c.get("Rskip") is not None else None
        O = _i32(c["O"]).reshape(L - 1) if c.get("O") is not None and L > 1 else None
        SC = _i32(c["stage_cap"]).reshape(c["deg"]) if c.get("stage_cap") is not None else None
        RC = _i32(c["Rcut"]).reshape(L - 1, S, S) if c.get("Rcut") is not None and L > 1 else None
        MS = _i32(c["M_stage"]).reshape(c["deg"], L, S) if c.get("M_stage") is not None else None
        srcs = t.get("skip_srcs") or []
        RSS = _i32(c["Rskips"]).reshape(len(srcs), L, S, S) if c.get("Rskips") is not None and srcs else None
        keep += [A, M, R, Rs, O, SC, RC, MS, RSS]
        cfgs[i] = uniap_config(c["deg"], c["c"], S, _p32(A), _p32(M), _p32(R), _p32(Rs), _p32(O), _p32(SC),
                               _p32(RC), _p32(MS), _p32(RSS))
    keep.append(cfgs)
    srcs = _i32(t.get("skip_srcs") or [0])
    keep.append(srcs)
    return uniap_tables(L, t["cap"], t.get("skip_src", -1), len(t["cfgs"]), cfgs, len(t.get("skip_srcs") or []),
                        _p32(srcs)), keep


_LAYER_DT = np.dtype([("fwd", np.uint64), ("param", np.int64), ("act", np.uint64), ("ctx", np.int64),
                      ("tpc", np.int64)])
_EDGE_DT = np.dtype([("src", np.int32), ("dst", np.int32), ("bytes", np.int64), ("mat", np.uint64),
                     ("cut", np.uint64)])


def _profile(p):
    """Marshal a profile dict into the ABI structs (vectorised: one numpy
    array per field, the struct arrays filled column-wise)."""
    m = p["model"]
    L = m["L"]
    ls = m["layers"]
    fwd = np.ascontiguousarray([ly["fwd_ns_per_sample"] for ly in ls], dtype=np.int64)
    act = np.ascontiguousarray([ly["act_bytes_per_sample"] for ly in ls], dtype=np.int64)
    assert C.sizeof(uniap_layer) == _LAYER_DT.itemsize and C.sizeof(uniap_edge) == _EDGE_DT.itemsize
    lay = np.zeros(L, _LAYER_DT)
    lay["fwd"] = fwd.ctypes.data + np.arange(L, dtype=np.uint64) * np.uint64(fwd.strides[0])
    lay["act"] = act.ctypes.data + np.arange(L, dtype=np.uint64) * np.uint64(act.strides[0])
    lay["param"] = [ly["param_bytes"] for ly in ls]
    lay["ctx"] = [ly["ctx_bytes"] for ly in ls]
    lay["tpc"] = [ly["tp_comm_bytes_per_sample"] for ly in ls]
    E = len(m["edges"])
    ed = np.zeros(max(E, 1), _EDGE_DT)
    mats = []
    if E:
        ed["src"] = [e["src"] for e in m["edges"]]
        ed["dst"] = [e["dst"] for e in m["edges"]]
        ed["bytes"] = [e["tensor_bytes_per_sample"] for e in m["edges"]]
        for i, e in enumerate(m["edges"]):  # optional per-edge matrices (uniap_edge)
            for key, col in (("reshard_ns_per_sample", "mat"), ("cut_ns_per_sample", "cut")):
                if e.get(key) is not None:
                    mat = np.ascontiguousarray(e[key], dtype=np.int64).reshape(-1)
                    mats.append(mat)
                    ed[col][i] = mat.ctypes.data
    cl = p["cluster"]
    dm = None
    if cl.get("dev_mem_bytes") is not None:  # optional per-device memory (heterogeneous devices)
        dm = np.ascontiguousarray(cl["dev_mem_bytes"], dtype=np.int64)
        mats.append(dm)
    cluster = uniap_cluster(cl["n_dev"], cl["node_size"], cl["mem_bytes"], cl["mem_reserve_bytes"],
                            cl["bw_intra_Bps"], cl["bw_inter_Bps"], cl["p2p_Bps"], cl["lat_ns"],
                            cl["ccoc_permille"], None if dm is None else dm.ctypes.data_as(_P64))
    o = p["options"]
    cand = None
    if o.get("cand"):
        cand = np.ascontiguousarray(np.array(o["cand"], dtype=np.int32).reshape(-1))
    opts = uniap_options(o["B"], o["precision"], o["Q"], o.get("quantum_ns", 0), _p32(cand),
                         0 if cand is None else len(cand) // 2, o.get("strategy_space", 0), o.get("schedule", 0))
    keep = [fwd, act, lay, ed, cand, mats]
    model = uniap_model(L, C.cast(lay.ctypes.data, C.POINTER(uniap_layer)), E,
                        C.cast(ed.ctypes.data, C.POINTER(uniap_edge)))
    return model, cluster, opts, keep


class Profile:
    """A profile marshalled once into the ABI structs (uniap_model /
    uniap_cluster / uniap_options over host arrays it owns).  Pass it to
    Handle.prepare / Handle.plan instead of the dict to skip the per-call
    dict -> struct conversion; every call still validates and uploads the
    host arrays (uniap_prepare).  The arrays can be edited in place
    (`fwd`, `act`: int64 [L][1+log2 n]) between calls."""

    def __init__(self, p):
        self.model, self.cluster, self.opts, self.keep = _profile(p)
        self.fwd, self.act = self.keep[0], self.keep[1]
        o = p["options"]
        self.n_cfg = len(o["cand"]) if o.get("cand") else len(candidates(p["cluster"]["n_dev"], o["B"]))


def _structs(p):
    if isinstance(p, Profile):
        return p.model, p.cluster, p.opts, p.keep, p.n_cfg
    model, cluster, opts, keep = _profile(p)
    o = p["options"]
    n = len(o["cand"]) if o.get("cand") else len(candidates(p["cluster"]["n_dev"], o["B"]))
    return model, cluster, opts, keep, n


def _result_dict(r, n_cfg, cfg_obj):
    # (slicing a ctypes array yields a list of Python ints)
    deg = r.deg
    L = r.L
    out = {"objective": r.objective, "cfg_index": r.cfg_index, "deg": deg, "c": r.c,
           "quantum_ns": r.quantum_ns, "dp_cells": r.dp_cells, "dp_relax": r.dp_relax,
           "dp_cells_canonical": r.dp_cells_canonical,
           "ms_gpu_dp": r.ms_gpu_dp, "ms_gpu_total": r.ms_gpu_total, "h2d_bytes": r.h2d_bytes,
           "d2h_bytes": r.d2h_bytes, "n_launches": r.n_launches, "n_k2_launches": r.n_k2_launches}
    if cfg_obj is not None:
        out["cfg_objective"] = cfg_obj[:n_cfg]
    if r.objective != INT64_MAX:
        out["stage_of"] = r.stage_of[:L]
        out["strategy_of"] = r.strategy_of[:L]
        out["stage_cost"] = r.stage_cost[:deg]
        out["cut_cost"] = r.cut_cost[:max(deg - 1, 0)]
        out["stage_mem"] = r.stage_mem[:deg]
    return out


def candidates(n, B):
    k = lib().uniap_candidates(n, B, None, 0)
    buf = (C.c_int32 * (2 * k))()
    lib().uniap_candidates(n, B, buf, k)
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(k)]


def selftest():
    """Host-only: every K2 kernel shape the planner can choose is compiled in."""
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    rc = lib().uniap_selftest(C.byref(a), C.byref(b), C.byref(c))
    return rc, (a.value, b.value, c.value)


def catalogue(g, space=0):
    k = lib().uniap_catalogue(g, space, None, 0)
    buf = (C.c_int32 * (3 * max(k, 1)))()
    lib().uniap_catalogue(g, space, buf, k)
    return [tuple(buf[3 * i:3 * i + 3]) for i in range(k)]


def shard_tables(t, world):
    """LPT owner rank of every config of level-1 tables (host only)."""
    tb, keep = _tables(t)
    owner = (C.c_int32 * len(t["cfgs"]))()
    st = lib().uniap_shard_tables(C.byref(tb), world, owner)
    if st != UNIAP_OK:
        raise UniapError(st, "shard_tables")
    return list(owner)


def pick(records: bytes, world: int):
    """uniap_pick over `world` host records (bytes of world * RECORD_BYTES)."""
    arr = (uniap_record * world).from_buffer_copy(records)
    r = uniap_result()
    st = lib().uniap_pick(arr, world, C.byref(r))
    if st not in (UNIAP_OK, UNIAP_ERR_INFEASIBLE):
        raise UniapError(st, "pick")
    r.L = arr[0].L
    return st, _result_dict(r, 0, None)


class Handle:
    """A libuniap handle on one CUDA device (owns its device buffers)."""

    def __init__(self, device=0, stream=None):
        self._h = C.c_void_p()
        st = lib().uniap_create(C.byref(self._h), device, C.c_void_p(stream) if stream else None)
        if st != UNIAP_OK:
            raise UniapError(st, f"uniap_create(device={device}) failed: needs a compute-capability 10.x GPU")
        self.n_cfg = 0
        self.device = device

    def close(self):
        if self._h:
            lib().uniap_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what, ok=(UNIAP_OK,)):
        if st not in ok:
            raise UniapError(st, f"{what}: {lib().uniap_last_error(self._h).decode()}")
        return st

    def solve_tables(self, t):
        tb, keep = _tables(t)
        n = self.n_cfg = len(t["cfgs"])
        cfg_obj = (C.c_int64 * n)()
        r = uniap_result()
        r.cfg_objective = cfg_obj
        st = self._check(lib().uniap_solve_tables(self._h, C.byref(tb), C.byref(r)), "solve_tables",
                         (UNIAP_OK, UNIAP_ERR_INFEASIBLE))
        out = _result_dict(r, n, cfg_obj)
        out["status"] = st
        return out

    def interval_table(self, t, cfg):
        tb, keep = _tables(t)
        L = t["L"]
        P = np.zeros(L * L, dtype=np.int32)
        self._check(lib().uniap_interval_table(self._h, C.byref(tb), cfg, P.ctypes.data_as(_P32)), "interval_table")
        return P.reshape(L, L)

    def plan(self, p):
        """p: a profile dict or a Profile."""
        model, cluster, opts, keep, n = _structs(p)
        self.n_cfg = n
        r, cfg_obj = self._result_buffers(n)
        st = self._check(lib().uniap_plan(self._h, C.byref(model), C.byref(cluster), C.byref(opts), C.byref(r)),
                         "plan", (UNIAP_OK, UNIAP_ERR_INFEASIBLE))
        out = _result_dict(r, n, cfg_obj)
        out["status"] = st
        return out

    def build_tables(self, p):
        """The K1 builder's tables in the documented block layout -> (tables dict, quantum, flat buffer)."""
        model, cluster, opts, keep = _profile(p)
        words, ncfg, skip, qn = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int64()
        self._check(lib().uniap_build_tables(self._h, C.byref(model), C.byref(cluster), C.byref(opts), None, 0,
                                             C.byref(words), C.byref(ncfg), C.byref(skip), C.byref(qn)), "build(size)")
        buf = np.zeros(words.value, dtype=np.int32)
        self._check(lib().uniap_build_tables(self._h, C.byref(model), C.byref(cluster), C.byref(opts),
                                             buf.ctypes.data_as(_P32), words.value, C.byref(words),
                                             C.byref(ncfg), C.byref(skip), C.byref(qn)), "build")
        L, cap = p["model"]["L"], p["options"]["Q"] - 1
        srcs = sorted({e["src"] for e in p["model"]["edges"] if e["dst"] != e["src"] + 1})
        cfgs, off = [], 0
        for _ in range(ncfg.value):
            deg, c, S, g = (int(x) for x in buf[off:off + 4])
            off += 4
            blk = {}
            for name, shape in (("A", (L, S)), ("M", (L, S)), ("R", (L - 1, S, S)), ("Rskip", (L, S, S)),
                                ("O", (L - 1,)), ("stage_cap", (deg,))):
                size = int(np.prod(shape))
                blk[name] = buf[off:off + size].reshape(shape)
                off += size
            has_rcut = int(buf[off])
            off += 1
            blk["Rcut"] = None
            if has_rcut:
                blk["Rcut"] = buf[off:off + (L - 1) * S * S].reshape(L - 1, S, S)
                off += (L - 1) * S * S
            has_ms = int(buf[off])
            off += 1
            blk["M_stage"] = None
            if has_ms:
                blk["M_stage"] = buf[off:off + deg * L * S].reshape(deg, L, S)
                off += deg * L * S
            blk["Rskips"] = None
            if len(srcs) >= 2:  # NEXT-4: each skip source's table at the block's tail
                blk["Rskips"] = buf[off:off + len(srcs) * L * S * S].reshape(len(srcs), L, S, S)
                off += len(srcs) * L * S * S
            cfgs.append({"deg": deg, "c": c, "n_strat": S, "g": g, **blk,
                         "Rskip": blk["Rskip"] if skip.value >= 0 else None})
        t = {"L": L, "cap": cap, "skip_src": skip.value, "cfgs": cfgs}
        if len(srcs) >= 2:
            t["skip_srcs"] = srcs
        return t, qn.value, buf

    # ---- split pipeline ----
    def prepare(self, p):
        """p: a profile dict or a Profile (validated and uploaded on every call)."""
        self._keep = _structs(p)
        model, cluster, opts, _, self.n_cfg = self._keep
        self._check(lib().uniap_prepare(self._h, C.byref(model), C.byref(cluster), C.byref(opts)), "prepare")

    def prepare_tables(self, t):
        tb, keep = _tables(t)
        self._check(lib().uniap_prepare_tables(self._h, C.byref(tb)), "prepare_tables")
        self.n_cfg = len(t["cfgs"])

    def run(self, rank=0, world=1, rec_dev_ptr=None):
        self._check(lib().uniap_run(self._h, rank, world, C.c_void_p(rec_dev_ptr) if rec_dev_ptr else None), "run")

    def plan_shard(self, p, rank, world, rec_dev_ptr):
        """uniap_plan_shard: this rank's LPT share of Algorithm 1 (prepare + run),
        its best record into the device buffer at rec_dev_ptr."""
        self._keep = _structs(p)
        model, cluster, opts, _, self.n_cfg = self._keep
        self._check(lib().uniap_plan_shard(self._h, C.byref(model), C.byref(cluster), C.byref(opts), rank, world,
                                           C.c_void_p(rec_dev_ptr)), "plan_shard")

    def run_phase(self, rank, world, rec_dev_ptr, phase, recs_dev_ptr=None):
        """uniap_run_phase: 1 = up to this rank's local winner (record header),
        2 = the traceback on the rank holding the global winner of the gathered
        phase-1 records (device array of `world` records)."""
        self._check(lib().uniap_run_phase(self._h, rank, world, C.c_void_p(rec_dev_ptr), phase,
                                          C.c_void_p(recs_dev_ptr) if recs_dev_ptr else None), f"run_phase({phase})")

    def _result_buffers(self, n):
        """A result struct and its per-config array, kept per handle (reused)."""
        if getattr(self, "_res", (None,))[0] != n:
            cfg_obj = (C.c_int64 * max(n, 1))()
            r = uniap_result()
            r.cfg_objective = cfg_obj
            self._res = (n, r, cfg_obj)
        return self._res[1], self._res[2]

    def fetch(self):
        r, cfg_obj = self._result_buffers(self.n_cfg)
        st = self._check(lib().uniap_fetch(self._h, C.byref(r)), "fetch", (UNIAP_OK, UNIAP_ERR_INFEASIBLE))
        out = _result_dict(r, self.n_cfg, cfg_obj)
        out["status"] = st
        return out

    def plan_distributed(self, p, group=None):
        """Multi-GPU plan, one process per GPU: this rank runs
        its LPT share of the candidate configs on its device up to its local
        winner (uniap_run_phase 1), writing the record header into a device
        buffer; the headers are all_gathered over the process group (NCCL over
        NVLink: the device buffers directly; gloo: through host memory); phase 2
        runs the traceback only on the rank holding the global winner; a
        second all_gather of the fixed-size records and uniap_pick on the host.
        (world = 1: one uniap_run.)  Returns the picked result dict (every
        rank gets the same) plus this rank's local per-config optima.  torch
        supplies only the memory and the process group."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.prepare(p)
        dev = torch.device("cuda", self.device)
        # persistent record buffers: the captured graphs keep their pointers
        if getattr(self, "_dist_bufs", (None,))[0] != world:
            self._dist_bufs = (world, torch.zeros(RECORD_BYTES, dtype=torch.uint8, device=dev),
                               torch.zeros(world * RECORD_BYTES, dtype=torch.uint8, device=dev))
        _, rec, allr = self._dist_bufs
        nccl = dist.get_backend(group) == "nccl"

        def gather():
            if nccl:
                dist.all_gather_into_tensor(allr, rec, group=group)
                torch.cuda.current_stream(dev).synchronize()
            else:
                parts = [torch.empty(RECORD_BYTES, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, rec.cpu(), group=group)
                allr.copy_(torch.cat(parts))
            return allr

        if world == 1:
            self.run(rank, world, rec.data_ptr())
        else:
            self.run_phase(rank, world, rec.data_ptr(), 1)
            self.fetch()  # synchronises the handle's stream: the header is complete
            hdrs = gather()
            self.run_phase(rank, world, rec.data_ptr(), 2, hdrs.data_ptr())
        local = self.fetch()  # synchronises the handle's stream: rec is complete
        host = gather().cpu().numpy().tobytes()
        st, out = pick(host, world)
        out["status"] = st
        out["cfg_objective_local"] = local.get("cfg_objective")
        out["quantum_ns"] = local["quantum_ns"]
        return out

    def fetch_intervals(self):
        """The last run's interval tables, flat: per config, one L*L block per
        cap level (uniap_fetch_intervals; UNIAP_INF = infeasible or not needed)."""
        n = C.c_int64()
        self._check(lib().uniap_fetch_intervals(self._h, None, 0, C.byref(n)), "fetch_intervals(size)")
        P = np.zeros(n.value, dtype=np.int32)
        self._check(lib().uniap_fetch_intervals(self._h, P.ctypes.data_as(_P32), P.size, None), "fetch_intervals")
        return P

    def shard_assign(self, world):
        owner = (C.c_int32 * max(self.n_cfg, 1))()
        self._check(lib().uniap_shard_assign(self._h, world, owner), "shard_assign")
        return list(owner[:self.n_cfg])
