"""Strategy-space ablation on the five synthetic workloads (PAPER.md:476-477,
Fig. 6): unified vs intra-only vs inter-dp vs
inter-pp (gen/ablation.py, reading A-25).  Tables from the GPU builder (K1),
each variant solved on the GPU through the C ABI and by the oracle (the two
must agree); prints one JSON line per (workload, variant) with the optimum as
time per iteration (Eq. 2) in seconds.  usage: python tools/ablation.py [W ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import ablation, profiles  # noqa: E402
from oracle import oracle  # noqa: E402

INT64_MAX = (1 << 63) - 1
h = pkg.Handle(0)
for w in (sys.argv[1:] or ["bert", "t5", "vit", "swin", "llama"]):
    p = profiles.make_profile(w)
    t, qn, _ = h.build_tables(p)
    n = p["cluster"]["n_dev"]
    base = None
    for v in ablation.VARIANTS:
        tv = ablation.restrict(t, v, n)
        line = {"workload": w, "variant": v, "n_dev": n, "B": p["options"]["B"], "quantum_ns": qn}
        if not tv["cfgs"]:
            line.update({"objective": None, "note": "no candidate in this space"})
            print(json.dumps(line), flush=True)
            continue
        got = h.solve_tables(tv)
        t0 = time.perf_counter()
        for _ in range(5):
            got = h.solve_tables(tv)
        gpu_ms = (time.perf_counter() - t0) / 5 * 1e3
        t0 = time.perf_counter()
        want = oracle.solve_tables(tv, n_threads=0)
        orc_s = time.perf_counter() - t0
        same = all(got[k] == want[k] for k in ("objective", "deg", "c")) and (
            want["objective"] == INT64_MAX or (got["stage_of"] == want["stage_of"]
                                               and got["strategy_of"] == want["strategy_of"]))
        obj = got["objective"]
        line.update({"objective": None if obj == INT64_MAX else obj,
                     "tpi_s": None if obj == INT64_MAX else obj * qn / 1e9,
                     "deg": got["deg"], "c": got["c"], "oracle_agrees": same,
                     "gpu_solve_ms_wall": round(gpu_ms, 3), "oracle_s": round(orc_s, 3)})
        if obj != INT64_MAX:
            if v == "unified":
                base = obj
            line["vs_unified"] = round(obj / base, 4) if base else None
            line["strategies_used"] = sorted(set(got["strategy_of"]))
        else:
            line["note"] = "SOL x: no feasible strategy (memory)"
        print(json.dumps(line), flush=True)
h.close()
