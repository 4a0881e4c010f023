"""GPipe vs synchronous 1F1B memory (NEXT-2, reading A-32) on the five bench
workloads and the Llama variants: the optimal objective (time per
iteration in quanta and in ms), the plan (deg, c) and the device time of the
solve, through the library (GPU).  usage: python tools/schedule_compare.py [out.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles  # noqa: E402

h = pkg.Handle(0)
rows = []
for w in ("bert", "t5", "vit", "swin", "llama", "llama-envc", "llama13b"):
    p = profiles.make_profile(w)
    row = {"workload": w}
    for sch in (0, 1):
        q = dict(p, options=dict(p["options"], schedule=sch))
        for _ in range(3):
            r = h.plan(q)
        row["gpipe" if sch == 0 else "1f1b"] = {
            "objective": r["objective"], "tpi_ms": r["objective"] * r["quantum_ns"] / 1e6 if r["objective"] < (1 << 62) else None,
            "deg": r["deg"], "c": r["c"], "ms_gpu_total": round(r["ms_gpu_total"], 4), "dp_relax": r["dp_relax"]}
    rows.append(row)
    print(json.dumps(row), flush=True)
h.close()
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
