"""Per-layer K2 latency of chain configs (deg=1 whole-chain sweeps and friends).
usage: python tools/k2_lat3.py TAG   (knobs via UNIAP_K2_* env vars; one JSON line per case)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import tables  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
h = pkg.Handle(0)
for (deg, S, Q, L) in [(1, 15, 1024, 48), (2, 15, 1024, 48), (1, 21, 4096, 32), (2, 21, 4096, 32), (1, 10, 1024, 32)]:
    t = tables.large_random_tables(1, L, [S], Q - 1, [(deg, 2)], mem_max=max(1, (2 * Q) // L))
    h.prepare_tables(t)
    best = 1e9
    for _ in range(8):
        h.run()
        r = h.fetch()
        best = min(best, r["ms_gpu_dp"])
    print(json.dumps({"tag": tag, "deg": deg, "S": S, "Q": Q, "L": L, "k2_us": round(1000 * best, 1),
                      "us_per_layer": round(1000 * best / L, 3),
                      "relax": r["dp_relax"], "Trelax_s": round(r["dp_relax"] / best / 1e9, 3)}), flush=True)
