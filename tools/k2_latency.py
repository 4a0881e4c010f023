"""Per-layer latency of K2 sweeps: single-config tables solved on the GPU.
Prints one JSON line per case (device ms of the K2 phase, per-layer us)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import tables  # noqa: E402

h = pkg.Handle(0)
for (deg, S, Q, L) in [(1, 21, 4096, 32), (1, 15, 4096, 32), (1, 15, 1024, 48), (1, 10, 1024, 32),
                       (2, 15, 4096, 32), (2, 10, 1024, 32), (4, 10, 4096, 32), (8, 6, 4096, 32)]:
    t = tables.large_random_tables(1, L, [S], Q - 1, [(deg, 2)], mem_max=max(1, (2 * Q) // L))
    h.prepare_tables(t)
    best = 1e9
    for _ in range(8):
        h.run()
        r = h.fetch()
        best = min(best, r["ms_gpu_dp"])
    print(json.dumps({"deg": deg, "S": S, "Q": Q, "L": L, "k2_ms": best, "us_per_layer": 1000 * best / L,
                      "relax": r["dp_relax"], "Trelax_s": r["dp_relax"] / best / 1e9}), flush=True)
