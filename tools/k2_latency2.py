"""Per-layer K2 latency vs the memory shift size (DSMEM fix-up volume)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import tables  # noqa: E402

h = pkg.Handle(0)
for (deg, S, Q, L) in [(1, 21, 4096, 32), (2, 15, 4096, 32), (4, 10, 4096, 32), (1, 15, 1024, 48)]:
    for mm in (1, 8, 64, 256, 1024):
        t = tables.large_random_tables(1, L, [S], Q - 1, [(deg, 2)], mem_max=mm, forbid_p=0.0)
        h.prepare_tables(t)
        best = 1e9
        for _ in range(6):
            h.run()
            r = h.fetch()
            best = min(best, r["ms_gpu_dp"])
        print(json.dumps({"deg": deg, "S": S, "Q": Q, "L": L, "mem_max": mm, "us_per_layer": 1000 * best / L}), flush=True)
