"""K2 forward-phase device time of single-config tables (tolerates a failed
traceback, for timing-only experiment flags).  usage: python tools/k2_lat4.py TAG"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_16375_b200 as pkg  # noqa: E402
from paper_2307_16375_b200 import binding as b  # noqa: E402
from gen import tables  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
h = pkg.Handle(0)
for (deg, S, Q, L) in [(1, 21, 4096, 32), (1, 15, 1024, 48), (1, 10, 1024, 32), (2, 15, 4096, 32)]:
    t = tables.large_random_tables(1, L, [S], Q - 1, [(deg, 2)], mem_max=max(1, (2 * Q) // L))
    h.prepare_tables(t)
    best = 1e9
    for _ in range(8):
        h.run()
        r = b.uniap_result()
        b.lib().uniap_fetch(h._h, C.byref(r))
        if r.ms_gpu_dp > 0:
            best = min(best, r.ms_gpu_dp)
    print(json.dumps({"tag": tag, "deg": deg, "S": S, "Q": Q, "L": L, "k2_us": round(1000 * best, 1),
                      "us_per_layer": round(1000 * best / L, 3)}), flush=True)
