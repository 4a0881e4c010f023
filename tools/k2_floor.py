"""Per-layer latency of one long chain (deg = 1, one instance) from the
UNIAP_TRACE timeline: python tools/k2_floor.py  (env selects the K2 class)."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.path.join(tempfile.mkdtemp(), "tr.txt")
os.environ["UNIAP_TRACE"] = path
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import tables  # noqa: E402

h = pkg.Handle(0)
L = 64
for S in (1, 3, 10, 21):
    for Q in (64, 256, 1024, 4096):
        t = tables.large_random_tables(1, L, [S], Q - 1, [(1, 1)], mem_max=max(1, Q // 8), forbid_p=0.0)
        h.prepare_tables(t)
        for _ in range(3):
            h.run()
            h.fetch()
        best = 1e9
        for _ in range(5):
            open(path, "w").close()
            h.run()
            h.fetch()
            recs = [tuple(int(x) for x in ln.split()) for ln in open(path).read().split("\n")[1:] if ln.strip()]
            k2 = [r for r in recs if not r[0] >> 31 and not (r[0] >> 25) & 1]
            best = min(best, max(r[2] - r[1] for r in k2) / 1e3)
        tag = k2[0][0]
        print(json.dumps({"S": S, "Q": Q, "V": (tag >> 6) & 15, "T": ((tag >> 10) & 63) * 32, "C": (tag >> 16) & 31,
                          "us": round(best, 2), "us_per_layer": round(best / (L - 1), 3)}), flush=True)
