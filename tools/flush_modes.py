"""How the L2 flush between timed steps changes one plan's step time (GPU box):
no flush; bench.py's 256 MiB memset; the memset followed by a 256 MiB read
of another buffer (the memset's dirty lines written back before the timed
region); a read-only flush.  Events as bench.py records them, medians."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import profiles  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "llama"
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
h = pkg.Handle(0, s.cuda_stream)
h.prepare(pkg.Profile(profiles.make_profile(w)))
modes = {"none": lambda: None, "memset": lambda: fl.zero_(),
         "memset+read": lambda: (fl.zero_(), rd.sum()), "read": lambda: rd.sum()}
res = {}
for _ in range(2):
    for name, pre in modes.items():
        for _ in range(5):
            h.run()
        out = []
        for _ in range(60):
            pre()
            torch.cuda.synchronize()
            e0.record(s)
            h.run()
            e1.record(s)
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e3)
        res[name] = round(statistics.median(out), 1)
    print(json.dumps(res | {"workload": w}))
