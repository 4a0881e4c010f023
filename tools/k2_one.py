"""One K2-dominated solve for profiling: python tools/k2_one.py DEG S Q L MEM_MAX"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_16375_b200 as pkg  # noqa: E402
from gen import tables  # noqa: E402

deg, S, Q, L, mm = (int(x) for x in sys.argv[1:6])
h = pkg.Handle(0)
t = tables.large_random_tables(1, L, [S], Q - 1, [(deg, 2)], mem_max=mm, forbid_p=0.0)
h.prepare_tables(t)
for _ in range(3):
    h.run()
    r = h.fetch()
print(r["ms_gpu_dp"])
