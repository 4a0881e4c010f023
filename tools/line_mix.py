"""Per-CUDA-line warp instructions executed / stall samples of one kernel from
`ncu -i rep --page source --csv --print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out = []
for r in rows[3:]:
    if r and r[0] and r[0].isdigit() and len(r) > 8:
        f = lambda x: int(x) if x.isdigit() else 0
        out.append((f(r[7]), f(r[4]), int(r[0]), r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
st = sum(o[1] for o in out) or 1
for n, s, ln, src in sorted(out, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{n:9d} {100*n/tot:5.1f}% stall {100*s/st:5.1f}%  L{ln:<4} {src}")
