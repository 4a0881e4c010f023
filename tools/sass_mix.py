"""Opcode mix (warp-level instructions executed) of one kernel from
`ncu -i rep --page source --csv --print-source sass` output."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ix = {h: i for i, h in enumerate(hdr)}
mix, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr) or r[0] == "Address":
        if r and r[0] == "Kernel Name":
            break
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    mix[op] += n
    tot += n
    stall[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
st = sum(stall.values())
print(f"total warp instr {tot}")
for op, n in mix.most_common(25):
    print(f"{op:12s} {n:12d} {100*n/tot:6.2f}%  stall-samples {100*stall[op]/max(st,1):5.1f}%")
