"""Writes tests/golden/*.json by calling ONLY oracle/ (the brute force).

Run from the repo root:  python tests/golden/make_golden.py
The toy instance is SURVEY.md Sec. 8c-P ("Frozen golden"); its expected keys
were derived there by brute force over every stage-and-strategy assignment,
and this script re-derives them with oracle/brute.py (Eqs. 2-8 literally).
They are NOT printed in the paper (the paper gives no worked numeric example
of Eq. 2 beyond its symbols).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from gen import tables  # noqa: E402
from oracle import brute  # noqa: E402


def main():
    t = tables.toy_tables()
    per_cfg = []
    for cfg in t["cfgs"]:
        f, so, sk = brute.solve_cfg(t, cfg)
        per_cfg.append({"deg": cfg["deg"], "c": cfg["c"], "objective": f, "stage_of": so, "strategy_of": sk})
    glob = {}
    for name, cands in (("grid", tables.TOY_GRID), ("algorithm1", [(1, 1), (2, 2)])):
        r = brute.solve_tables(tables.toy_tables(cands))
        glob[name] = {"objective": r["objective"], "deg": r["deg"], "c": r["c"],
                      "stage_of": r["stage_of"], "strategy_of": r["strategy_of"]}
    out = {"source": "SURVEY.md Sec. 8c-P frozen toy; derived by oracle/brute.py (Eqs. 2-8, PAPER.md:122-202)",
           "per_config": per_cfg, "global": glob}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "toy.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
