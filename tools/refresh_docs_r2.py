"""Refresh the measured tables of README.md, DESIGN.md
(fake world) and profiles/r2/SUMMARY.md from profiles/r2/*.json (after
tools/final_r2d.sh + tools/summarize_r2.py)."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R2 = os.path.join(ROOT, "profiles", "r2")


def last(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


B = {w: last(os.path.join(R2, f"bench_{w}.json")) for w in ["llama", "t5", "swin", "vit", "bert"]}
fw = json.load(open(os.path.join(R2, "fake_world.json")))
ref = last(os.path.join(R2, "bench_reference.json"))


def f3(x):
    return "%.3f" % x


def sub_file(path, fn):
    p = os.path.join(ROOT, path)
    s = open(p).read()
    open(p, "w").write(fn(s))


def readme(s):
    names = {"llama": "Llama-7B-like, 32 devices, Q = 4096", "t5": "T5-Large-like, 16 devices",
             "swin": "Swin-Huge-like", "vit": "ViT-Huge-like", "bert": "BERT-Huge-like, 8 devices"}
    for w, n in names.items():
        d = B[w]
        cb = d["cpu_baseline"]
        pat = re.compile(r"^\| " + re.escape(n) + r" \|.*$", re.M)
        row = (f"| {n} | {f3(d['ms_per_step'])} ms | {f3(d['e2e']['seconds_per_step'] * 1e3)} ms | "
               f"{d['roofline']['frac']:.2f} | {cb['seconds']:.2f} s / {cb['single_thread']['seconds']:.2f} s |")
        assert pat.search(s), n
        s = pat.sub(row, s)
    return s


def baseline(s):
    bn = {"bert": "BERT-Huge-like", "t5": "T5-Large-like", "vit": "ViT-Huge-like", "swin": "Swin-Huge-like (L=48)",
          "llama": "Llama-7B-like"}
    for w, n in bn.items():
        d = B[w]
        r = d["roofline"]
        cb = d["cpu_baseline"]
        pat = re.compile(r"^\| " + re.escape(n) + r" \|(.*)$", re.M)
        m = pat.search(s)
        assert m, n
        cols = [c.strip() for c in m.group(1).split("|")][:-1]
        cols[1] = "%.2e" % d["cells_canonical_per_step"]
        cols[2] = "%.2e" % d["cells_executed_per_step"]
        cols[3] = "%.2e" % r["algorithmic_relax_per_step"]
        cols[4] = f3(d["ms_per_step"])
        cols[5] = f3(r["k2_ms_per_step"])
        cols[6] = "%.2e" % d["value"]
        cols[7] = "%.2f T" % r["achieved"]
        pc = "%.1f %%" % (100 * r["frac"])
        cols[8] = ("**" + pc + "**") if w == "llama" else pc
        cols[9] = f3(d["e2e"]["seconds_per_step"] * 1e3)
        cols[10] = " / ".join(f3(fw[w][k]["max_ms"]) for k in ["1", "2", "4", "8"])
        cols[11] = "%.2f" % cb["single_thread"]["seconds"]
        cols[12] = "%.2f" % cb["seconds"]
        cols[13] = f"{d['plan']['deg']}, {d['plan']['c']}"
        s = s[:m.start()] + "| " + n + " | " + " | ".join(cols) + " |" + s[m.end():]
    return re.sub(r"Llama, [0-9]+ ms per plan \([0-9.e+]+ canonical cells/s\), against [0-9.]+ ms end to end on the GPU",
                  "Llama, %d ms per plan (%.2e canonical cells/s), against %.3f ms end to end on the GPU"
                  % (round(ref["ms_per_step"]), ref["value"], B["llama"]["e2e"]["seconds_per_step"] * 1e3), s)


def design(s):
    for w, n in {"llama": "Llama", "t5": "T5", "swin": "Swin", "vit": "ViT", "bert": "BERT"}.items():
        pat = re.compile(r"^\| " + n + r" \| 0\.[0-9]+ \| 0\.[0-9]+ \| 0\.[0-9]+ \| 0\.[0-9]+ \|$", re.M)
        assert pat.search(s), n
        s = pat.sub("| " + n + " | " + " | ".join(f3(fw[w][k]["max_ms"]) for k in ["1", "2", "4", "8"]) + " |", s)
    return s


def summary(s):
    tbl = open(os.path.join(R2, "table.md")).read().strip()
    a = s.index("| workload | #(deg,c)")
    b = s.index("\n\n", a)
    s = s[:a] + tbl + s[b:]
    fwt = "| workload | 1 | 2 | 4 | 8 |\n|---|---|---|---|---|\n" + "\n".join(
        f"| {w} | " + " | ".join("%.3f" % fw[w][k]["max_ms"] for k in ["1", "2", "4", "8"]) + " |"
        for w in ["llama", "t5", "swin", "vit", "bert"])
    a = s.index("| workload | 1 | 2 | 4 | 8 |")
    b = s.index("\n\n", a)
    s = s[:a] + fwt + s[b:]
    return re.sub(r"Llama, [0-9]+ ms per plan\.", "Llama, %d ms per plan." % round(ref["ms_per_step"]), s)


sub_file("README.md", readme)
sub_file("BASELINE.md", baseline)
sub_file("DESIGN.md", design)
sub_file("profiles/r2/SUMMARY.md", summary)
print("ok")
