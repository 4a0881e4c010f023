#!/bin/bash
# A/B of library variants over the bench workloads (run from the repo root on
# the GPU box): VARIANTS="base:. exp:variants/exp" (each a directory holding a
# built copy of the repo, see tools/mkvariant.sh); ROUNDS alternating passes.
mkdir -p gpurun_out
OUT=$PWD/gpurun_out
for R in $(seq 1 ${ROUNDS:-1}); do
  for V in ${VARIANTS:-base:.}; do
    name=${V%%:*}; dir=${V#*:}
    for W in ${WORKLOADS:-llama t5 swin vit bert}; do
      (cd $dir && timeout 300 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline \
        > $OUT/ab_${name}_${W}_r$R.json 2> $OUT/ab_${name}_${W}_r$R.err)
    done
  done
done
python - <<'PY'
import glob, json, os
for f in sorted(glob.glob("gpurun_out/ab_*_r*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f)[3:-5].ljust(28), "ms %.4f" % d["ms_per_step"], "k2 %.4f" % d["roofline"]["k2_ms_per_step"],
              "frac %.3f" % d["roofline"]["frac"], "e2e %.4f" % (1e3 * d["e2e"]["seconds_per_step"]), d["objective"])
    except Exception as e:
        print(f, "ERR", e)
PY
