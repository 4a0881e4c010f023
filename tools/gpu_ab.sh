#!/bin/bash
# A/B of env knob variants over every bench workload: VARIANTS="name:ENV=val,ENV2=val name2:..."
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q --maxfail=10 > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for V in ${VARIANTS:-base:X=0}; do
  name=${V%%:*}; envs=${V#*:}
  for W in ${WORKLOADS:-llama t5 swin vit bert}; do
    env ${envs//,/ } timeout 300 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ab_${name}_$W.json 2> gpurun_out/ab_${name}_$W.err
  done
done
python - <<'PY'
import glob, json, os
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f)[3:-5].ljust(24), "ms %.4f" % d["ms_per_step"], "k2 %.4f" % d["roofline"]["k2_ms_per_step"],
              "frac %.3f" % d["roofline"]["frac"], "e2e %.4f" % (1e3 * d["e2e"]["seconds_per_step"]), d["objective"])
    except Exception as e:
        print(f, "ERR", e)
PY
