#!/bin/bash
# round 2: GPU tests, measured DPX peak, sanitizer logs, A/B vs the previous commit
mkdir -p gpurun_out/san
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2d.log
timeout 300 python tools/alu_peak.py 3 > gpurun_out/alu_peak_r2.json 2>&1; cp MEASURED_ALU.json gpurun_out/ 2>/dev/null
python tools/sanitize_cases.py toy > /dev/null 2>&1  # warm the oracle build
for tool in memcheck racecheck synccheck; do
  for c in toy bert cluster skip; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py $c > gpurun_out/san/${tool}_$c.log 2>&1
    echo "rc=$?" >> gpurun_out/san/${tool}_$c.log
  done
done
ROUNDS=2 VARIANTS="base:variants/base new:." bash tools/gpu_ab.sh > gpurun_out/ab_r2d.txt 2>&1
