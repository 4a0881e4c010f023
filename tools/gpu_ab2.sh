#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plan_parity.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_gpu_ab2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ab2.log
ROUNDS=2 VARIANTS="base:variants/base new:." bash tools/gpu_ab.sh > gpurun_out/ab_ab2.txt 2>&1
for W in llama t5; do timeout 120 python tools/k2_trace.py $W > gpurun_out/trace_new_$W.txt 2>&1; done
