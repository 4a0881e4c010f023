#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2e.log
ROUNDS=1 VARIANTS="base:variants/base new:." bash tools/gpu_ab.sh > gpurun_out/ab_r2e.txt 2>&1
