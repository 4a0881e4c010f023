#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2h.log
ROUNDS=2 VARIANTS="head:variants/head new:." bash tools/gpu_ab.sh > gpurun_out/ab_r2h.txt 2>&1
WORKLOADS="llama bert" VARIANTS="head:variants/head new:." bash tools/gpu_tr.sh
