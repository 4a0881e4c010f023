#!/bin/bash
# iteration session: new-feature GPU tests first, then the whole GPU suite,
# an A/B against variants/base and the per-class rates of the new build
mkdir -p gpurun_out
timeout 600 python -m pytest ${FIRST_TESTS:-tests/test_gpu_split_chain.py} -m gpu -q -x > gpurun_out/pytest_first.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_first.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
ROUNDS=${ROUNDS:-2} VARIANTS="base:variants/base new:." bash tools/gpu_ab.sh > gpurun_out/ab.txt 2>&1
timeout 300 python tools/k2_class_rate.py llama t5 > gpurun_out/rate_new.txt 2>&1
for W in ${TRACE:-llama}; do timeout 120 python tools/k2_trace.py $W > gpurun_out/trace_$W.txt 2>&1; done
