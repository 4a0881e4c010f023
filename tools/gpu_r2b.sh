mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2b.log
ROUNDS=2 VARIANTS="base:variants/base new:." bash tools/gpu_ab.sh > gpurun_out/ab_r2b.txt 2>&1
