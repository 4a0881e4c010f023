#!/bin/bash
# iteration session: GPU tests, bench on every workload, launch list (+ optional full ncu of K2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for W in ${WORKLOADS:-llama bert t5 vit swin}; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
W=${NCU_WORKLOAD:-llama}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > /dev/null 2>&1
if [ -n "$NCU_FULL" ]; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$NCU_FULL -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-6} \
    -o gpurun_out/prof_$W python bench.py --steps 1 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ncu_full_$W.log 2>&1
fi
