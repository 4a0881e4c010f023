#!/bin/bash
# Round-2 closing measurement session (1 GPU), refreshed after the lone-chain
# clusters and the parallel K5a plan: bench lines, reference arm, GPU tests,
# smoke, fake world, host timing, traces, per-class rates, launch lists.
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for W in llama t5 swin vit bert; do
  timeout 900 python bench.py --steps 20 --warmup 3 --workload $W > $O/bench_$W.json 2> $O/bench_$W.err
done
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for W in llama bert; do timeout 300 python tools/host_overhead.py $W > $O/host_$W.json 2>&1; done
timeout 600 python tools/fake_world.py $O/fake_world.json > $O/fake_world.txt 2>&1
for W in llama t5 swin vit bert; do timeout 120 python tools/k2_trace.py $W > $O/trace_$W.txt 2>&1; done
timeout 300 python tools/k2_class_rate.py llama t5 swin vit bert > $O/class_rate.txt 2>&1
for W in llama t5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$W.csv \
    python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > /dev/null 2>&1
done
