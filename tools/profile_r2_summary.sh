set -x
for W in llama t5; do
  WORKLOAD=$W bash tools/profile_r2.sh
  python tools/ncu_summary.py gpurun_out/ncu_summary_$W.json $W gpurun_out/prof_k2_$W.ncu-rep gpurun_out/prof_rest_$W.ncu-rep > gpurun_out/ncu_summary_$W.log 2>&1
  ncu -i gpurun_out/prof_k2_$W.ncu-rep --page source --csv > /dev/null 2>&1
  rm -f gpurun_out/prof_*_$W.ncu-rep
done
