#!/bin/bash
# compute-sanitizer over every kernel family (incl. 1F1B and DAG copies)
mkdir -p gpurun_out/final/san
O=gpurun_out/final
for tool in memcheck racecheck synccheck; do
  for c in toy bert cluster skip levels cut 1f1b dag; do
    timeout 500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py $c > $O/san/${tool}_$c.log 2>&1
    echo "rc=$?" >> $O/san/${tool}_$c.log
  done
done
