#!/bin/bash
# compute-sanitizer over the risky kernels (scripts/sanitize.py); logs into gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
for case in fused claim tc stream chol; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --kernel-name regex:'ocsc|k_' --print-limit 20 \
      python scripts/sanitize.py $case > gpurun_out/sanitize_${case}_${tool}.log 2>&1
    echo "$case $tool exit $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${case}_${tool}.log | head -2 | tr '\n' ' ')"
  done
done
