#!/bin/bash
# compute-sanitizer over scripts/sanitize_case.py; logs to gpurun_out/sanitizer/
OUT=gpurun_out/sanitizer
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python scripts/sanitize_case.py > $OUT/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a $OUT/summary.txt
  tail -3 $OUT/$tool.txt
done
