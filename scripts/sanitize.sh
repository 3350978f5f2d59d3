#!/bin/bash
# compute-sanitizer over every pass-kernel family (scripts/sanitize.py)
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  q=""; [ $tool != memcheck ] && q="--quick"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py $q > $OUT/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/sanitize_$tool.txt | tail -1) $(grep -c '^ok' $OUT/sanitize_$tool.txt) cases"
done
# C1 latency floor probe (tests/native/c1_floor.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/c1_floor tests/native/c1_floor.cu && /tmp/c1_floor > $OUT/c1_floor.txt 2>&1; cat $OUT/c1_floor.txt
