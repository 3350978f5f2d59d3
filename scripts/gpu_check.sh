#!/bin/bash
# One GPU round: parity tests, bench lines, ncu launch list + one full capture.
# Usage (from the build container): gpurun -- 'bash scripts/gpu_check.sh [tag]'
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.txt
tail -3 $OUT/pytest_gpu_$TAG.txt
for c in c2 c1 c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $( [ $c != c2 ] && echo --no-cpu ) > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err
  cat $OUT/bench_${c}_$TAG.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_ref_$TAG.json 2>&1; cat $OUT/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c2_$TAG.csv \
   python bench.py --config c2 --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 4 -c 1 -o $OUT/prof_c2_$TAG -f \
   python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > $OUT/ncu_full_c2_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 4 -c 2 -o $OUT/prof_c4_$TAG -f \
   python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu_full_c4_$TAG.log 2>&1
ls -la $OUT
