#!/bin/bash
# One GPU round: parity tests, bench lines, ncu launch list + full captures.
# Usage (from the build container): gpurun -- 'bash scripts/gpu_check.sh [tag] [quick]'
set -u
TAG=${1:-r01}
MODE=${2:-full}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu_$TAG.txt 2>&1
if [ "$MODE" != "benchonly" ]; then
  timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.txt 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.txt
  tail -3 $OUT/pytest_gpu_$TAG.txt
fi
for c in c2 c1 c3 c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $( [ $c != c2 ] && echo --no-cpu ) > $OUT/bench_${c}_$TAG.json 2> $OUT/bench_${c}_$TAG.err
  cat $OUT/bench_${c}_$TAG.json
done
[ "$MODE" == "quick" ] && exit 0
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_ref_$TAG.json 2>&1; cat $OUT/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c2_$TAG.csv \
   python bench.py --config c2 --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
for c in c2 c1 c3 c4; do
  n=2; [ $c == c2 ] && n=1; [ $c == c1 ] && n=1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c $n -o $OUT/prof_${c}_$TAG -f \
     python bench.py --config $c --steps 2 --warmup 3 --no-cpu > $OUT/ncu_full_${c}_$TAG.log 2>&1
done
ls -la $OUT | tail -30
