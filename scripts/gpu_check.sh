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
  # skip the 3 warm-up steps: capture the first timed step's launch(es)
  n=2; sk=6; [ $c == c2 ] && n=1 && sk=3; [ $c == c1 ] && n=1 && sk=6
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s $sk -c $n -o $OUT/prof_${c}_$TAG -f \
     python bench.py --config $c --steps 2 --warmup 3 --no-cpu > $OUT/ncu_full_${c}_$TAG.log 2>&1
done
# keep the merge-back under gpurun's 64 MiB cap: raw CSV for every capture,
# the .ncu-rep only for the headline config
for c in c2 c1 c3 c4; do
  [ -f $OUT/prof_${c}_$TAG.ncu-rep ] && ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page raw --csv > $OUT/prof_${c}_$TAG.raw.csv 2>/dev/null
  [ $c != c2 ] && rm -f $OUT/prof_${c}_$TAG.ncu-rep
done
du -sh $OUT; ls -la $OUT | tail -30
