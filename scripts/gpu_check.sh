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
for c in c2 c3 c4; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fft_pass --csv \
   --log-file $OUT/launches_${c}_$TAG.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
for c in c2 c1 c3 c4; do
  # skip the warm-up launches: capture every pass of the first timed step
  # (c1 replays a CUDA graph of 64 launches: 64 pre-capture + 3 x 64 warm-up)
  case $c in c2) sk=3; n=1;; c1) sk=256; n=1;; c3) sk=9; n=3;; c4) sk=6; n=2;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s $sk -c $n -o $OUT/prof_${c}_$TAG -f \
     python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_full_${c}_$TAG.log 2>&1
done
# keep the merge-back under gpurun's 64 MiB cap: raw CSV for every capture,
# the .ncu-rep only for the headline config
for c in c2 c1 c3 c4; do
  [ -f $OUT/prof_${c}_$TAG.ncu-rep ] && ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page raw --csv > $OUT/prof_${c}_$TAG.raw.csv 2>/dev/null
  [ $c != c2 ] && rm -f $OUT/prof_${c}_$TAG.ncu-rep
done
du -sh $OUT; ls -la $OUT | tail -30
