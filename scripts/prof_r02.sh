#!/bin/bash
# Round-2 profile: parity subset, C3 per-pass timing, ncu full captures (source
# level) of the C3 passes and of the C2 kernel.
# Usage: gpurun -- 'bash scripts/prof_r02.sh <tag>'
set -u
TAG=${1:-r02g}
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/prof_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "16384 or 2048 or 4096 or fourstep or c3 or golden or largest" > $OUT/pytest_$TAG.txt 2>&1; tail -2 $OUT/pytest_$TAG.txt >> $S
for c in c3 c2; do
  echo "$c $(timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
done
timeout 600 python scripts/sweep.py --dims 1 --sizes 14 19 20 21 22 --reps 10 >> $S 2>&1
timeout 600 python scripts/sweep.py --dims 2 --sizes 11 12 --reps 10 >> $S 2>&1
for c in c3 c2; do
  case $c in c2) sk=3; n=1;; c3) sk=6; n=2;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s $sk -c $n -o $OUT/prof_${c}_$TAG -f \
     python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-nested > $OUT/ncu_full_${c}_$TAG.log 2>&1
  ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page raw --csv > $OUT/prof_${c}_$TAG.raw.csv 2>/dev/null
  ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/prof_${c}_$TAG.src.csv 2>/dev/null
done
cat $S
du -sh $OUT
