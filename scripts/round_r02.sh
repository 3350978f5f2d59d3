#!/bin/bash
# Round-2 evidence run: C5 sweep, default bench line, per-config ncu launch
# lists and full captures (gzipped CSV).  Usage: gpurun -- 'bash scripts/round_r02.sh <tag>'
set -u
TAG=${1:-r02}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python scripts/sweep.py --dims 1 --sizes 8 9 10 11 12 13 14 15 16 17 18 19 20 21 22 23 24 --reps 10 > $OUT/sweep1d_$TAG.jsonl 2>&1
timeout 900 python scripts/sweep.py --dims 2 --sizes 8 9 10 11 12 --reps 10 > $OUT/sweep2d_$TAG.jsonl 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
for c in c3 c2 c4 c1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fft_pass --csv \
     --log-file $OUT/launches_${c}_$TAG.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-nested > /dev/null 2>&1
done
bash scripts/prof_ncu.sh $TAG c3 6 2
bash scripts/prof_ncu.sh $TAG c2 3 1
bash scripts/prof_ncu.sh $TAG c4 6 2
bash scripts/prof_ncu.sh $TAG c1 256 1
cat $OUT/bench_$TAG.json
du -sh $OUT
