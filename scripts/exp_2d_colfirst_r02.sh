#!/bin/bash
# 2D columns-first two-pass plan (TCFFT_2D_COLFIRST=1, plan.cpp build_2d_colfirst)
# vs the row-first plan: 2D parity subset under the new plan, then the C5 2D
# sweep points and C4 both ways (twice).  Usage: gpurun -- 'bash scripts/exp_2d_colfirst_r02.sh <tag>'
set -u
TAG=${1:-cf}
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_2d_colfirst_$TAG.txt; : > $S
TCFFT_EXPERIMENTS=1 TCFFT_2D_COLFIRST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "2d or c4 or golden" > $OUT/pytest_cf_$TAG.txt 2>&1; tail -2 $OUT/pytest_cf_$TAG.txt >> $S
for i in 1 2; do
  for cf in 0 1; do
    echo "colfirst=$cf c4 $(TCFFT_EXPERIMENTS=1 TCFFT_2D_COLFIRST=$cf timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"], d["roofline"]["per_pass_ms"])')" >> $S
    TCFFT_EXPERIMENTS=1 TCFFT_2D_COLFIRST=$cf timeout 300 python scripts/sweep.py --dims 2 --sizes 9 10 11 12 13 14 --reps 10 --no-cpu | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('colfirst=$cf', d['nx'], d['ny'], d['ms'], d['roofline_frac'])" >> $S
  done
done
cat $S
