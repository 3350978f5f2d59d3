#!/bin/bash
# Quick GPU check after a kernel change: strided / multi-pass parity subset,
# headline configs, C5 sweep of the multi-pass and one-CTA-per-SM shapes.
# Usage: gpurun -- 'bash scripts/quick_r02.sh <tag> [pytest -k expr]'
set -u
TAG=${1:-q}
K=${2:-"16384 or 2048 or 4096 or fourstep or c3 or c4 or golden or largest or strided or 512"}
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/quick_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_batched_tensor.py -q -x -k "$K" > $OUT/pytest_$TAG.txt 2>&1; tail -2 $OUT/pytest_$TAG.txt >> $S
for c in c3 c4 c2 c1; do
  echo "$c $(timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
done
timeout 600 python scripts/sweep.py --dims 1 --sizes 14 15 17 19 20 21 22 23 24 --reps 10 >> $S 2>&1
timeout 600 python scripts/sweep.py --dims 2 --sizes 9 10 11 12 --reps 10 >> $S 2>&1
cat $S
