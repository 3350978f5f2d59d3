#!/bin/bash
# L2 promotion of the strided TMA boxes (TCFFT_L2PROMO 0 / 64 / 128 / 256)
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_promo.txt; : > $S
export TCFFT_EXPERIMENTS=1
for rnd in 1 2; do
for v in 0 64 128 256; do
  echo "promo=$v c3 $(TCFFT_L2PROMO=$v timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  echo "promo=$v $(TCFFT_L2PROMO=$v timeout 300 python scripts/sweep.py --dims 2 --sizes 10 11 12 --reps 10 | python -c 'import json,sys; print([(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])')" >> $S
  echo "promo=$v $(TCFFT_L2PROMO=$v timeout 300 python scripts/sweep.py --dims 1 --sizes 19 20 21 --reps 10 | python -c 'import json,sys; print([(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])')" >> $S
done
done
cat $S
