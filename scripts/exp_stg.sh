#!/bin/bash
# Experiment: thread-issued output stores (TCFFT_STG_OUT 0 / 1 / 2).
set -u
TAG=${1:-stg}
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_$TAG.txt; : > $S
export TCFFT_EXPERIMENTS=1
for v in 1 2; do
TCFFT_STG_OUT=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_batched_tensor.py -q -x > $OUT/pytest_${TAG}_$v.txt 2>&1; echo "stg=$v $(tail -1 $OUT/pytest_${TAG}_$v.txt)" >> $S
done
run() {
  echo "== $*" >> $S
  for c in c3 c4 c2; do
  echo "$c $(env "$@" timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  done
  env "$@" timeout 300 python scripts/sweep.py --dims 1 --sizes 8 12 14 15 17 19 20 21 22 23 24 --reps 10 | python -c 'import json,sys; print("1d", [(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])' >> $S
  env "$@" timeout 300 python scripts/sweep.py --dims 2 --sizes 8 9 10 11 12 --reps 10 | python -c 'import json,sys; print("2d", [(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])' >> $S
}
for rnd in 1 2; do
run TCFFT_STG_OUT=0
run TCFFT_STG_OUT=1
run TCFFT_STG_OUT=2
done
cat $S
