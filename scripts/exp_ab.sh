#!/bin/bash
# Generic A/B of experiment variables: parity under the B setting, then
# headline configs + C5 sweep for each setting, two rounds.
# Usage: gpurun -- 'bash scripts/exp_ab.sh <tag> "<A env>" "<B env>" ...'
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_$TAG.txt; : > $S
export TCFFT_EXPERIMENTS=1
last="${@: -1}"
env $last timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_batched_tensor.py -q -x > $OUT/pytest_$TAG.txt 2>&1; echo "parity ($last): $(tail -1 $OUT/pytest_$TAG.txt)" >> $S
run() {
  echo "== $1" >> $S
  for c in c3 c4 c2 c1; do
  echo "$c $(env $1 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  done
  env $1 timeout 300 python scripts/sweep.py --dims 1 --sizes 8 12 14 15 17 19 20 21 22 23 24 --reps 10 | python -c 'import json,sys; print("1d", [(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])' >> $S
  env $1 timeout 300 python scripts/sweep.py --dims 2 --sizes 8 9 10 11 12 --reps 10 | python -c 'import json,sys; print("2d", [(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])' >> $S
}
for rnd in 1 2; do
  for v in "$@"; do run "$v"; done
done
cat $S
