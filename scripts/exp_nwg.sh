#!/bin/bash
# Experiment: three-stage strided 2048 / 4096 passes and 4 warpgroups for
# one-CTA-per-SM passes.  Usage: gpurun -- 'bash scripts/exp_nwg.sh <tag>'
set -u
TAG=${1:-nwg}
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_$TAG.txt; : > $S
export TCFFT_EXPERIMENTS=1
TCFFT_STRIDED_R64=0 TCFFT_NWG=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "2048 or 4096 or 16384 or c3 or fourstep or largest" > $OUT/pytest_$TAG.txt 2>&1; tail -2 $OUT/pytest_$TAG.txt >> $S
run() {
  echo "== $*" >> $S
  echo "c3 $(env "$@" timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  env "$@" timeout 300 python scripts/sweep.py --dims 1 --sizes 14 19 20 21 22 --reps 10 | python -c 'import json,sys; print("1d", [(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])' >> $S
  env "$@" timeout 300 python scripts/sweep.py --dims 2 --sizes 11 12 --reps 10 | python -c 'import json,sys; print("2d", [(d["nx"], d["roofline_frac"]) for d in map(json.loads, sys.stdin)])' >> $S
}
for rnd in 1 2; do
run TCFFT_X=0
run TCFFT_STRIDED_R64=0
run TCFFT_STRIDED_R64=0 TCFFT_NWG=4
run TCFFT_NWG=1
run TCFFT_ONEBUF=0 TCFFT_NWG=4
done
cat $S
