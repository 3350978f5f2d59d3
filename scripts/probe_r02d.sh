#!/bin/bash
# blocked two-pass 2^19..2^22: parity + timing (vs three-pass), onebuf A/B of the rowTB pass
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/probe_r02d.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fourstep or c3 or golden or largest or 16384" > $OUT/pytest_r02d.txt 2>&1; tail -3 $OUT/pytest_r02d.txt >> $S
export TCFFT_EXPERIMENTS=1
for rnd in 1 2; do
for v in "TCFFT_BLOCKED=1" "TCFFT_BLOCKED=1 TCFFT_ONEBUF=0" "TCFFT_BLOCKED=0"; do
  echo "$v c3 $(env $v timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  echo "$v sweep $(env $v timeout 300 python scripts/sweep.py --dims 1 --sizes 19 20 21 22 --reps 10 | python -c 'import json,sys; print([ (d["nx"], d["roofline_frac"], d["gflops_5nlogn"]) for d in map(json.loads, sys.stdin)])')" >> $S
done
done
cat $S
