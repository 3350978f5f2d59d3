#!/bin/bash
# C3 scheduling variants: chunk tickets, PDL trigger point, ticketed tail length
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_c3misc.txt; : > $S
export TCFFT_EXPERIMENTS=1
for rnd in 1 2; do
for v in "TCFFT_X=0" "TCFFT_DYNAMIC=0" "TCFFT_DYNAMIC=1" "TCFFT_PDL=2" "TCFFT_PDL=0" "TCFFT_DYN_TAIL=4" "TCFFT_LATE_WAIT=0"; do
  echo "$v $(env $v timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
done
done
cat $S
