#!/bin/bash
# C1 variants (A/B of experiment hooks on the C1 bench line): CTAs per SM for small row chunks
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_c1.txt; : > $S
export TCFFT_EXPERIMENTS=1
TCFFT_SMALL_CTAS=6 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "small or c1 or golden or impulse or tone" > $OUT/pytest_c1.txt 2>&1; echo "parity (6): $(tail -1 $OUT/pytest_c1.txt)" >> $S
for rnd in 1 2; do
for v in "TCFFT_SMALL_CTAS=4" "TCFFT_SMALL_CTAS=5" "TCFFT_SMALL_CTAS=6"; do
  echo "$v $(env $v timeout 300 python bench.py --config c1 --steps 64 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')" >> $S
done
done
cat $S
