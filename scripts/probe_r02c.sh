#!/bin/bash
# single-buffer (two CTAs/SM) 16384-element passes: parity + timing
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/probe_r02c.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "16384 or 2048 or 4096 or c3 or c4 or c2" > $OUT/pytest_r02c.txt 2>&1; tail -3 $OUT/pytest_r02c.txt >> $S
export TCFFT_EXPERIMENTS=1
for v in 1 0; do
  echo "onebuf=$v sweep $(TCFFT_ONEBUF=$v timeout 300 python scripts/sweep.py --dims 1 --sizes 14 --reps 10 | tr '\n' ' ')" >> $S
  echo "onebuf=$v sweep $(TCFFT_ONEBUF=$v timeout 300 python scripts/sweep.py --dims 2 --sizes 11 12 --reps 10 | tr '\n' ' ')" >> $S
  echo "onebuf=$v 2pass16k $(TCFFT_ONEBUF=$v TCFFT_THREE_PASS=0 TCFFT_SCHUNK_2048=16384 TCFFT_RCHUNK_2048=16384 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
done
TCFFT_THREE_PASS=0 TCFFT_SCHUNK_2048=16384 TCFFT_RCHUNK_2048=16384 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "4194304 or c3" >> $S 2>&1
cat $S
