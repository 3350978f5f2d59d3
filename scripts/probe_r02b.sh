#!/bin/bash
# round-2 probes: L2 promotion of strided boxes, two-pass C3, 1-CTA/SM profile
set -u
OUT=gpurun_out; mkdir -p $OUT
export TCFFT_EXPERIMENTS=1
S=$OUT/probe_r02b.txt; : > $S
for rnd in 1 2; do
for v in 0 128 256; do
  for c in c3 c4; do
    echo "promo=$v $c $(TCFFT_L2PROMO=$v timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  done
  echo "promo=$v sweep $(TCFFT_L2PROMO=$v timeout 300 python scripts/sweep.py --dims 2 --sizes 11 12 --reps 10 | tr '\n' ' ')" >> $S
  # two-pass C3 variants
  echo "promo=$v 2pass16k $(TCFFT_L2PROMO=$v TCFFT_THREE_PASS=0 TCFFT_SCHUNK_2048=16384 TCFFT_RCHUNK_2048=16384 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  echo "promo=$v 2pass8k $(TCFFT_L2PROMO=$v TCFFT_THREE_PASS=0 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
done
done
cat $S
# 1-CTA/SM kernel source-level profile (1D 16384 x 8192)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 3 -c 1 -o $OUT/prof_1d16k_r02b -f \
   python scripts/sweep.py --dims 1 --sizes 14 --reps 2 > $OUT/ncu_1d16k.log 2>&1
ncu -i $OUT/prof_1d16k_r02b.ncu-rep --page source --csv --print-source sass > $OUT/prof_1d16k_r02b.src.csv 2>/dev/null
ncu -i $OUT/prof_1d16k_r02b.ncu-rep --page raw --csv > $OUT/prof_1d16k_r02b.raw.csv 2>/dev/null
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > $OUT/bench_ref_r02b.json 2> $OUT/bench_ref_r02b.err
cat $OUT/bench_ref_r02b.json; tail -4 $OUT/bench_ref_r02b.err
