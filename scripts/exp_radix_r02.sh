#!/bin/bash
# Radix-order A/B for the one-pass 1D 8192 / 16384 rows (TCFFT_RADICES_<n>):
# parity of each variant against the reference restatement, then the C5 sweep point.
# Usage: gpurun -- 'bash scripts/exp_radix_r02.sh <tag>'
set -u
TAG=${1:-rx}
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/exp_radix_$TAG.txt; : > $S
chk() {  # n
python - "$1" <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2104_11471_b200 as tc
from oracle import restate as R
n = int(sys.argv[1]); b = 8
x = R.random_pairs([5, n], b, n)
t = torch.from_numpy(x).cuda(); tc.execute(tc.plan_1d(n, b), t); y = R.to_complex(t.cpu().numpy())
ref = R.to_complex(R.fft_half(x))
print("relL2 vs reference %.3e" % max(R.rel_l2(y[i], ref[i]) for i in range(b)), end=" ")
PY
}
for r in 16,32,32 64,16,16 32,16,32 16,16,64 16,32,32; do
  echo "16384 [$r] $(TCFFT_EXPERIMENTS=1 TCFFT_RADICES_16384=$r chk 16384) $(TCFFT_EXPERIMENTS=1 TCFFT_RADICES_16384=$r timeout 300 python scripts/sweep.py --dims 1 --sizes 14 --reps 20 --no-cpu | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms"], d["roofline_frac"])')" >> $S
done
for r in 16,16,32 32,16,16 16,32,16 64,16,8 16,16,32; do
  echo "8192 [$r] $(TCFFT_EXPERIMENTS=1 TCFFT_RADICES_8192=$r chk 8192) $(TCFFT_EXPERIMENTS=1 TCFFT_RADICES_8192=$r timeout 300 python scripts/sweep.py --dims 1 --sizes 13 --reps 20 --no-cpu | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms"], d["roofline_frac"])')" >> $S
done
cat $S
