#!/bin/bash
# dual-context 16384-element passes: smoke with a short timeout, parity, timing vs TCFFT_DUAL=0
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$OUT/probe_r02e.txt; : > $S
timeout 120 python -c "
import torch, paper_2104_11471_b200 as tc
for a in [(16384,None,4),(2048,2048,1),(1<<22,None,1)]:
    x=(torch.rand((a[2], a[0]*(a[1] or 1), 2), device='cuda')*2-1).half()
    p=tc.plan_1d(a[0],a[2]) if a[1] is None else tc.plan_2d(a[0],a[1],a[2])
    tc.execute(p,x); torch.cuda.synchronize(); print('ok',a, torch.isfinite(x.float()).all().item(), flush=True)
" >> $S 2>&1
echo "smoke rc=$?" >> $S
grep -q "smoke rc=0" $S || { cat $S; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_batched_tensor.py -q -x -k "16384 or 2048 or 4096 or fourstep or c3 or golden or largest or strided" > $OUT/pytest_r02e.txt 2>&1; tail -3 $OUT/pytest_r02e.txt >> $S
export TCFFT_EXPERIMENTS=1
for rnd in 1 2; do
for v in "TCFFT_DUAL=1" "TCFFT_DUAL=0"; do
  echo "$v c3 $(env $v timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e --no-nested | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["per_pass_frac"])')" >> $S
  echo "$v sweep $(env $v timeout 300 python scripts/sweep.py --dims 1 --sizes 14 19 20 21 22 --reps 10 | python -c 'import json,sys; print([ (d["nx"], d["roofline_frac"], d["gflops_5nlogn"]) for d in map(json.loads, sys.stdin)])')" >> $S
  echo "$v sweep2d $(env $v timeout 300 python scripts/sweep.py --dims 2 --sizes 11 12 --reps 10 | python -c 'import json,sys; print([ (d["nx"], d["roofline_frac"], d["gflops_5nlogn"]) for d in map(json.loads, sys.stdin)])')" >> $S
done
done
cat $S
