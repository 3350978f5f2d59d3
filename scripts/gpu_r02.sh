#!/bin/bash
# Round-2 GPU check: parity tests, smoke, headline bench (C3 + nested), reference arm.
# Usage: gpurun -- 'bash scripts/gpu_r02.sh <tag> [tests|bench|ref|all]'
set -u
TAG=${1:-r02}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu_$TAG.txt 2>&1
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu_$TAG.txt 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.txt
  tail -25 $OUT/pytest_gpu_$TAG.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; tail -2 $OUT/smoke_$TAG.txt
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
  cat $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
fi
if [[ $WHAT == all || $WHAT == ref ]]; then
  ( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
  cat $OUT/bench_ref_$TAG.json; tail -4 $OUT/bench_ref_$TAG.err
fi
