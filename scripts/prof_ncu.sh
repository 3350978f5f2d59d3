#!/bin/bash
# ncu --set full (source level) of one bench config; keeps gzipped raw/source
# CSVs (the .ncu-rep is dropped to stay under gpurun's 64 MiB merge-back).
# Usage: gpurun -- 'bash scripts/prof_ncu.sh <tag> <config> <skip> <count> [extra bench args]'
set -u
TAG=$1; c=$2; sk=$3; n=$4; shift 4
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass -s $sk -c $n -o $OUT/prof_${c}_$TAG -f \
   python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-nested "$@" > $OUT/ncu_full_${c}_$TAG.log 2>&1
ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page raw --csv > $OUT/prof_${c}_$TAG.raw.csv 2>/dev/null
ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/prof_${c}_$TAG.src.csv 2>/dev/null
ncu -i $OUT/prof_${c}_$TAG.ncu-rep --page details --csv > $OUT/prof_${c}_$TAG.details.csv 2>/dev/null
rm -f $OUT/prof_${c}_$TAG.ncu-rep
gzip -f $OUT/prof_${c}_$TAG.*.csv
du -sh $OUT
