#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/tune.txt
for lib in libdgb200.so libdgb200_m2.so libdgb200_m3.so libdgb200_m3e4.so; do
  echo "=== $lib" >> gpurun_out/tune.txt
  DG_LIB_PATH=$PWD/paper_2504_04673_b200/$lib timeout 600 python scripts/prof_spmm.py --f 16 41 --reps 5 >> gpurun_out/tune.txt 2>&1
  for al in 4 32; do
    DG_LIB_PATH=$PWD/paper_2504_04673_b200/$lib timeout 600 python scripts/prof_spmm.py --f 602 --reps 3 --ld-align $al --slab 64 128 256 384 >> gpurun_out/tune.txt 2>&1
  done
done
grep -E "===|f=" gpurun_out/tune.txt
