#!/bin/bash
# SpMM occupancy sweep (1 GPU): CTAs/SM target and lane shape via env overrides
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
O=gpurun_out/spmm_sweep_minb.txt
: > $O
for mb in 0 3 4; do
  echo "== MINB=$mb default shape" >> $O
  DG_SPMM_MINB=$mb timeout 600 python scripts/prof_spmm.py --f 602 41 100 --reps 5 >> $O 2>&1
  echo "== MINB=$mb G=8 CPL=1" >> $O
  DG_SPMM_MINB=$mb DG_SPMM_FORCE_G=8 DG_SPMM_FORCE_CPL=1 timeout 600 python scripts/prof_spmm.py --f 41 --reps 5 >> $O 2>&1
done
grep -v "^\[bench\]" $O
