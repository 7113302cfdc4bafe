#!/bin/bash
# SpMM occupancy / pipeline-depth sweep (1 GPU) via env overrides
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
O=gpurun_out/spmm_sweep_e.txt
: > $O
for cfg in "0 4" "3 4" "2 6" "2 8"; do
  set -- $cfg
  echo "== MINB=$1 E=$2" >> $O
  DG_SPMM_MINB=$1 DG_SPMM_E=$2 timeout 600 python scripts/prof_spmm.py --f 602 100 41 --reps 5 >> $O 2>&1
  echo "== MINB=$1 E=$2 G=8 CPL=1" >> $O
  DG_SPMM_MINB=$1 DG_SPMM_E=$2 DG_SPMM_FORCE_G=8 DG_SPMM_FORCE_CPL=1 timeout 600 python scripts/prof_spmm.py --f 41 --reps 5 >> $O 2>&1
done
grep -v "^\[bench\]" $O
