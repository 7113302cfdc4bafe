#!/bin/bash
# SpMM sweep (1 GPU): CTAs/SM (DG_SPMM_MINB), entries per step (DG_SPMM_E),
# two-level fp32 accumulation (DG_SPMM_TWO); lane shape (DG_SPMM_FORCE_G/CPL)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
O=gpurun_out/spmm_sweep_acc.txt
: > $O
for cfg in "0 0 0" "4 2 0" "4 2 1" "3 4 1" "3 2 1" "4 4 1"; do
  set -- $cfg
  echo "== MINB=$1 E=$2 TWO=$3" >> $O
  DG_SPMM_MINB=$1 DG_SPMM_E=$2 DG_SPMM_TWO=$3 timeout 600 python scripts/prof_spmm.py --f 602 100 --reps 5 >> $O 2>&1
  DG_SPMM_MINB=$1 DG_SPMM_E=$2 DG_SPMM_TWO=$3 DG_SPMM_FORCE_G=8 DG_SPMM_FORCE_CPL=1 timeout 600 python scripts/prof_spmm.py --f 41 --reps 5 >> $O 2>&1
  DG_SPMM_MINB=$1 DG_SPMM_E=$2 DG_SPMM_TWO=$3 timeout 600 python scripts/prof_spmm.py --workload products --community --f 100 --reps 5 >> $O 2>&1
done
grep -v "^\[bench\]\|community-ordered" $O
