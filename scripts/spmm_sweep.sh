#!/bin/bash
# SpMM sweep (1 GPU) over env overrides: DG_SPMM_MINB (CTAs/SM), DG_SPMM_E
# (entries per step), DG_SPMM_TWO (two-level fp32 accumulation), DG_SPMM_STG
# (entries staged in shared memory by cp.async); lane shape DG_SPMM_FORCE_G/CPL
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
O=gpurun_out/spmm_sweep_stg.txt
: > $O
DG_SPMM_STG=1 DG_SPMM_MINB=4 DG_SPMM_E=2 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 >> $O
for cfg in "0 0 0 0" "3 4 0 1" "4 2 0 1" "4 2 1 1" "3 4 1 1"; do
  set -- $cfg
  echo "== MINB=$1 E=$2 TWO=$3 STG=$4" >> $O
  export DG_SPMM_MINB=$1 DG_SPMM_E=$2 DG_SPMM_TWO=$3 DG_SPMM_STG=$4
  timeout 600 python scripts/prof_spmm.py --f 602 100 --reps 5 >> $O 2>&1
  DG_SPMM_FORCE_G=8 DG_SPMM_FORCE_CPL=1 timeout 600 python scripts/prof_spmm.py --f 41 --reps 5 >> $O 2>&1
  timeout 600 python scripts/prof_spmm.py --workload products --community --f 100 --reps 5 >> $O 2>&1
done
grep -v "^\[bench\]\|community-ordered" $O
