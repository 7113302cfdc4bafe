#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout 600 python scripts/prof_spmm.py --f 602 16 41 --reps 3 --cusparse > gpurun_out/cusparse.txt 2>&1
timeout 300 python scripts/prof_spmm.py --f 602 --reps 1 > gpurun_out/plain602.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v2_602 python scripts/prof_spmm.py --f 602 --reps 1 > gpurun_out/ncu602.log 2>&1
timeout 300 python scripts/prof_spmm.py --f 16 --reps 1 > gpurun_out/plain16.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v2_16 python scripts/prof_spmm.py --f 16 --reps 1 > gpurun_out/ncu16.log 2>&1
cat gpurun_out/cusparse.txt | grep "f="
