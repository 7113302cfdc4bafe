#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python scripts/prof_spmm.py --f 602 16 41 --slab 0 32 64 128 256 --acc 1 0 > gpurun_out/sweep.txt 2>&1
timeout 300 python scripts/prof_spmm.py --f 602 --reps 1 > gpurun_out/plain602.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_rows -s 1 -c 1 -o gpurun_out/prof_spmm602 python scripts/prof_spmm.py --f 602 --reps 1 > gpurun_out/ncu602.log 2>&1
timeout 300 python scripts/prof_spmm.py --f 16 --reps 1 > gpurun_out/plain16.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_rows -s 1 -c 1 -o gpurun_out/prof_spmm16 python scripts/prof_spmm.py --f 16 --reps 1 > gpurun_out/ncu16.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt; cat gpurun_out/sweep.txt | grep "f="
