#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python scripts/prof_spmm.py --f 602 16 41 --slab 0 64 128 256 --acc 1 0 ${SWEEP_ARGS} > gpurun_out/sweep.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt; grep "f=" gpurun_out/sweep.txt
