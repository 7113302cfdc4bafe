#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -n 15 gpurun_out/pytest_gpu.txt
bash scripts/gpu_n1.sh
