#!/bin/bash
# round-end style check: GPU tests, smoke, default bench (N=1) and the reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo "rc=$?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.log; echo "rc=$?" >> gpurun_out/bench_reference.log
tail -n 2 gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench_default.log gpurun_out/bench_reference.log
