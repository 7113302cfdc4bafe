#!/bin/bash
# one gpurun call (1 GPU): sharded-path tests, full GPU suite, papers probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_sharded.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_sharded.txt
tail -n 30 gpurun_out/pytest_sharded.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
tail -n 3 gpurun_out/pytest_gpu.txt
timeout 1200 python scripts/papers_probe.py --p ${PROBE_P:-4} --scale ${PROBE_SCALE:-1.0} > gpurun_out/papers_probe.txt 2>&1; echo "rc=$?" >> gpurun_out/papers_probe.txt
tail -n 20 gpurun_out/papers_probe.txt
