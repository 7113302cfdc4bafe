#!/bin/bash
# one gpurun call: GPU tests, smoke, short benches (each bounded)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --workload rmat14 --steps 5 --warmup 3 > gpurun_out/bench_rmat14.json 2> gpurun_out/bench_rmat14.log; echo "rc=$?" >> gpurun_out/bench_rmat14.log
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_reddit.json 2> gpurun_out/bench_reddit.log; echo "rc=$?" >> gpurun_out/bench_reddit.log
tail -n 3 gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench_rmat14.log gpurun_out/bench_reddit.log
