#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 tests/mp_gpu_worker.py > gpurun_out/mp_worker.txt 2>&1; echo "rc=$?" >> gpurun_out/mp_worker.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.log; echo "rc=$?" >> gpurun_out/bench_n2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.log; echo "rc=$?" >> gpurun_out/bench_n1.log
tail -5 gpurun_out/mp_worker.txt; tail -3 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/bench_n2.log; tail -2 gpurun_out/bench_n1.log
