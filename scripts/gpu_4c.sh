#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node=4 --master-port 29621 tests/mp_gpu_worker.py > gpurun_out/mp4.txt 2>&1; echo "rc=$?" >> gpurun_out/mp4.txt
run() { name=$1; shift; timeout 900 $TR --nproc-per-node=$N --master-port $((29630 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/c_$name.json 2> gpurun_out/c_$name.log; echo "rc=$?" >> gpurun_out/c_$name.log; }
N=4 run reddit_n4
N=2 run reddit_n2
N=1 run reddit_n1
N=4 run products_n4 --workload products
for f in gpurun_out/c_*.log; do echo "$f: $(tail -n 1 $f)"; done
