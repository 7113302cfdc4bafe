#!/bin/bash
# gpurun --gpus 4: the round's multi-GPU measurements with the current kernels
cd "$(dirname "$0")/.."
O=gpurun_out/final4; mkdir -p $O
make -C paper_2504_04673_b200/csrc > $O/build.txt 2>&1 || { tail -20 $O/build.txt; exit 1; }
nvidia-smi topo -m > $O/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() { local name=$1 np=$2; shift 2; timeout 1800 $TR --nproc-per-node $np --master-port $((29600 + RANDOM % 300)) bench.py "$@" > $O/$name.json 2> $O/$name.log; echo "$name rc=$?"; }
timeout 900 $TR --nproc-per-node 4 --master-port 29611 tests/mp_gpu_worker.py > $O/mp4.txt 2>&1; echo "mp4 rc=$?"
run reddit_n2 2 --gpus 2 --steps 10 --warmup 3
run reddit_n4 4 --gpus 4 --steps 10 --warmup 3
run reddit_n4_p8 4 --gpus 4 --ranks-per-gpu 2 --steps 10 --warmup 3
run reddit_n4_p8_15d_c2 4 --gpus 4 --ranks-per-gpu 2 --c 2 --variant 15d-sparse --steps 10 --warmup 3 --no-transform-first
run products_n4 4 --workload products --gpus 4 --steps 10 --warmup 3
run products_n4_gvb 4 --workload products --partition gvb --gpus 4 --steps 10 --warmup 3 --no-transform-first
run products_n4_gvb_obl 4 --workload products --partition gvb --variant 1d-oblivious --gpus 4 --steps 10 --warmup 3 --no-transform-first
run products_p8_gvb_15d_c2 4 --workload products --partition gvb --ranks-per-gpu 2 --c 2 --variant 15d-sparse --gpus 4 --steps 10 --warmup 3 --no-transform-first
run products_p16_gvb_15d_c4 4 --workload products --partition gvb --ranks-per-gpu 4 --c 4 --variant 15d-sparse --gpus 4 --steps 10 --warmup 3 --no-transform-first
run papers_n4 4 --workload papers --gpus 4 --steps 5 --warmup 3
python3 - <<'PY'
import json, glob, os
for f in sorted(glob.glob('gpurun_out/final4/*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel_ms'], (d.get('exchange') or {}).get('frac'), d['comm_elements_per_epoch']['ratio'])
    except Exception as e:
        print(f, 'ERR', e)
PY
