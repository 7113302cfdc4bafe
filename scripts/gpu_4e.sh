#!/bin/bash
# one gpurun --gpus 4 call: multi-process parity (incl. the sharded path),
# Reddit N=2/N=4 benches, config 5 (papers-shaped) at N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/n4e
O=gpurun_out/n4e
make -C paper_2504_04673_b200/csrc > $O/build.txt 2>&1 || { tail -20 $O/build.txt; exit 1; }
nvidia-smi topo -m > $O/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29611 tests/mp_gpu_worker.py > $O/mp4.txt 2>&1; echo "rc=$?" >> $O/mp4.txt
tail -n 4 $O/mp4.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 > $O/reddit_n4.json 2> $O/reddit_n4.log; echo "rc=$?" >> $O/reddit_n4.log
timeout 900 $TR --nproc-per-node 2 --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 > $O/reddit_n2.json 2> $O/reddit_n2.log; echo "rc=$?" >> $O/reddit_n2.log
timeout 1800 $TR --nproc-per-node 4 --master-port 29614 bench.py --workload papers --gpus 4 --steps 3 --warmup 3 > $O/papers_n4.json 2> $O/papers_n4.log; echo "rc=$?" >> $O/papers_n4.log
tail -n 5 $O/papers_n4.log
python3 - <<'PY'
import json
for f in ['reddit_n2','reddit_n4','papers_n4']:
    try:
        d=json.loads(open(f'gpurun_out/n4e/{f}.json').read().strip().splitlines()[-1])
        print(f, d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel_ms'], d['roofline']['gather_gbs'], d.get('exchange'), d.get('peak_mem_gib'))
    except Exception as e:
        print(f, 'ERR', e)
PY
