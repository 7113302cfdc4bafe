#!/bin/bash
# gpurun --gpus 4: N=2 and N=4 benches with the current kernels (Reddit, products, papers)
cd "$(dirname "$0")/.."
O=gpurun_out/n4g; mkdir -p $O
make -C paper_2504_04673_b200/csrc > $O/build.txt 2>&1 || { tail -20 $O/build.txt; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29611 tests/mp_gpu_worker.py > $O/mp4.txt 2>&1; echo "rc=$?" >> $O/mp4.txt
grep -a "checked\|FAIL\|rc=" $O/mp4.txt | head -6
timeout 900 $TR --nproc-per-node 2 --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 > $O/reddit_n2.json 2> $O/reddit_n2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 > $O/reddit_n4.json 2> $O/reddit_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29615 bench.py --workload products --gpus 4 --steps 10 --warmup 3 > $O/products_n4.json 2> $O/products_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29616 bench.py --gpus 4 --ranks-per-gpu 2 --steps 10 --warmup 3 > $O/reddit_n4_p8.json 2> $O/reddit_n4_p8.log
timeout 1800 $TR --nproc-per-node 4 --master-port 29614 bench.py --workload papers --gpus 4 --steps 3 --warmup 3 > $O/papers_n4.json 2> $O/papers_n4.log
python3 - <<'PY'
import json
for f in ['reddit_n2','reddit_n4','reddit_n4_p8','products_n4','papers_n4']:
    try:
        d=json.loads(open(f'gpurun_out/n4g/{f}.json').read().strip().splitlines()[-1])
        print(f, d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel_ms'], (d.get('exchange') or {}).get('frac'), d.get('epoch_breakdown_ms'))
    except Exception as e:
        print(f, 'ERR', e)
PY
