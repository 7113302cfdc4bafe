#!/bin/bash
# gpurun --gpus 4: config 5 (papers-shaped) at N=4, then products 1D at N=4
cd "$(dirname "$0")/.."
O=gpurun_out/n4p; mkdir -p $O
make -C paper_2504_04673_b200/csrc > $O/build.txt 2>&1 || { tail -20 $O/build.txt; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 $TR --nproc-per-node 4 --master-port 29614 bench.py --workload papers --gpus 4 --steps 5 --warmup 3 > $O/papers_n4.json 2> $O/papers_n4.log; echo "rc=$?" >> $O/papers_n4.log
grep -v "^\[rank[123]\]" $O/papers_n4.log | tail -n 25
[ "$1" = "papers" ] || timeout 900 $TR --nproc-per-node 4 --master-port 29615 bench.py --workload products --gpus 4 --steps 10 --warmup 3 > $O/products_n4.json 2> $O/products_n4.log; echo "rc=$?" >> $O/products_n4.log
python3 - <<'PY'
import json
for f in ['papers_n4','products_n4']:
    try:
        d=json.loads(open(f'gpurun_out/n4p/{f}.json').read().strip().splitlines()[-1])
        print(f, d['value'], d['roofline']['kernel_ms'], d['roofline']['gather_gbs'], d.get('exchange'), d.get('peak_mem_gib'), d.get('epoch_breakdown_ms'))
    except Exception as e:
        print(f, 'ERR', e)
PY
