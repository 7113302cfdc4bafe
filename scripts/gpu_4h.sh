#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/n4h; mkdir -p $O
make -C paper_2504_04673_b200/csrc > $O/build.txt 2>&1 || { tail -20 $O/build.txt; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29611 tests/mp_gpu_worker.py > $O/mp4.txt 2>&1; echo "rc=$?" >> $O/mp4.txt
grep -a "checked\|FAIL\|rc=" $O/mp4.txt | head -6
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 1800 $TR --nproc-per-node 4 --master-port 29614 bench.py --workload papers --gpus 4 --steps 5 --warmup 3 > $O/papers_n4.json 2> $O/papers_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 > $O/reddit_n4.json 2> $O/reddit_n4.log
python3 - <<'PY'
import json
for f in ['papers_n4','reddit_n4']:
    try:
        d=json.loads(open(f'gpurun_out/n4h/{f}.json').read().strip().splitlines()[-1])
        print(f, d['value'], d.get('epoch_ms_each_rank0'), d.get('peak_mem_gib'), d.get('epoch_breakdown_ms'))
    except Exception as e:
        print(f, 'ERR', e)
PY
