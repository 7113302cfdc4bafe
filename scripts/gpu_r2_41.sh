TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_xchg.py -q -x 2>&1 | tail -1
timeout 2400 $TR --nproc-per-node 4 --master-port 30501 bench.py --gpus 4 --workload papers --steps 3 --warmup 2 > gpurun_out/r2f_papers_n4.json 2> gpurun_out/r2f_papers_n4.log; echo "papers $?"
timeout 900 $TR --nproc-per-node 4 --master-port 30502 bench.py --gpus 4 --workload products --steps 10 --warmup 3 > gpurun_out/r2f_products_n4.json 2> gpurun_out/r2f_products_n4.log; echo "products $?"
timeout 900 $TR --nproc-per-node 4 --master-port 30503 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2f_reddit_n4.json 2> gpurun_out/r2f_reddit_n4.log; echo "reddit $?"
for f in gpurun_out/r2f_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel_ms'], d['exchange']['frac'], d['comm_elements_per_epoch']['ratio'], d.get('overlap_xchg_ctas'))" 2>&1 | tail -1; done
