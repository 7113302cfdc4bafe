TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --workload products --graph off --steps 10 --warmup 3 --no-cpu-baseline --no-transform-first > gpurun_out/r2h_products_n1_eager.json 2> gpurun_out/r2h_products_n1_eager.log; echo "n1 $?"
timeout 900 $TR --nproc-per-node 4 --master-port 30101 bench.py --gpus 4 --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2h_products_n4.json 2> gpurun_out/r2h_products_n4.log; echo "n4 $?"
timeout 900 $TR --nproc-per-node 4 --master-port 30102 bench.py --gpus 4 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2h_reddit_n4.json 2> gpurun_out/r2h_reddit_n4.log; echo "reddit n4 $?"
for f in gpurun_out/r2h_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ['value','eager_host_issue_ms','cuda_graph']}); print(d.get('epoch_breakdown_ms'))" 2>&1 | tail -2; done
