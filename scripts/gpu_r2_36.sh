TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 30111 bench.py --gpus 4 --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2n_products_n4.json 2> gpurun_out/r2n_products_n4.log; echo "n4 $?"
timeout 900 $TR --nproc-per-node 2 --master-port 30112 bench.py --gpus 2 --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2n_products_n2.json 2> gpurun_out/r2n_products_n2.log; echo "n2 $?"
for f in gpurun_out/r2n_products_n*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d.get('narrow_phase')); print(d.get('epoch_breakdown_ms'))" 2>&1 | tail -2; done
tail -5 gpurun_out/r2n_products_n4.log
