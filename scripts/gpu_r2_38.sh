TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_xchg.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_multigpu.py -q 2>&1 | tail -2
timeout 300 python scripts/xchg_nvlink_probe.py --reps 5 2>&1 | grep xchg
P=30300
for N in 2 4; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 5 --no-transform-first > gpurun_out/r2c_reddit_n$N.json 2> gpurun_out/r2c_reddit_n$N.log; echo "reddit N=$N $?"
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2c_products_n$N.json 2> gpurun_out/r2c_products_n$N.log; echo "products N=$N $?"
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2c_products_15d_c2.json 2> gpurun_out/r2c_products_15d_c2.log; echo "15d $?"
for f in gpurun_out/r2c_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); b=d['epoch_breakdown_ms']; print('$f', d['value'], d['e2e']['value'], d['exchange']['exchange_ms'], {k: v for k, v in b.items() if 'spmm' in k}, d.get('narrow_phase'))"; done
