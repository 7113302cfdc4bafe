TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=30700
for N in 2 4; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --workload products --steps 10 --warmup 3 > gpurun_out/r2m_products_n$N.json 2> gpurun_out/r2m_products_n$N.log
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2m_reddit_n$N.json 2> gpurun_out/r2m_reddit_n$N.log
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --p-in 0.95 --steps 10 --warmup 3 > gpurun_out/r2m_pin_products_n4_1d-sparse.json 2> gpurun_out/r2m_pin.log
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 > gpurun_out/r2m_products_15d_c2.json 2> gpurun_out/r2m_15d.log
for f in gpurun_out/r2m_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel_ms'], d['exchange']['frac'], d['comm_elements_per_epoch']['ratio'], d.get('overlap_xchg_ctas'))" 2>&1 | tail -1; done
