TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_xchg.py -q -x 2>&1 | grep -E "Error|assert|passed|failed|^E " | head -30
P=30400
for W in products reddit; do for N in 4 2; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --workload $W --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2d_${W}_n$N.json 2> gpurun_out/r2d_${W}_n$N.log; echo "$W N=$N $?"
done; done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2d_products_15d_c2.json 2> gpurun_out/r2d_products_15d_c2.log; echo "15d $?"
for f in gpurun_out/r2d_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); b=d['epoch_breakdown_ms']; print('$f', d['value'], d['e2e']['value'], d['exchange']['exchange_ms'], d.get('overlap_xchg_ctas'), {k: v for k, v in b.items() if 'spmm' in k})"; done
