# sparsity-aware saving on a more strongly clustered products-shaped graph (p_in = 0.95)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29980
for V in 1d-sparse 1d-oblivious; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --p-in 0.95 --variant $V --steps 10 --warmup 3 --no-transform-first --no-cpu-baseline > gpurun_out/r2pin_products_n4_$V.json 2> gpurun_out/r2pin_products_n4_$V.log; echo "$V $?"
done
for f in gpurun_out/r2pin_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d.get('exchange'), d.get('comm_elements_per_epoch'), d['epoch_breakdown_ms'])"; done
