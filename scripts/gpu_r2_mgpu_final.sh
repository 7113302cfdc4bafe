# round 2 final multi-GPU lines (gpurun --gpus 4)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29960
for N in 2 4; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2mf_reddit_n$N.json 2> gpurun_out/r2mf_reddit_n$N.log; echo "reddit N=$N $?"
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --workload products --steps 10 --warmup 3 > gpurun_out/r2mf_products_n$N.json 2> gpurun_out/r2mf_products_n$N.log; echo "products N=$N $?"
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --impl reference --steps 20 --warmup 5 > gpurun_out/r2mf_ref_reddit_n4.json 2> gpurun_out/r2mf_ref_reddit_n4.log; echo "ref N=4 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 > gpurun_out/r2mf_products_15d_c2.json 2> gpurun_out/r2mf_products_15d_c2.log; echo "15d c2 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --rank-map cyclic --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2mf_products_15d_c2_cyclic.json 2> gpurun_out/r2mf_products_15d_c2_cyclic.log; echo "15d c2 cyclic $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 1d-oblivious --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2mf_products_n4_obl.json 2> gpurun_out/r2mf_products_n4_obl.log; echo "obl $?"
# the N=8 code path: 8 processes on 4 GPUs (two per GPU: host barriers)
P=$((P+1)); timeout 900 $TR --nproc-per-node 8 --master-port $P bench.py --gpus 8 --steps 5 --warmup 3 --no-transform-first > gpurun_out/r2mf_reddit_8proc_on4.json 2> gpurun_out/r2mf_reddit_8proc_on4.log; echo "8 procs $?"
for f in gpurun_out/r2mf_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ['value','ms_per_step','e2e','value_kind']}); print(d.get('exchange'), d.get('comm_elements_per_epoch'))" 2>&1 | tail -2; done
