# round 2 final multi-GPU lines (gpurun --gpus 4)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29800
for N in 2 4; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/r2m2_reddit_n$N.json 2> gpurun_out/r2m2_reddit_n$N.log; echo "reddit N=$N $?"
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --impl reference --steps 3 --warmup 1 > gpurun_out/r2m2_ref_reddit_n$N.json 2> gpurun_out/r2m2_ref_reddit_n$N.log; echo "ref N=$N $?"
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 2 --master-port $P bench.py --gpus 2 --workload products --steps 10 --warmup 3 > gpurun_out/r2m2_products_n2.json 2> gpurun_out/r2m2_products_n2.log; echo "products n2 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --steps 10 --warmup 3 > gpurun_out/r2m2_products_n4.json 2> gpurun_out/r2m2_products_n4.log; echo "products n4 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 1d-oblivious --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m2_products_n4_obl.json 2> gpurun_out/r2m2_products_n4_obl.log; echo "products n4 obl $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m2_products_15d_c2.json 2> gpurun_out/r2m2_products_15d_c2.log; echo "products 15d c2 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-oblivious --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m2_products_15d_c2_obl.json 2> gpurun_out/r2m2_products_15d_c2_obl.log; echo "products 15d c2 obl $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --partition gvb --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m2_products_n4_gvb.json 2> gpurun_out/r2m2_products_n4_gvb.log; echo "products gvb $?"
P=$((P+1)); timeout 1800 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload papers --steps 3 --warmup 2 > gpurun_out/r2m2_papers_n4.json 2> gpurun_out/r2m2_papers_n4.log; echo "papers $?"
for f in gpurun_out/r2m2_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ['value','ms_per_step','e2e','clocks','value_kind']}); print(d.get('exchange'), d.get('comm_elements_per_epoch'), (d.get('roofline') or {}).get('kernel_ms'))" 2>&1 | tail -3; done
