set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_multigpu.py -q > gpurun_out/r2m5_multigpu_tests.log 2>&1; echo "mp tests $?"; tail -2 gpurun_out/r2m5_multigpu_tests.log
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fused.py -q > gpurun_out/r2m5_sharded.log 2>&1; echo "sharded $?"; tail -2 gpurun_out/r2m5_sharded.log
P=29940
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m5_products_n4.json 2> gpurun_out/r2m5_products_n4.log; echo "products n4 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --steps 20 --warmup 3 --no-transform-first > gpurun_out/r2m5_reddit_n4.json 2> gpurun_out/r2m5_reddit_n4.log; echo "reddit n4 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 2 --master-port $P bench.py --gpus 2 --steps 20 --warmup 3 --no-transform-first > gpurun_out/r2m5_reddit_n2.json 2> gpurun_out/r2m5_reddit_n2.log; echo "reddit n2 $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m5_products_15d_c2.json 2> gpurun_out/r2m5_products_15d_c2.log; echo "15d $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 2 --master-port $P bench.py --gpus 2 --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m5_products_n2.json 2> gpurun_out/r2m5_products_n2.log; echo "products n2 $?"
for f in gpurun_out/r2m5_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['epoch_breakdown_ms'])" 2>&1 | tail -2; done
