set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_multigpu.py -q > gpurun_out/r2mg8_multigpu_tests.log 2>&1; echo "mp tests $?"; tail -1 gpurun_out/r2mg8_multigpu_tests.log
P=30010
P=$((P+1)); timeout 2400 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload papers --steps 3 --warmup 2 > gpurun_out/r2mg8_papers_n4.json 2> gpurun_out/r2mg8_papers_n4.log; echo "papers $?"
for N in 2 4; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2mg8_reddit_n$N.json 2> gpurun_out/r2mg8_reddit_n$N.log; echo "reddit N=$N $?"
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --workload products --steps 10 --warmup 3 > gpurun_out/r2mg8_products_n$N.json 2> gpurun_out/r2mg8_products_n$N.log; echo "products N=$N $?"
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --steps 10 --warmup 3 > gpurun_out/r2mg8_products_15d_c2.json 2> gpurun_out/r2mg8_products_15d_c2.log; echo "15d $?"
for f in gpurun_out/r2mg8_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ['value','e2e']}); print(d.get('exchange',{}) and d['exchange'].get('frac'), d.get('peak_mem_gib'))" 2>&1 | tail -2; done
P=30090
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 1d-oblivious --steps 10 --warmup 3 > gpurun_out/r2mg8_products_n4_obl.json 2> gpurun_out/r2mg8_products_n4_obl.log; echo "obl $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --rank-map cyclic --steps 10 --warmup 3 > gpurun_out/r2mg8_products_15d_c2_cyclic.json 2> gpurun_out/r2mg8_products_15d_c2_cyclic.log; echo "cyclic $?"
for W in 1d-sparse 1d-oblivious; do P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --p-in 0.95 --variant $W --steps 10 --warmup 3 > gpurun_out/r2mg8_pin_products_n4_$W.json 2> gpurun_out/r2mg8_pin_products_n4_$W.log; echo "pin $W $?"; done
for f in gpurun_out/r2mg8_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], (d.get('e2e') or {}).get('value'), d['roofline']['kernel_ms'], d['exchange']['frac'], d['comm_elements_per_epoch']['ratio'], d.get('overlap_xchg_ctas'))" 2>&1 | tail -1; done
