# round 2: the multi-GPU evidence (gpurun --gpus 4)
set -x
nvidia-smi -L
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_multigpu.py -v -s > gpurun_out/r2m_multigpu_tests.log 2>&1; echo "mp tests $?"
grep -E "PASS|FAIL|checked|rank map" gpurun_out/r2m_multigpu_tests.log | tail -20
timeout 300 python scripts/xchg_nvlink_probe.py --reps 5 > gpurun_out/r2m_xchg_probe.txt 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes.sum.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:xchg -c 4 --csv --log-file gpurun_out/r2m_xchg_ncu.csv python scripts/xchg_nvlink_probe.py --reps 1 > gpurun_out/r2m_xchg_ncu.log 2>&1; echo "xchg ncu $?"
cat gpurun_out/r2m_xchg_probe.txt
P=29700
for N in 2 4; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/r2m_reddit_n$N.json 2> gpurun_out/r2m_reddit_n$N.log; echo "reddit N=$N $?"
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --steps 10 --warmup 3 > gpurun_out/r2m_products_n4.json 2> gpurun_out/r2m_products_n4.log; echo "products 1d $?"
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 1d-oblivious --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m_products_n4_obl.json 2> gpurun_out/r2m_products_n4_obl.log; echo "products 1d obl $?"
for RM in block cyclic; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 2 --ranks-per-gpu 2 --rank-map $RM --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m_products_15d_c2_$RM.json 2> gpurun_out/r2m_products_15d_c2_$RM.log; echo "products 15d c2 $RM $?"
done
P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --workload products --variant 15d-sparse --c 4 --ranks-per-gpu 4 --rank-map cyclic --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2m_products_15d_c4_cyclic.json 2> gpurun_out/r2m_products_15d_c4_cyclic.log; echo "products 15d c4 $?"
for f in gpurun_out/r2m_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('value'), d.get('e2e',{}).get('value'), d.get('exchange'), d.get('comm_elements_per_epoch'), d.get('run_config',{}).get('rank_map'))" 2>&1 | tail -2; done
