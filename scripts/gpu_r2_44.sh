TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 8 --master-port 30801 bench.py --gpus 8 --steps 10 --warmup 3 > gpurun_out/r2n8_reddit_8proc_on4.json 2> gpurun_out/r2n8_reddit_8proc_on4.log; echo "n8 $?"
timeout 900 $TR --nproc-per-node 8 --master-port 30802 bench.py --gpus 8 --workload products --variant 15d-sparse --c 2 --steps 5 --warmup 3 > gpurun_out/r2n8_products15d_8proc_on4.json 2> gpurun_out/r2n8_products15d_8proc_on4.log; echo "n8 15d $?"
timeout 900 $TR --nproc-per-node 8 --master-port 30803 bench.py --impl reference --gpus 8 --steps 2 --warmup 1 > gpurun_out/r2n8_ref.json 2> gpurun_out/r2n8_ref.log; echo "n8 ref $?"
for f in gpurun_out/r2n8_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d.get('n_gpus'), d.get('impl'), (d.get('e2e') or {}).get('value'), d.get('overlap_xchg_ctas'))" 2>&1 | tail -1; done
tail -3 gpurun_out/r2n8_reddit_8proc_on4.log
