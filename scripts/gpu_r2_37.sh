TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cap in 0 12 24 48 96 192; do echo "cap=$cap"; DG_XCHG_CTAS=$cap timeout 300 python scripts/xchg_nvlink_probe.py --reps 5 2>&1 | grep xchg; done
P=30200
for cap in 0 24 48 96; do
  P=$((P+1)); DG_XCHG_CTAS=$cap timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2x_reddit_n4_$cap.json 2> gpurun_out/r2x_reddit_n4_$cap.log
  python -c "
import json; d=json.loads(open('gpurun_out/r2x_reddit_n4_$cap.json').read().strip().splitlines()[-1]); print('reddit n4 cap=$cap', d['value'], d['epoch_breakdown_ms']['fwd_spmm_f602'], d['exchange']['exchange_ms'], d['roofline']['kernel_ms'])"
done
