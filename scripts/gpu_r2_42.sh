TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_xchg.py -q -x 2>&1 | tail -1
for cap in 0 48 96 143; do echo "cap=$cap"; timeout 300 python scripts/xchg_nvlink_probe.py --reps 5 --ctas $cap 2>&1 | grep xchg; done
P=30600
for K in 1500 2500 4000; do for W in products reddit; do
  P=$((P+1)); timeout 900 $TR --nproc-per-node 4 --master-port $P scripts/bench_overlap_k.py $K --gpus 4 --workload $W --steps 10 --warmup 3 --no-transform-first --no-cpu-baseline > gpurun_out/r2k_${W}_$K.json 2> gpurun_out/r2k_${W}_$K.log
  python -c "
import json; d=json.loads(open('gpurun_out/r2k_${W}_$K.json').read().strip().splitlines()[-1]); b=d['epoch_breakdown_ms']; print('$W K=$K', d['value'], d.get('overlap_xchg_ctas'), {k: v for k, v in b.items() if 'spmm' in k})"
done; done
