set -x
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_gcn.py -x -q > gpurun_out/r2_fused_tests.log 2>&1; echo "tests $?"; tail -15 gpurun_out/r2_fused_tests.log
timeout 900 python bench.py --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2_bench_products_fused.json 2> gpurun_out/r2_bench_products_fused.log; echo "bench $?"
timeout 900 python bench.py --steps 20 --warmup 3 --no-transform-first > gpurun_out/r2_bench_reddit_fused.json 2> gpurun_out/r2_bench_reddit_fused.log; echo "bench $?"
for f in gpurun_out/r2_bench_products_fused.json gpurun_out/r2_bench_reddit_fused.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['epoch_breakdown_ms'], d['clocks'])"; done
