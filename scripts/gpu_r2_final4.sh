# round 2 final validation (1 GPU), after the dense 4-row tile
set -x
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/r2f4_gputest.log 2>&1; echo "pytest $?"
tail -4 gpurun_out/r2f4_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f4_smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/r2f4_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f4_bench_reddit.json 2> gpurun_out/r2f4_bench_reddit.log; echo "reddit $?"
timeout 900 python bench.py --workload products --steps 10 --warmup 3 > gpurun_out/r2f4_bench_products.json 2> gpurun_out/r2f4_bench_products.log; echo "products $?"
for f in gpurun_out/r2f4_bench_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ['value','e2e','clocks']}); print(d['epoch_breakdown_ms'])"; done
