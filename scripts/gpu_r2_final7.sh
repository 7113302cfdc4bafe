# round 2 final validation, 1 GPU
set -x
timeout 3000 python -m pytest tests -m gpu -q -rs --durations=5 > gpurun_out/r2f7_gputest.log 2>&1; echo "pytest $?"
tail -8 gpurun_out/r2f7_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f7_smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/r2f7_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f7_bench_reddit.json 2> gpurun_out/r2f7_bench_reddit.log; echo "reddit $?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f7_ref_reddit.json 2> gpurun_out/r2f7_ref_reddit.log; echo "ref $?"
timeout 900 python bench.py --workload products --steps 10 --warmup 3 > gpurun_out/r2f7_bench_products.json 2> gpurun_out/r2f7_bench_products.log; echo "products $?"
timeout 900 python bench.py --workload rmat14 --steps 20 --warmup 5 > gpurun_out/r2f7_bench_rmat14.json 2> gpurun_out/r2f7_bench_rmat14.log; echo "rmat14 $?"
timeout 900 ncu --nvtx --nvtx-include "timed_epochs/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f7_launches_reddit.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-transform-first > gpurun_out/r2f7_launches_reddit.log 2>&1; echo "launches $?"
for f in gpurun_out/r2f7_bench_*.json gpurun_out/r2f7_ref_*.json; do echo "== $f"; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ['value','ms_per_step','e2e','clocks','gpu_launches','value_kind','wall_s']}); print(d.get('roofline'))"; done
