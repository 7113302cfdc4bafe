#!/bin/bash
# gpurun (1 GPU): GPU tests, smoke, N=1 benches (Reddit, products, rmat14), ncu launch list
cd "$(dirname "$0")/.."
O=gpurun_out/final1; mkdir -p $O
make -C paper_2504_04673_b200/csrc > $O/build.txt 2>&1 || { tail -20 $O/build.txt; exit 1; }
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt; tail -n 2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt; tail -n 2 $O/smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/reddit_n1.json 2> $O/reddit_n1.log; echo "reddit rc=$?"
timeout 900 python bench.py --workload products --steps 10 --warmup 3 > $O/products_n1.json 2> $O/products_n1.log; echo "products rc=$?"
timeout 900 python bench.py --workload rmat14 --steps 10 --warmup 3 > $O/rmat14_n1.json 2> $O/rmat14_n1.log; echo "rmat14 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_n1.json 2> $O/reference_n1.log; echo "reference rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-transform-first"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_epochs/" --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1; echo "ncu rc=$?"
python3 - <<'PY'
import json, glob, os
for f in sorted(glob.glob('gpurun_out/final1/*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), d['value'], (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('kernel_ms'), (d.get('cpu_baseline') or {}).get('value'))
    except Exception as e:
        print(f, 'ERR', e)
PY
