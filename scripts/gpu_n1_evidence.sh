#!/bin/bash
# one gpurun call (1 GPU): GPU tests, N=1 bench (Reddit + products), ncu launch
# list of the timed epochs, ncu --set full of the layer-1 SpMM (f=602 and f=100)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
tail -n 2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.log; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 900 python bench.py --workload products --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_products_n1.json 2> gpurun_out/bench_products_n1.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-transform-first"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_epochs/" --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
P="python scripts/prof_spmm.py --f 602 --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v4_602 $P > gpurun_out/ncu602.log 2>&1
P="python scripts/prof_spmm.py --workload products --f 100 --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v4_products_100 $P > gpurun_out/ncu100.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv
python3 - <<'PY'
import json
for f in ['gpurun_out/bench_n1.json','gpurun_out/bench_products_n1.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d['value'], d['e2e'], d['roofline']['kernel_ms'], d['roofline']['gather_gbs'], d.get('epoch_breakdown_ms'))
    except Exception as e:
        print(f, 'ERR', e)
PY
