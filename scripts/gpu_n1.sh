#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/n1_reddit.json 2> gpurun_out/n1_reddit.log
timeout 900 python bench.py --workload products --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n1_products.json 2> gpurun_out/n1_products.log
python3 -c "
import json
for f in ['gpurun_out/n1_reddit.json','gpurun_out/n1_products.json']:
    d=json.loads(open(f).read()); print(f, d['value'], d['roofline']['kernel_ms'], d['roofline']['gather_gbs'], d['epoch_breakdown_ms'])
"
