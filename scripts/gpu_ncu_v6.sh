#!/bin/bash
# 1 GPU: ncu --set full of the current layer-1 SpMM (Reddit f=602, products f=100 community),
# and the reference arm line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { tail -20 gpurun_out/build.txt; exit 1; }
P="python scripts/prof_spmm.py --f 602 --reps 1"
$P > gpurun_out/p602.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v6_602 $P > gpurun_out/ncu602.log 2>&1
P="python scripts/prof_spmm.py --workload products --community --f 100 --reps 1"
$P > gpurun_out/p100.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v6_products_100 $P > gpurun_out/ncu100.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.log
ls -la gpurun_out/*.ncu-rep; tail -c 600 gpurun_out/ref_arm.json
