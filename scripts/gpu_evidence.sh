#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/ev_plain.json 2> gpurun_out/ev_plain.log && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_epochs/" --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ev_ncu.log 2>&1
P="python scripts/prof_spmm.py --f 602 --reps 1"
$P > gpurun_out/ev_p602.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v3_602 $P > gpurun_out/ev_ncu602.log 2>&1
P16="python scripts/prof_spmm.py --f 16 --reps 1"
$P16 > gpurun_out/ev_p16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 1 -c 1 -o gpurun_out/prof_v3_16 $P16 > gpurun_out/ev_ncu16.log 2>&1
timeout 900 python bench.py --workload products --steps 3 --warmup 2 > gpurun_out/ev_products_n1.json 2> gpurun_out/ev_products_n1.log
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv; tail -n 2 gpurun_out/ev_products_n1.log
