set -x
CMD="python scripts/prof_spmm.py --workload reddit --f 602 --reps 1"
timeout 600 $CMD > gpurun_out/r2n_reddit_plain.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -c 1 -o gpurun_out/r2n_prof_reddit602 $CMD > gpurun_out/r2n_ncu_reddit.log 2>&1; echo "ncu reddit $?"
CMD="python scripts/prof_spmm.py --workload products --f 100 16 47 --reps 1 --order lpa-part"
timeout 600 $CMD > gpurun_out/r2n_products_plain.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -c 5 -o gpurun_out/r2n_prof_products $CMD > gpurun_out/r2n_ncu_products.log 2>&1; echo "ncu products $?"
