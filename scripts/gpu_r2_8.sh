set -x
timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 --reps 3 --slab 0 64 128 256 512 > gpurun_out/r2_reddit_slabs.txt 2>&1; echo "slabs $?"
grep " ms" gpurun_out/r2_reddit_slabs.txt
timeout 600 python scripts/dense_probe.py > gpurun_out/r2_dense_probe2.txt 2>&1; grep xent gpurun_out/r2_dense_probe2.txt
timeout 300 python -m pytest tests/test_gpu_dense.py -q -x 2>&1 | tail -2
CMD="python scripts/prof_spmm.py --workload products --f 16 47 --reps 1 --order lpa-part"
timeout 600 $CMD > gpurun_out/r2_prof_products_1647_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -c 4 -o gpurun_out/r2_prof_products_1647 $CMD > gpurun_out/r2_ncu_products_1647.log 2>&1; echo "ncu $?"
