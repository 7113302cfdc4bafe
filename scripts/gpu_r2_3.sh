set -x
timeout 300 python scripts/gather_tma_probe.py > gpurun_out/r2_tma_probe.txt 2>&1; echo "probe $?"
cat gpurun_out/r2_tma_probe.txt
timeout 2400 python -m pytest tests/test_gpu_configs.py tests/test_gpu_locality.py -v -s -x > gpurun_out/r2_configs.log 2>&1; echo "configs $?"
grep -E "PASS|FAIL|Error|Y_|passed|failed" gpurun_out/r2_configs.log | tail -30
CMD="python scripts/prof_spmm.py --workload products --f 100 16 --reps 1 --order lpa-part"
timeout 600 $CMD > gpurun_out/r2_prof_products_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -c 2 -o gpurun_out/r2_prof_products $CMD > gpurun_out/r2_ncu_products.log 2>&1; echo "ncu $?"
timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 16 --reps 3 > gpurun_out/r2_reddit_auto.txt 2>&1
cat gpurun_out/r2_prof_products_plain.txt gpurun_out/r2_reddit_auto.txt | grep ms
