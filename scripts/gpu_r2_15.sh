set -x
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r2_dense_tests2.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2_dense_tests2.log
timeout 600 python scripts/dense_probe.py > gpurun_out/r2_dense_probe3.txt 2>&1; echo "probe $?"
grep -v legacy gpurun_out/r2_dense_probe3.txt
CMD="python scripts/gather_tma_probe.py"
timeout 300 $CMD > gpurun_out/r2_tma_probe3.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:gather_tma_probe -c 1 -o gpurun_out/r2_prof_gather4 $CMD > gpurun_out/r2_ncu_gather4.log 2>&1; echo "ncu $?"
