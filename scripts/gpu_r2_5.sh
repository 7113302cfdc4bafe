set -x
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r2_dense_tests.log 2>&1; echo "dense tests $?"
tail -5 gpurun_out/r2_dense_tests.log
timeout 600 python scripts/dense_probe.py > gpurun_out/r2_dense_probe.txt 2>&1; echo "probe $?"
cat gpurun_out/r2_dense_probe.txt
timeout 1200 python scripts/diag_grad.py products > gpurun_out/r2_diag_grad2.txt 2>&1; echo "diag $?"
grep -v Warn gpurun_out/r2_diag_grad2.txt | tail -16
