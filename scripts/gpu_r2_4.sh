set -x
timeout 300 python scripts/gather_tma_probe.py > gpurun_out/r2_tma_probe2.txt 2>&1; echo "probe $?"
cat gpurun_out/r2_tma_probe2.txt
timeout 1200 python scripts/diag_grad.py products > gpurun_out/r2_diag_grad.txt 2>&1; echo "diag $?"
grep -v Warn gpurun_out/r2_diag_grad.txt | tail -30
