set -x
timeout 3000 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r2_gputest2.log 2>&1; echo "pytest $?"
tail -25 gpurun_out/r2_gputest2.log
timeout 900 python bench.py --workload products --steps 10 --warmup 3 > gpurun_out/r2_bench_products3.json 2> gpurun_out/r2_bench_products3.log; echo "bench $?"
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_reddit3.json 2> gpurun_out/r2_bench_reddit3.log; echo "bench $?"
timeout 600 python scripts/diag_lpa.py > gpurun_out/r2_diag_lpa.txt 2>&1; echo "lpa $?"
cat gpurun_out/r2_diag_lpa.txt | grep -v Warn
