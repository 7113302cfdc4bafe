set -x
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2_gputest.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/r2_gputest.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_reddit.json 2> gpurun_out/r2_bench_reddit.log; echo "bench exit $?"
timeout 900 python bench.py --workload products --steps 10 --warmup 3 > gpurun_out/r2_bench_products.json 2> gpurun_out/r2_bench_products.log; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref_reddit.json 2> gpurun_out/r2_ref_reddit.log; echo "ref exit $?"
cat gpurun_out/r2_bench_reddit.json | cut -c1-600
