timeout 900 python -m pytest tests/test_gpu_dense.py -k xent -q 2>&1 | tail -3; timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_gcn.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -5
timeout 300 python scripts/xent_probe.py 20 2>&1 | tail -2
timeout 600 python bench.py --workload reddit --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_xent_bench_reddit.json 2> gpurun_out/r2_xent_bench_reddit.log; tail -c 600 gpurun_out/r2_xent_bench_reddit.json
