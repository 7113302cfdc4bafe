set -x
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r2_dense_tests3.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2_dense_tests3.log
timeout 300 python scripts/dense_one.py wgrad 232965 602 16 10
timeout 300 python scripts/dense_one.py wgrad 2449029 100 16 10
timeout 300 python scripts/dense_one.py wgrad 2449029 16 47 10
timeout 300 python scripts/dense_one.py wgrad 2449029 16 16 10
