set -x
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q 2>&1 | tail -2
timeout 600 python scripts/dense_probe.py 2>&1 | grep -v legacy
