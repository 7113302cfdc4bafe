set -x
export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_rpt4.so
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q 2>&1 | tail -2
for lib in default rpt4; do
  if [ $lib = default ]; then export DG_LIB_PATH=paper_2504_04673_b200/libdgb200.so; else export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_$lib.so; fi
  echo "== $lib"
  timeout 300 python scripts/dense_one.py fwd 232965 602 16 10
  timeout 300 python scripts/dense_one.py fwd 2449029 100 16 10
  timeout 300 python scripts/dense_one.py fwd 2449029 16 16 10
done
