set -x
timeout 900 python -m pytest tests/test_gpu_numerics.py tests/test_gpu_parity.py tests/test_gpu_locality.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_bf_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/r2_bf_tests.log
for lib in new prev; do
  if [ $lib = new ]; then export DG_LIB_PATH=paper_2504_04673_b200/libdgb200.so; else export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_prev.so; fi
  timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 16 41 --reps 5 > gpurun_out/r2_bf_reddit_$lib.txt 2>&1
  timeout 600 python scripts/prof_spmm.py --workload products --f 100 16 47 --reps 5 --order lpa-part > gpurun_out/r2_bf_products_$lib.txt 2>&1
  echo "== $lib"; grep -h " ms" gpurun_out/r2_bf_reddit_$lib.txt gpurun_out/r2_bf_products_$lib.txt
done
