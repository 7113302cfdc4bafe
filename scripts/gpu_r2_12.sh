set -x
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/r2_xent_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2_xent_tests.log
timeout 300 python scripts/xent_probe.py 10
for lib in head v2; do
  if [ $lib = head ]; then export DG_LIB_PATH=paper_2504_04673_b200/libdgb200.so; else export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_v2.so; fi
  timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 16 41 --reps 5 > gpurun_out/r2_v2_reddit_$lib.txt 2>&1
  timeout 600 python scripts/prof_spmm.py --workload products --f 100 16 47 --reps 5 --order lpa-part > gpurun_out/r2_v2_products_$lib.txt 2>&1
  echo "== $lib"; grep -h " ms" gpurun_out/r2_v2_reddit_$lib.txt gpurun_out/r2_v2_products_$lib.txt
done
