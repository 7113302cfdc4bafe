set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fused.py -x -q > gpurun_out/r2_sharded_tests.log 2>&1; echo "sharded tests $?"; tail -2 gpurun_out/r2_sharded_tests.log
for lib in default tn2; do
  if [ $lib = default ]; then export DG_LIB_PATH=paper_2504_04673_b200/libdgb200.so; else export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_$lib.so; fi
  echo "== $lib"
  timeout 300 python scripts/dense_one.py wgrad 232965 602 16 10
  timeout 300 python scripts/dense_one.py wgrad 2449029 100 16 10
  timeout 300 python scripts/dense_one.py wgrad 2449029 16 47 10
done
unset DG_LIB_PATH
CMD="python scripts/dense_one.py wgrad 232965 602 16 2"
timeout 300 $CMD > gpurun_out/r2_tn602_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_tn_tma -c 1 -o gpurun_out/r2_prof_tn602 $CMD > gpurun_out/r2_ncu_tn602.log 2>&1; echo "ncu $?"
