set -x
for lib in default v8b16 v8b8 onechunk; do
  if [ $lib = default ]; then export DG_LIB_PATH=paper_2504_04673_b200/libdgb200.so; else export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_$lib.so; fi
  timeout 600 python scripts/prof_spmm.py --workload products --f 16 47 --reps 5 --order lpa-part > gpurun_out/r2_lanes_products_$lib.txt 2>&1
  timeout 600 python scripts/prof_spmm.py --workload reddit --f 16 41 --reps 5 > gpurun_out/r2_lanes_reddit_$lib.txt 2>&1
  echo "== $lib"; grep " ms" gpurun_out/r2_lanes_products_$lib.txt gpurun_out/r2_lanes_reddit_$lib.txt
done
unset DG_LIB_PATH
timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 --reps 3 --slab-major 64 > gpurun_out/r2_reddit_slabmajor.txt 2>&1
grep " ms" gpurun_out/r2_reddit_slabmajor.txt
