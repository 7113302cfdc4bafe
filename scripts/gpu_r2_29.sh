set -x
for lib in default g1; do
  if [ $lib = default ]; then export DG_LIB_PATH=paper_2504_04673_b200/libdgb200.so; else export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_$lib.so; fi
  echo "== $lib"
  timeout 600 python scripts/prof_spmm.py --workload reddit --f 16 --reps 5 2>&1 | grep " ms"
  timeout 600 python scripts/prof_spmm.py --workload products --f 16 --reps 5 --order lpa-part 2>&1 | grep " ms"
done
