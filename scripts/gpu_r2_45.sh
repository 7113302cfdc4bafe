for n in default E2 E2M3 E2M2; do
  if [ $n = default ]; then LP=""; else LP="DG_LIB_PATH=$PWD/paper_2504_04673_b200/libdgb200_$n.so"; fi
  echo "== $n"
  env $LP timeout 600 python scripts/prof_spmm.py --workload products --order lpa-part --f 47 --reps 10 2>&1 | grep "^f="
  env $LP timeout 600 python scripts/prof_spmm.py --workload reddit --f 41 --reps 10 2>&1 | grep "^f="
done
