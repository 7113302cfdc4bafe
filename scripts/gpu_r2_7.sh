set -x
for w in 131072 262144 524288 1048576 2097152 4194304; do
  timeout 600 python scripts/prof_spmm.py --workload products --f 100 16 47 --reps 5 --order lpa-part --window $w > gpurun_out/r2_win_$w.txt 2>&1
  echo "window $w"; grep " ms" gpurun_out/r2_win_$w.txt
done
