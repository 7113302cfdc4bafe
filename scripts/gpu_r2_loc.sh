# round 2: locality schedules (windowed bucketing + LPA order) on the GPU
set -x
timeout 900 python -m pytest tests/test_gpu_locality.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_loc_tests.log 2>&1; echo "tests $?"
tail -3 gpurun_out/r2_loc_tests.log
for o in none lpa lpa-part; do
  timeout 600 python scripts/prof_spmm.py --workload products --f 100 16 47 --reps 5 --order $o > gpurun_out/r2_loc_products_$o.txt 2>&1; echo "prof $o $?"
done
timeout 600 python scripts/prof_spmm.py --workload products --f 100 16 --reps 5 --order lpa-part --window 1099511627776 > gpurun_out/r2_loc_products_lpa-part_globalsort.txt 2>&1
timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 16 41 --reps 3 > gpurun_out/r2_loc_reddit.txt 2>&1; echo "reddit $?"
timeout 600 python scripts/prof_spmm.py --workload reddit --f 602 16 --reps 3 --window 1099511627776 > gpurun_out/r2_loc_reddit_globalsort.txt 2>&1
timeout 900 python bench.py --workload products --steps 10 --warmup 3 --no-transform-first > gpurun_out/r2_bench_products_lpa.json 2> gpurun_out/r2_bench_products_lpa.log; echo "bench $?"
grep -h "ms" gpurun_out/r2_loc_*.txt | grep -v Warn
