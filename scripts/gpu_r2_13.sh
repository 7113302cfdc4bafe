set -x
timeout 900 python -m pytest tests/test_gpu_numerics.py tests/test_gpu_parity.py tests/test_gpu_locality.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_v2_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2_v2_tests.log
export DG_LIB_PATH=paper_2504_04673_b200/libdgb200_v3.so
timeout 600 python scripts/prof_spmm.py --workload products --f 100 --reps 5 --order lpa-part > gpurun_out/r2_v3_products.txt 2>&1
grep -h " ms" gpurun_out/r2_v3_products.txt
unset DG_LIB_PATH
timeout 900 python bench.py --workload products --steps 10 --warmup 3 > gpurun_out/r2_bench_products4.json 2> gpurun_out/r2_bench_products4.log; echo "bench $?"
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_reddit4.json 2> gpurun_out/r2_bench_reddit4.log; echo "bench $?"
for f in gpurun_out/r2_bench_products4.json gpurun_out/r2_bench_reddit4.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['epoch_breakdown_ms'], d['clocks'])"; done
