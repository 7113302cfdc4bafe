B="python bench.py --workload products --steps 2 --warmup 3 --no-cpu-baseline --no-transform-first"
timeout 600 $B > gpurun_out/r2_p_plain.json 2>/dev/null; echo "plain $?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_epochs/" --csv --log-file gpurun_out/r2_launches_products.csv $B > gpurun_out/r2_launches_products.log 2>&1; echo "ncu rc=$?"
