timeout 900 python scripts/prof_spmm.py --workload products --order lpa-part --f 16 --reps 10 --slab-major 8 2>&1 | grep -v Warn
timeout 900 python scripts/prof_spmm.py --workload products --order lpa-part --f 48 --reps 10 --slab-major 16 2>&1 | grep "f=" 
timeout 900 python scripts/prof_spmm.py --workload products --order lpa-part --f 100 --reps 5 --slab-major 32 2>&1 | grep "f="
