set -x
free -g | head -2; nproc
timeout 2400 python bench.py --impl reference --ref-full --steps 1 --warmup 0 > gpurun_out/r2_ref_full_reddit.json 2> gpurun_out/r2_ref_full_reddit.log; echo "ref full $?"
tail -3 gpurun_out/r2_ref_full_reddit.log; cut -c1-1500 gpurun_out/r2_ref_full_reddit.json
