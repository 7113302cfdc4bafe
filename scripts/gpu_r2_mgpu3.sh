set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_multigpu.py -v > gpurun_out/r2m3_multigpu_tests.log 2>&1; echo "mp tests $?"; grep -E "PASS|FAIL" gpurun_out/r2m3_multigpu_tests.log
timeout 2400 $TR --nproc-per-node 4 --master-port 29911 bench.py --gpus 4 --workload papers --steps 3 --warmup 2 > gpurun_out/r2m3_papers_n4.json 2> gpurun_out/r2m3_papers_n4.log; echo "papers $?"
tail -c 2000 gpurun_out/r2m3_papers_n4.json
