timeout 900 python -m pytest tests/test_gpu_xchg.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_cabi.py -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_multigpu.py -q 2>&1 | tail -2
timeout 600 python bench.py --workload rmat14 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_rmat14.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2e_rmat14.json').read().strip().splitlines()[-1]); print('rmat14', d['value'], d['e2e']['value'])"
