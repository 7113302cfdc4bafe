#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -C paper_2504_04673_b200/csrc > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() { name=$1; shift; timeout 1500 $TR --nproc-per-node=$N --master-port $((29630 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline --no-transform-first "$@" > gpurun_out/d_$name.json 2> gpurun_out/d_$name.log; echo "rc=$?" >> gpurun_out/d_$name.log; }
N=4 run prod_gvb_1d --workload products --partition gvb
N=4 run prod_gvb_1d_obl --workload products --partition gvb --variant 1d-oblivious
N=4 run prod_gvb_c2 --workload products --partition gvb --variant 15d-sparse --c 2 --ranks-per-gpu 2
N=4 run prod_gvb_c2_obl --workload products --partition gvb --variant 15d-oblivious --c 2 --ranks-per-gpu 2
N=4 run prod_gvb_c4 --workload products --partition gvb --variant 15d-sparse --c 4 --ranks-per-gpu 4
N=4 run reddit_p8_c2 --variant 15d-sparse --c 2 --ranks-per-gpu 2
for f in gpurun_out/d_*.log; do echo "$f: $(tail -n 1 $f)"; done
python3 - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/d_*.json')):
    try: d = json.loads(open(f).read())
    except Exception as e: print(f, 'ERR', e); continue
    ex = d.get('exchange') or {}
    print(f"{f:34s} {d['value']:8.2f} ms p={d['config']['p']} c={d['config']['c']} part={d['config']['partition'][:40]} ratio={d['comm_elements_per_epoch']['ratio']} xchg={ex.get('achieved')}")
PY
