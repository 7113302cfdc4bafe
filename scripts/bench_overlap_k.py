"""Diagnostics: bench.py with engine.OVERLAP_XCHG_K set from the first
argument (the exchange-cap sweep of profiles/r02/xchg_cap/).

    torchrun ... scripts/bench_overlap_k.py 1500 --gpus 4 --workload products ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_04673_b200.engine as E  # noqa: E402

E.OVERLAP_XCHG_K = float(sys.argv.pop(1))
import bench  # noqa: E402

sys.exit(bench.main())
