"""Single-GPU probe of the sharded papers-shaped path: generation, sharded
operand, device plans for p emulated ranks, one f=16 multiply phase.
Prints timings and memory (sizing check before the 4-GPU run)."""
import argparse
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2504_04673_b200 import sharded  # noqa: E402
from paper_2504_04673_b200.engine import DevicePlan  # noqa: E402
from paper_2504_04673_b200.plan import build_variant_plan  # noqa: E402
from paper_2504_04673_b200.runtime import ProcessGrid  # noqa: E402


def gib(x):
    return f"{x / 2**30:.1f} GiB"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    print(subprocess.run(["bash", "-c", "free -g; nproc; cat /sys/fs/cgroup/memory.max 2>/dev/null"],
                         capture_output=True, text=True).stdout, flush=True)
    n = int(111_059_956 * a.scale)
    nnz = int(3_231_371_744 * a.scale)
    t = time.time()
    g = sharded.chung_lu_sharded(n, nnz // 2, a.p, alpha=0.7, max_weight=30_000, seed=0,
                                 log=print)
    print(f"gen {time.time() - t:.1f}s nnz {g.nnz_total:,} mem {gib(torch.cuda.memory_allocated())}"
          f" peak {gib(torch.cuda.max_memory_allocated())}", flush=True)
    t = time.time()
    op = sharded.ShardedOperand(g)
    print(f"operand {time.time() - t:.1f}s halo rows per rank {op.counts.sum(1).tolist()} "
          f"peak {gib(torch.cuda.max_memory_allocated())}", flush=True)
    t = time.time()
    grid = ProcessGrid(a.p, 1)
    vp = build_variant_plan(op, grid, "1d-sparse")
    dp = DevicePlan(vp)
    g.release()
    torch.cuda.empty_cache()
    print(f"plans {time.time() - t:.1f}s info {dp.info} mem {gib(torch.cuda.memory_allocated())}"
          f" peak {gib(torch.cuda.max_memory_allocated())}", flush=True)
    f = 16
    hs = {r: torch.randn((g.boundaries[r][1] - g.boundaries[r][0], f), device="cuda")
          for r in range(a.p)}
    out = dp.run(hs, f, f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        out = dp.run(hs, f, f, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"phase f=16 (exchange + SpMM, {a.p} ranks on one GPU): {ms:.2f} ms; "
          f"gather {8 * g.nnz_total + 64 * g.nnz_total:,} B -> "
          f"{(8 + 64) * g.nnz_total / ms / 1e6:.0f} GB/s; mem peak {gib(torch.cuda.max_memory_allocated())}",
          flush=True)


if __name__ == "__main__":
    main()
