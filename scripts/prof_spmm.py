"""Profile helper: build a benchmark graph and run the local SpMM at given
widths / slab widths (timing sweeps and the ncu target).

    python scripts/prof_spmm.py --workload reddit --f 602 16 --reps 3 [--acc 1] [--slab 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_04673_b200 as P  # noqa: E402
from paper_2504_04673_b200 import _lib as L  # noqa: E402
from paper_2504_04673_b200.engine import pad4  # noqa: E402
from paper_2504_04673_b200.spmm import device_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="reddit")
    ap.add_argument("--f", type=int, nargs="+", default=[602])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--acc", type=int, nargs="+", default=[2])
    ap.add_argument("--slab", type=int, nargs="+", default=[0])
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--ld-align", type=int, default=0)
    ap.add_argument("--order", default="none", choices=["none", "lpa", "lpa-part"],
                    help="lpa: SpMM row order by label-propagation communities (plan only); "
                         "lpa-part: relabel the graph by lpa_partition(k=1) (as bench.py)")
    ap.add_argument("--slab-major", type=int, default=0,
                    help="also time the wide layer from a slab-major copy of H: slabs of this "
                         "many floats stored contiguously, one dg_spmm_run per slab")
    ap.add_argument("--window", type=int, default=0,
                    help="entries per length-bucketing window of the plan (0: default)")
    ap.add_argument("--cusparse", action="store_true",
                    help="also time torch.sparse.mm (cuSPARSE) on the same matrix (comparator)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    a = bench.make_graph(args.workload)
    if args.order == "lpa-part":
        from paper_2504_04673_b200.locality import lpa_partition
        part = lpa_partition(a, 1)
        a, _ = P.apply_partition(a, None, part)
        print("lpa community-ordered layout", flush=True)
    grid = P.ProcessGrid(1, 1)
    dm = P.build_dist_matrices(a, [(0, a.n_rows)], grid)
    import paper_2504_04673_b200.engine as E
    if args.chunk:
        E.MAX_CHUNK = args.chunk
    E.SPMM_WINDOW_NNZ = args.window
    if args.order == "lpa":
        dm.fwd.row_order = "lpa"
    dp = device_plan(dm.fwd, grid, "1d-sparse")
    lib = L.lib()
    for f in args.f:
        ld = pad4(f) if args.ld_align == 0 else (f + args.ld_align - 1) // args.ld_align * args.ld_align
        h = torch.randn((a.n_rows, ld), device="cuda")
        h[:, f:] = 0
        z = torch.empty_like(h)
        for acc in args.acc:
            for slab in args.slab:
                def go():
                    L.check(lib.dg_spmm_run(dp._splan, L.ptr_array([h]), L.ptr_array([h]),
                                            L.ptr_array([z]), f, ld, ld, acc, slab, 0,
                                            L.stream_ptr()))
                go()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.reps):
                    go()
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / args.reps
                gather = 4.0 * f * a.nnz
                print(f"f={f} slab={slab} acc={acc} chunk={args.chunk}: {t:.3f} ms  "
                      f"gather {gather / t / 1e6:.0f} GB/s  nnz*f/s {a.nnz * f / t / 1e6:.3g} G",
                      flush=True)
        if args.slab_major and f > args.slab_major:
            sw = args.slab_major
            ns = (f + sw - 1) // sw
            slabs = [h[:, k * sw:min(f, (k + 1) * sw)].contiguous() for k in range(ns)]
            slabs = [torch.nn.functional.pad(x, (0, (-x.shape[1]) % 8)) for x in slabs]
            z2 = torch.zeros_like(z)

            def go_sm():
                for k, x in enumerate(slabs):
                    fk = min(f, (k + 1) * sw) - k * sw
                    L.check(lib.dg_spmm_run(dp._splan, L.ptr_array([x]), L.ptr_array([x]),
                                            L.ptr_array([z2[:, k * sw:].data_ptr()]), fk,
                                            x.shape[1], ld, 2, 0, 0, L.stream_ptr()))
            go_sm()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                go_sm()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / args.reps
            full = (f // sw) * sw          # a narrow last slab takes the <= 48-float kernel
            same = bool(torch.equal(z2[:, :full], z[:, :full]))
            print(f"f={f} slab-major {sw}-float slabs ({ns} launches): {t:.3f} ms  "
                  f"gather {4.0 * f * a.nnz / t / 1e6:.0f} GB/s  bitwise equal to row-major: {same}",
                  flush=True)
        if args.cusparse:
            import numpy as np
            sp = torch.sparse_csr_tensor(torch.from_numpy(a.row_ptr), torch.from_numpy(a.col_idx),
                                         torch.from_numpy(a.values.astype(np.float32)),
                                         size=(a.n_rows, a.n_cols), device="cuda")
            hd = h[:, :f].contiguous()
            torch.sparse.mm(sp, hd)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                zc = torch.sparse.mm(sp, hd)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / args.reps
            ref = z[:, :f]
            rel = float(((zc - ref).abs().max() / ref.abs().max()).item())
            print(f"f={f} cuSPARSE (torch.sparse.mm fp32): {t:.3f} ms  max rel diff vs ours {rel:.2e}",
                  flush=True)
            del sp


if __name__ == "__main__":
    main()
