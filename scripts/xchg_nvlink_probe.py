"""NVLink evidence for the halo exchange kernel: ONE process drives GPU 0's
xchg_kernel (the production dg_xchg_run) storing the selected H rows into
halo buffers on the other GPUs through peer pointers -- the same stores the
multi-process path issues through CUDA-IPC mappings -- so ncu can capture
the kernel with its NVLink counters (ncu never wraps a multi-rank command).
Row lists: sorted random subsets (the shape of NnzCols lists), products-
shaped rows (f=100, 512-B pitch) and f=16.  Prints one line per case with
the CUDA-event time and GB/s of payload.

    python scripts/xchg_nvlink_probe.py                 # >= 2 GPUs
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,\
nvltx__bytes_data_user.sum -k regex:xchg python scripts/xchg_nvlink_probe.py --reps 1
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04673_b200 import _lib as L  # noqa: E402
from paper_2504_04673_b200.engine import pad4  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rows", type=int, default=306_128)      # one products block at p=8
    ap.add_argument("--ctas", type=int, default=0,
                    help="CTA cap over all segments (dg_xchg_run_ctas; 0: none)")
    args = ap.parse_args()
    ng = torch.cuda.device_count()
    if ng < 2:
        print("needs >= 2 GPUs")
        return
    lib = L.lib()
    torch.cuda.set_device(0)
    for d in range(1, ng):
        L.check(lib.dg_enable_peer(d))
    for f in (100, 16):
        ld = pad4(f)
        h = torch.randn(args.rows, ld, device="cuda:0")
        g = torch.Generator().manual_seed(f)
        # one segment per peer: 60% of the block's rows, sorted (NnzCols-like)
        segs = []
        for d in range(1, ng):
            idx = torch.sort(torch.randperm(args.rows, generator=g)[: int(0.6 * args.rows)])[0]
            segs.append(idx.to(torch.int32).cuda(0))
        halo = [torch.empty(s.numel(), ld, device=f"cuda:{d}")
                for d, s in zip(range(1, ng), segs)]
        xh = C.c_void_p()
        n = len(segs)
        L.check(lib.dg_xchg_plan_create(
            C.byref(xh), n, L.i32_array([0] * n), L.i64_array([s.numel() for s in segs]),
            (C.c_void_p * n)(*[s.data_ptr() for s in segs]), L.i64_array([0] * n),
            L.i32_array(list(range(n))), L.i64_array([0] * n)))
        st = torch.cuda.current_stream(0)

        def go():
            L.check(lib.dg_xchg_run_ctas(xh, L.ptr_array([h]), 1, L.ptr_array(halo), n, f, ld,
                                         1, args.ctas, C.c_void_p(st.cuda_stream)))
        go()
        for d in range(ng):
            torch.cuda.synchronize(d)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            go()
        e1.record(st)
        for d in range(ng):
            torch.cuda.synchronize(d)
        t = e0.elapsed_time(e1) / args.reps / 1e3
        payload = sum(s.numel() for s in segs) * f * 4
        wire = sum(s.numel() for s in segs) * ((f * 4 + 31) // 32 * 32)
        ok = all(torch.equal(hb[:, :f].cpu(), h[s.long()][:, :f].cpu())
                 for hb, s in zip(halo, segs))
        print(f"xchg f={f} ld={ld}: GPU0 -> {n} peer(s), {sum(s.numel() for s in segs):,} rows, "
              f"{t * 1e3:.3f} ms, payload {payload / t / 1e9:.0f} GB/s "
              f"(wire {wire / t / 1e9:.0f} GB/s, {wire / t / 1e9 / n:.0f} GB/s per peer link), "
              f"correct={ok}", flush=True)
        L.check(lib.dg_xchg_plan_destroy(xh))
        del h, halo, segs


if __name__ == "__main__":
    main()
