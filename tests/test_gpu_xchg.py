"""The halo exchange kernel through the C-ABI (dg_xchg_run / dg_xchg_run_ctas):
every segment's rows land in the destination halo exactly (bit copies,
padding chunks included), whatever the CTA cap -- the overlapped phase runs
it with a small grid beside the own-block SpMM."""

import ctypes as C

import pytest
import torch

from paper_2504_04673_b200 import _lib as L
from paper_2504_04673_b200.engine import pad4

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("f", [10, 16, 47, 100, 602])
@pytest.mark.parametrize("ctas", [0, 1, 3, 48, 5000])
def test_xchg_rows_land_exactly(f, ctas):
    lib = L.lib()
    g = torch.Generator().manual_seed(f + ctas)
    ld = pad4(f)
    n_src = 3
    srcs = [torch.randn(1000 + 37 * i, ld, device="cuda") for i in range(n_src)]
    # segments: (source, rows or a contiguous range, destination buffer)
    segs = []
    for i in range(n_src):
        idx = torch.sort(torch.randperm(srcs[i].shape[0], generator=g)[:300 + 50 * i])[0]
        segs.append((i, idx.to(torch.int32).cuda(), None, i % 2))
    segs.append((1, None, (10, 400), 0))                    # idx NULL: rows 10..409
    segs.append((2, torch.zeros(0, dtype=torch.int32, device="cuda"), None, 1))   # empty
    counts = []
    for s, idx, rng, b in segs:
        counts.append(rng[1] if idx is None else idx.numel())
    off = [0, 0]
    dst_row0 = []
    for (s, idx, rng, b), c in zip(segs, counts):
        dst_row0.append(off[b])
        off[b] += c
    bufs = [torch.full((max(o, 1), ld), float("nan"), device="cuda") for o in off]
    n = len(segs)
    xh = C.c_void_p()
    L.check(lib.dg_xchg_plan_create(
        C.byref(xh), n, L.i32_array([s for s, *_ in segs]), L.i64_array(counts),
        (C.c_void_p * n)(*[0 if idx is None else idx.data_ptr() for _, idx, _, _ in segs]),
        L.i64_array([0 if rng is None else rng[0] for _, _, rng, _ in segs]),
        L.i32_array([b for *_, b in segs]), L.i64_array(dst_row0)))
    try:
        L.check(lib.dg_xchg_run_ctas(xh, L.ptr_array(srcs), n_src, L.ptr_array(bufs), 2, f, ld,
                                     0, ctas, L.stream_ptr()))
        torch.cuda.synchronize()
        for (s, idx, rng, b), c, d0 in zip(segs, counts, dst_row0):
            rows = (torch.arange(rng[0], rng[0] + rng[1], device="cuda") if idx is None
                    else idx.long())
            want = srcs[s][rows]
            got = bufs[b][d0:d0 + c]
            # whole 32-B chunks (the SpMM's 256-bit reads) carry the padding
            nf = min(ld, 8 * ((f + 7) // 8)) if ld % 8 == 0 else f
            assert torch.equal(got[:, :nf], want[:, :nf])
    finally:
        L.check(lib.dg_xchg_plan_destroy(xh))
