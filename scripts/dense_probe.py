"""Time the GCN step's dense kernels at the benchmark shapes: forward
transform (+ReLU), backward transform (+ReLU mask) and weight gradient,
TMA-fed (default) vs the register-staged kernels (dg_dense_legacy=1); HBM
GB/s counts the algorithmic bytes (tall operands read once, outputs written
once); xent too.  Inputs > L2 for the large shapes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04673_b200 import _lib as L  # noqa: E402
from paper_2504_04673_b200.engine import pad4  # noqa: E402
from paper_2504_04673_b200.gcn import _Dense, _Xent  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


flag = ctypes.c_int.in_dll(L.lib(), "dg_dense_legacy")
d = _Dense(torch.device("cuda"))
shapes = [(232965, 602, 16), (232965, 16, 41), (2449029, 100, 16), (2449029, 16, 16),
          (2449029, 16, 47)]
for n, fi, fo in shapes:
    li, lo = pad4(fi), pad4(fo)
    t = torch.randn(n, li, device="cuda")
    t[:, fi:] = 0
    w = torch.randn(li, lo, device="cuda")
    m = torch.randn(n, lo, device="cuda")
    m[:, fo:] = 0
    zp = torch.randn(n, li, device="cuda")
    for legacy in (0, 1):
        flag.value = legacy
        tag = "legacy" if legacy else "tma"
        ms = timed(lambda: d.fwd(t, w, fi, fo, True))
        gb = n * (fi + 2 * lo) * 4 / 1e9
        print(f"{tag:6s} fwd   n={n} K={fi} N={fo}: {ms:.3f} ms  {gb / ms:.2f} TB/s", flush=True)
        ms = timed(lambda: d.bwd(m, w, fi, fo, zp))
        gb = n * (fo + 2 * li) * 4 / 1e9
        print(f"{tag:6s} bwd   n={n} K={fo} N={fi}: {ms:.3f} ms  {gb / ms:.2f} TB/s", flush=True)
        ms = timed(lambda: d.wgrad(t, m, fi, fo, li, lo))
        gb = n * (fi + fo) * 4 / 1e9
        print(f"{tag:6s} wgrad n={n} K={fi} N={fo}: {ms:.3f} ms  {gb / ms:.2f} TB/s", flush=True)
    flag.value = 0
    del t, w, m, zp

for n, C in [(232965, 41), (2449029, 47)]:
    ld = pad4(C)
    x = torch.randn(n, ld, device="cuda")
    lab = torch.randint(0, C, (n,), device="cuda")
    mask = torch.ones(n, dtype=torch.uint8, device="cuda")
    g = torch.empty_like(x)
    st = torch.zeros(2, dtype=torch.float64, device="cuda")
    xe = _Xent(n, torch.device("cuda"))
    ms = timed(lambda: xe(x, C, lab, mask, n, g, st))
    print(f"xent n={n} C={C}: {ms:.3f} ms  {2 * n * C * 4 / 1e9 / ms:.2f} TB/s", flush=True)
    del x, g
