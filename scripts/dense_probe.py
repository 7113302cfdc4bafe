import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2504_04673_b200.gcn import _Dense
from paper_2504_04673_b200.engine import pad4
d = _Dense(torch.device("cuda"))
for n, fi, fo in [(232965, 602, 16), (2449029, 16, 48), (2449029, 48, 16), (2449029, 100, 16)]:
    li, lo = pad4(fi), pad4(fo)
    t = torch.randn(n, li, device="cuda")
    w = torch.randn(li, lo, device="cuda")
    z, h = d.fwd(t, w, fi, fo, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        z, h = d.fwd(t, w, fi, fo, True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    gb = (n * li + 2 * n * lo) * 4 / 1e9
    print(f"fwd n={n} K={fi} N={fo}: {ms:.3f} ms  {gb / ms:.2f} TB/s", flush=True)

# masked softmax cross-entropy (dg_xent) at the benchmark shapes
from paper_2504_04673_b200.gcn import _Xent  # noqa: E402
for n, C in [(232965, 41), (2449029, 47), (27764989, 172)]:
    ld = pad4(C)
    x = torch.randn(n, ld, device="cuda")
    lab = torch.randint(0, C, (n,), device="cuda")
    mask = torch.ones(n, dtype=torch.uint8, device="cuda")
    g = torch.empty_like(x)
    st = torch.zeros(2, dtype=torch.float64, device="cuda")
    xe = _Xent(n, torch.device("cuda"))
    xe(x, C, lab, mask, n, g, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        xe(x, C, lab, mask, n, g, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"xent n={n} C={C}: {ms:.3f} ms  {2 * n * ld * 4 / 1e9 / ms:.2f} TB/s", flush=True)
    del x, g
