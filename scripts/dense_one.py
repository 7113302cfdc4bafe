"""One dense transform at a benchmark shape (ncu target):
python scripts/dense_one.py fwd|wgrad n K N [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04673_b200.engine import pad4  # noqa: E402
from paper_2504_04673_b200.gcn import _Dense  # noqa: E402

kind, n, fi, fo = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
d = _Dense(torch.device("cuda"))
li, lo = pad4(fi), pad4(fo)
t = torch.randn(n, li, device="cuda")
w = torch.randn(li, lo, device="cuda")
m = torch.randn(n, lo, device="cuda")
fn = (lambda: d.fwd(t, w, fi, fo, True)) if kind == "fwd" else \
    (lambda: d.wgrad(t, m, fi, fo, li, lo))
fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(reps):
    fn()
e1.record()
torch.cuda.synchronize()
print(f"{kind} n={n} K={fi} N={fo}: {e0.elapsed_time(e1) / reps:.3f} ms", flush=True)
