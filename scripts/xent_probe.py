"""Time dg_xent (masked softmax cross-entropy + gradient) at the benchmark
shapes; the ncu target for the loss kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_04673_b200.engine import pad4  # noqa: E402
from paper_2504_04673_b200.gcn import _Xent  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for n, C in [(2449029, 47), (232965, 41)]:
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
    for _ in range(reps):
        xe(x, C, lab, mask, n, g, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"xent n={n} C={C}: {ms:.3f} ms  {(2 * n * ld * 4 + 9 * n) / 1e9 / ms:.2f} TB/s", flush=True)
