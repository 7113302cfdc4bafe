"""Fused SpMM + transform (+ReLU) vs SpMM followed by dense_rows on the
benchmark graphs, per (f, n_out) layer shape."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_04673_b200 as P  # noqa: E402
import paper_2504_04673_b200.engine as E  # noqa: E402
from paper_2504_04673_b200.gcn import _Dense  # noqa: E402
from paper_2504_04673_b200.plan import build_variant_plan  # noqa: E402


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


torch.cuda.set_device(0)
for wl, shapes in (("products", [(16, 16), (16, 47)]), ("reddit", [(16, 41), (16, 16)])):
    a = bench.make_graph(wl)
    if wl == "products":
        from paper_2504_04673_b200.locality import lpa_partition
        a, _ = P.apply_partition(a, None, lpa_partition(a, 1))
    grid = P.ProcessGrid(1, 1)
    dm = P.build_dist_matrices(a, [(0, a.n_rows)], grid)
    dp = E.DevicePlan(build_variant_plan(dm.fwd, grid, "1d-sparse"), max_ld=64)
    d = _Dense(torch.device("cuda"))
    n = a.n_rows
    for f, no in shapes:
        ld, ldo = E.pad4(f), E.pad4(no)
        h = torch.randn(n, ld, device="cuda")
        w = torch.zeros(ld, ldo, device="cuda")
        w[:f, :no] = torch.randn(f, no, device="cuda")
        t = torch.empty(n, ld, device="cuda")
        z = {0: torch.empty(n, ldo, device="cuda")}
        hr = {0: torch.empty(n, ldo, device="cuda")}
        t_sep = timed(lambda: d.fwd(dp.run({0: h}, f, ld, out={0: t})[0], w, f, no, True))
        t_spmm = timed(lambda: dp.run({0: h}, f, ld, out={0: t}))
        t_fused = timed(lambda: dp.run_fused({0: h}, f, ld, w, no, ldo, z, hr))
        print(f"{wl} {f}->{no}: SpMM {t_spmm:.3f} ms, SpMM + dense {t_sep:.3f} ms, "
              f"fused {t_fused:.3f} ms, split rows {dp.info[1]}", flush=True)
    del dp, a
    torch.cuda.empty_cache()
