"""The fused forward epilogue (SpMM + transform + ReLU in one
kernel, T never in HBM) gives the same numbers as SpMM followed by the
dense transform: the SpMM sums T identically and both accumulate z = t W
in ascending k in fp32 -- checked for the kernels directly (including
split rows, whose epilogue runs in the fix-up kernel) and for whole GCN
runs (p=1 thread driver, lock-step ranks, the CUDA-graph driver)."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P
import paper_2504_04673_b200.engine as E
from paper_2504_04673_b200 import graphgen
from paper_2504_04673_b200.gcn import GcnRun, _Dense

pytestmark = pytest.mark.gpu


def _plan(a):
    from paper_2504_04673_b200.plan import build_variant_plan
    grid = P.ProcessGrid(1, 1)
    dm = P.build_dist_matrices(a, [(0, a.n_rows)], grid)
    return E.DevicePlan(build_variant_plan(dm.fwd, grid, "1d-sparse"))


@pytest.mark.parametrize("f,n_out", [(16, 16), (16, 47), (13, 33), (16, 64), (15, 41)])
def test_fused_equals_spmm_then_dense(f, n_out):
    torch.cuda.set_device(0)
    # a star plus R-MAT: rows longer than one 1024-entry item exercise the
    # split-row (fix-up) epilogue
    n = 5000
    base = graphgen.rmat(12, 8, 3)
    rows = np.concatenate([base.row_of_nnz(), np.zeros(3000, np.int64)])
    cols = np.concatenate([base.col_idx, np.arange(1, 3001)])
    a = P.gcn_normalize(graphgen.symmetric_unit(n, rows, cols))
    a.values = a.values.astype(np.float32).astype(np.float64)
    dp = _plan(a)
    ld, ldo = E.pad4(f), E.pad4(n_out)
    h = E.to_device(np.random.default_rng(f).standard_normal((n, f)).astype(np.float32), ld)
    w = torch.zeros((ld, ldo), device="cuda")
    w[:f, :n_out] = torch.randn(f, n_out, device="cuda")
    t = dp.run({0: h}, f, ld)[0]
    z_ref, h_ref = _Dense(torch.device("cuda")).fwd(t, w, f, n_out, True)
    z = {0: torch.full((n, ldo), 7.0, device="cuda")}
    hr = {0: torch.full((n, ldo), 7.0, device="cuda")}
    dp.run_fused({0: h}, f, ld, w, n_out, ldo, z, hr)
    assert np.array_equal(z[0].cpu().numpy(), z_ref.cpu().numpy())
    assert np.array_equal(hr[0].cpu().numpy(), h_ref.cpu().numpy())
    assert not z[0][:, n_out:].any()
    assert dp.info[1] > 0                     # the graph has split rows


def test_fused_gcn_runs_identical():
    torch.cuda.set_device(0)
    a = P.gcn_normalize(graphgen.rmat(11, 8, 5))
    a.values = a.values.astype(np.float32).astype(np.float64)
    n = a.n_rows
    rng = np.random.default_rng(2)
    x = rng.standard_normal((n, 24)).astype(np.float32)
    y = rng.integers(0, 10, n)
    mask = np.ones(n, bool)
    cfg = P.TrainConfig(layers=4, hidden=16, lr=0.1, epochs=3, seed=4, variant="1d-sparse")
    out = {}
    for fuse in (False, True):
        for p, mode in ((1, "run"), (1, "graph"), (4, "lockstep")):
            gr = GcnRun(a, x, y, mask, cfg, p=p, fuse=fuse)
            run = {"run": gr.run, "graph": gr.run_graph, "lockstep": gr.run_lockstep}[mode]()
            out[(fuse, p, mode)] = gr.result(run)
            gr.close()
    for (fuse, p, mode), res in out.items():
        ref = out[(False, p, mode)]              # the same driver, unfused
        assert np.array_equal(res.losses, ref.losses), (fuse, p, mode)
        for w1, w2 in zip(res.weights, ref.weights):
            assert np.array_equal(w1, w2), (fuse, p, mode)
    # and the drivers agree with each other at p=1
    assert np.array_equal(out[(True, 1, "graph")].losses, out[(True, 1, "run")].losses)
