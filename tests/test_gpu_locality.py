"""Locality schedules on the GPU: the SpMM row order (label-propagation
communities) and the length-bucketing window change which rows are in
flight together, never a number -- outputs and GCN losses are bitwise
identical with and without them, and both match the oracle."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P
import paper_2504_04673_b200.engine as E
from paper_2504_04673_b200 import graphgen
from paper_2504_04673_b200.locality import lpa_partition

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planted():
    torch.cuda.set_device(0)
    a, _ = graphgen.chung_lu_device(60_000, 60_000 * 15, alpha=0.55, max_weight=2000, seed=5,
                                    communities=24, p_in=0.8, return_communities=True)
    ah = P.gcn_normalize(a)
    ah.values = ah.values.astype(np.float32).astype(np.float64)
    return ah


def _spmm(a, h, f, order, window=0):
    from paper_2504_04673_b200.plan import build_variant_plan
    grid = P.ProcessGrid(1, 1)
    dm = P.build_dist_matrices(a, [(0, a.n_rows)], grid)
    old = E.SPMM_WINDOW_NNZ
    E.SPMM_WINDOW_NNZ = window
    try:
        dp = E.DevicePlan(build_variant_plan(dm.fwd, grid, "1d-sparse"), row_order=order)
    finally:
        E.SPMM_WINDOW_NNZ = old
    ld = E.pad4(f)
    hd = E.to_device(h, ld)
    return dp.run({0: hd}, f, ld)[0][:, :f].cpu().numpy()


@pytest.mark.parametrize("f", [16, 47, 100])
def test_row_order_and_window_bitwise_identical(planted, f):
    a = planted
    h = np.random.default_rng(f).standard_normal((a.n_rows, f)).astype(np.float32)
    base = _spmm(a, h, f, None)
    assert np.array_equal(base, _spmm(a, h, f, "lpa"))
    assert np.array_equal(base, _spmm(a, h, f, "lpa", window=1 << 14))
    assert np.array_equal(base, _spmm(a, h, f, None, window=1 << 40))   # one global window
    # and the oracle bound
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    import distgcn_oracle as O
    oa = O.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    ref = O.local_spmm(oa, h.astype(np.float64))
    mag = O.local_spmm(O.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, np.abs(a.values)),
                       np.abs(h.astype(np.float64)))
    assert np.all(np.abs(base - ref) <= 1e-5 * mag + 1e-30)


def test_gcn_row_order_same_losses_and_lpa_partition(planted):
    a = planted
    n = a.n_rows
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, 24)).astype(np.float32)
    y = rng.integers(0, 7, n)
    mask = np.ones(n, bool)
    cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=3, seed=2, variant="1d-sparse")
    from paper_2504_04673_b200.gcn import GcnRun
    runs = []
    for order in (None, "lpa"):
        gr = GcnRun(a, x, y, mask, cfg, p=2, row_order=order)
        runs.append(gr.result(gr.run()))
        gr.close()
    assert np.array_equal(runs[0].losses, runs[1].losses)
    for w0, w1 in zip(runs[0].weights, runs[1].weights):
        assert np.array_equal(w0, w1)
    # the graph-derived partition drives the reference's own train() API
    part = lpa_partition(a, 2)
    res = P.train(a, x, y, mask, cfg, p=2, partition=part)
    ser = P.train(a, x, y, mask, P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=3, seed=2,
                                               variant="serial"))
    assert np.allclose(res.losses, ser.losses, rtol=1e-5, atol=0)
