"""Accumulation error of the SpMM's summation modes on adversarial rows
(long, all-positive terms: no cancellation to hide rounding), against a
float64 reference.  The contract: |z - ref| <= 1e-5 *
(|A| |H|).  Two-level fp32 (acc=2, the default for rows >= 32 floats):
<= (32 + len/32) ulp of sum |terms| per 1024-entry item; fp64 folds
(acc=1): <= 4 ulp per window + fp64 noise."""

import numpy as np
import pytest
import torch

from paper_2504_04673_b200.engine import ACC_FP64, ACC_TWO_LEVEL, DevicePlan, _LocalPlan, pad4
from paper_2504_04673_b200.plan import RankOperand

pytestmark = pytest.mark.gpu
U = 2.0 ** -24


@pytest.mark.parametrize("acc", [ACC_FP64, ACC_TWO_LEVEL])
@pytest.mark.parametrize("f,deg", [(64, 1024), (602, 3000), (41, 777), (128, 100)])
def test_long_positive_rows(acc, f, deg):
    rng = np.random.default_rng(f + deg)
    n_rows, n_cols = 64, 5000
    rows = np.repeat(np.arange(n_rows), deg)
    cols = rng.integers(0, n_cols, size=rows.size)
    key = np.unique(rows * n_cols + cols)
    rows, cols = key // n_cols, key % n_cols
    vals = rng.uniform(0.5, 1.5, size=rows.size).astype(np.float32)
    rp = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=rp[1:])
    ro = RankOperand(0, 0, 0, n_rows, n_cols, rp, cols.astype(np.int32), vals, 0, {})
    plan = DevicePlan(_LocalPlan(ro), standalone=True, acc=acc)
    ld = pad4(f)
    h = torch.zeros((n_cols, ld), device="cuda")
    h[:, :f] = torch.rand((n_cols, f), device="cuda") + 0.5
    z = plan.run({0: h}, f, ld)[0][:, :f].double().cpu().numpy()
    import distgcn_oracle as O                     # CPU float64 checker
    a = O.Csr(n_rows, n_cols, rp, cols.astype(np.int64), vals.astype(np.float64))
    ref = O.local_spmm(a, h[:, :f].double().cpu().numpy())
    # all terms positive: sum |terms| == ref
    err = np.abs(z - ref) / ref
    assert err.max() <= 1e-5
    bound = (4 + 2) * U if acc == ACC_FP64 else (32 + 1024 / 32 + 2) * U
    assert err.max() <= bound, (err.max() / U, "ulp")


@pytest.mark.parametrize("f", [3, 16, 41, 47, 100, 602])
def test_padding_columns_stay_zero(f):
    """Z's padding up to the next 32-byte boundary is written (as zeros,
    from H's zero padding); wide rows' remaining pitch padding (128-B rows)
    is never written -- and never read: every consumer bounds its K / N by
    the logical width."""
    rng = np.random.default_rng(f)
    n = 3000
    rows = np.repeat(np.arange(n), 40)
    cols = rng.integers(0, n, size=rows.size)
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    ro = RankOperand(0, 0, 0, n, n, rp, cols.astype(np.int32),
                     rng.uniform(-1, 1, size=rows.size).astype(np.float32), 0, {})
    plan = DevicePlan(_LocalPlan(ro), standalone=True)
    ld = pad4(f)
    h = torch.zeros((n, ld), device="cuda")
    h[:, :f] = torch.randn((n, f), device="cuda")
    z = torch.full((n, ld), float("nan"), device="cuda")
    plan.run({0: h}, f, ld, out={0: z})
    assert torch.isfinite(z[:, :f]).all()
    top = min(ld, (f + 7) // 8 * 8)
    if top > f:
        assert not z[:, f:top].any(), "padding columns must be written as zeros"
