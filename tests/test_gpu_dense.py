"""Numerics of the GCN step kernels (dense transforms, xent) against a
plain PyTorch float64 reference of the same op.  Tolerance: rtol 1e-5
scaled by the sum of |terms| (fp32 storage, reduction-order differences)."""

import numpy as np
import pytest
import torch

from paper_2504_04673_b200 import _lib as L
from paper_2504_04673_b200.engine import pad4
from paper_2504_04673_b200.gcn import _Dense, _Xent

pytestmark = pytest.mark.gpu


def _pad(x, ld):
    out = torch.zeros((x.shape[0], ld), device="cuda")
    out[:, :x.shape[1]] = x
    return out


@pytest.fixture(params=["tma", "legacy"])
def dense_path(request):
    """The TMA-fed kernels (default) and the register-staged ones."""
    import ctypes
    flag = ctypes.c_int.in_dll(L.lib(), "dg_dense_legacy")
    flag.value = int(request.param == "legacy")
    yield request.param
    flag.value = 0


@pytest.mark.parametrize("n,fi,fo", [(1000, 602, 16), (777, 16, 41), (5000, 100, 16),
                                     (333, 16, 47), (64, 3, 2), (1, 16, 16), (3001, 16, 172),
                                     (1500, 128, 16), (700, 16, 250), (257, 41, 7),
                                     (20000, 602, 16), (9000, 16, 64), (4099, 48, 33)])
def test_dense_fwd_bwd_wgrad(n, fi, fo, dense_path):
    torch.manual_seed(n + fi + fo)
    d = _Dense(torch.device("cuda"))
    l0 = L.launch_count()
    li, lo = pad4(fi), pad4(fo)
    t = _pad(torch.randn(n, fi, device="cuda"), li)
    w = torch.zeros((li, lo), device="cuda")
    w[:fi, :fo] = torch.randn(fi, fo, device="cuda")
    z, h = d.fwd(t, w, fi, fo, True)
    ref = t.double() @ w.double()
    mag = t.double().abs() @ w.double().abs()
    assert torch.all((z.double() - ref).abs() <= 1e-5 * mag + 1e-30)
    assert torch.equal(h, torch.clamp_min(z, 0.0))
    assert not z[:, fo:].any()
    m = _pad(torch.randn(n, fo, device="cuda"), lo)
    zp = _pad(torch.randn(n, fi, device="cuda"), li)
    g = d.bwd(m, w, fi, fo, zp)
    ref = (m.double() @ w.double().T) * (zp.double() > 0)
    mag = m.double().abs() @ w.double().abs().T
    assert torch.all((g.double() - ref).abs() <= 1e-5 * mag + 1e-30)
    assert not g[:, fi:].any()
    y = d.wgrad(t, m, fi, fo, li, lo)
    ref = t.double().T @ m.double()
    mag = t.double().abs().T @ m.double().abs()
    assert y.shape == (li, lo)
    assert torch.all((y.double() - ref).abs() <= 1e-5 * mag + 1e-30)
    assert not y[fi:, :].any() and not y[:, fo:].any()
    y2 = d.wgrad(t, m, fi, fo, li, lo)
    assert torch.equal(y, y2)                      # deterministic
    # fwd: dense_rows (or cuBLAS); bwd: dense_rows (or cuBLAS + dg_relu_grad_mul); wgrad: 2
    ours = int(d._rows_ok(fi, fo)) + 1 + 2 * 2 * int(fo <= 64)
    assert L.launch_count() - l0 == ours           # our kernels (cuBLAS only for N > 64)



@pytest.mark.parametrize("n,C", [(10, 4), (1000, 41), (4097, 47), (300, 16), (50, 172),
                                 (20, 600)])
def test_xent_against_torch(n, C):
    torch.manual_seed(C)
    ld = pad4(C)
    x = _pad(torch.randn(n, C, device="cuda") * 3, ld)
    lab = torch.randint(0, C, (n,), device="cuda")
    mask = (torch.rand(n, device="cuda") < 0.7)
    mask[0] = True
    denom = int(mask.sum())
    g = torch.empty_like(x)
    stats = torch.zeros(2, dtype=torch.float64, device="cuda")
    _Xent(n, torch.device("cuda"))(x, C, lab, mask.to(torch.uint8), denom, g, stats)
    xd = x[:, :C].double()
    lsm = torch.log_softmax(xd, 1)
    loss = -(lsm[mask, lab[mask]]).sum()
    assert abs(float(stats[0]) - float(loss)) <= 1e-6 * abs(float(loss)) + 1e-9
    gr = torch.softmax(xd, 1)
    gr[torch.arange(n), lab] -= 1
    gr = gr / denom * mask[:, None]
    assert torch.allclose(g[:, :C].double(), gr, rtol=1e-5, atol=1e-7)
    assert not g[:, C:].any()
    corr = int(((xd.argmax(1) == lab) & mask).sum())
    assert float(stats[1]) == corr


@pytest.mark.parametrize("C", [3, 41, 47, 172])
def test_xent_ties_and_pad_garbage(C):
    """Tied maxima pick the first class (numpy argmax), -inf logits add
    nothing, and NaN in the padding columns never reaches the outputs."""
    torch.manual_seed(7 + C)
    n, ld = 999, pad4(C) + 4
    x = torch.full((n, ld), float("nan"), device="cuda")
    x[:, :C] = torch.randint(0, 3, (n, C), device="cuda").float()
    x[::5, C // 2] = float("-inf")
    lab = torch.randint(0, C, (n,), device="cuda")
    lab[::5] = (C // 2 + 1) % C                    # finite loss: the label logit is finite
    mask = torch.rand(n, device="cuda") < 0.6
    denom = int(mask.sum())
    g = torch.full_like(x, float("nan"))
    stats = torch.zeros(2, dtype=torch.float64, device="cuda")
    _Xent(n, torch.device("cuda"))(x, C, lab, mask.to(torch.uint8), denom, g, stats)
    xd = x[:, :C].double()
    loss = -(torch.log_softmax(xd, 1)[mask, lab[mask]]).sum()
    assert abs(float(stats[0]) - float(loss)) <= 1e-6 * abs(float(loss)) + 1e-9
    gr = torch.softmax(xd, 1)
    gr[torch.arange(n), lab] -= 1
    gr = gr / denom * mask[:, None]
    assert torch.allclose(g[:, :C].double(), gr, rtol=1e-5, atol=1e-7)
    assert not g[:, C:].any()
    first = xd.cpu().numpy().argmax(1)
    corr = int(((torch.from_numpy(first).cuda() == lab) & mask).sum())
    assert float(stats[1]) == corr
