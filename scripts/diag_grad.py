"""Diagnostic: locate a weight-gradient mismatch of one products-shaped
epoch.  Records every wgrad / bwd / fwd call of GcnRun (inputs copied to
the host as float64) and checks each call against float64 math on its own
inputs, then chains the reference."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_04673_b200 as P  # noqa: E402
from paper_2504_04673_b200 import gcn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "products"
torch.cuda.set_device(0)
# 1. isolated dense_tn at the shapes of the products epoch
d = gcn._Dense(torch.device("cuda", 0))
for n, K, N, ldk, ldn in [(2449029, 16, 16, 16, 16), (2449029, 16, 47, 16, 48),
                          (2449029, 100, 16, 128, 16), (300000, 16, 16, 16, 16)]:
    h = torch.randn(n, ldk, device="cuda")
    h[:, K:] = 0
    m = torch.randn(n, ldn, device="cuda")
    m[:, N:] = 0
    y = d.wgrad(h, m, K, N, ldk, ldn)[:K, :N].double()
    ref = (h[:, :K].double().T @ m[:, :N].double())
    mag = (h[:, :K].double().abs().T @ m[:, :N].double().abs())
    print(f"wgrad n={n} K={K} N={N}: max err/mag {float(((y - ref).abs() / mag).max()):.2e}",
          flush=True)
# 2. the epoch, call by call
a = bench.make_graph(name)
wl = bench.WORKLOADS[name]
x, yl, mask = bench.make_inputs(wl, a.n_rows)
log = []
of, ob, ow = gcn._Dense.fwd, gcn._Dense.bwd, gcn._Dense.wgrad


def fwd(self, t, w, f_in, f_out, relu, z=None):
    zz, hh = of(self, t, w, f_in, f_out, relu, z)
    torch.cuda.synchronize()
    log.append(("fwd", t[:, :f_in].double().cpu(), w[:f_in, :f_out].double().cpu(),
                zz[:, :f_out].double().cpu()))
    return zz, hh


def bwd(self, m, w, f_in, f_out, zprev):
    g = ob(self, m, w, f_in, f_out, zprev)
    torch.cuda.synchronize()
    log.append(("bwd", m[:, :f_out].double().cpu(), w[:f_in, :f_out].double().cpu(),
                g[:, :f_in].double().cpu(), zprev[:, :f_in].double().cpu()))
    return g


def wgrad(self, h, m, f_in, f_out, ld_in, ld_out):
    y = ow(self, h, m, f_in, f_out, ld_in, ld_out)
    torch.cuda.synchronize()
    log.append(("wgrad", h[:, :f_in].double().cpu(), m[:, :f_out].double().cpu(),
                y[:f_in, :f_out].double().cpu()))
    return y


gcn._Dense.fwd, gcn._Dense.bwd, gcn._Dense.wgrad = fwd, bwd, wgrad
cfg = P.TrainConfig(layers=wl["layers"], hidden=wl["hidden"], lr=100.0, epochs=1, seed=1)
gr = gcn.GcnRun(a, x, yl, mask, cfg, p=1)
gr.result(gr.run())
for e in log:
    if e[0] == "fwd":
        _, t, w, z = e
        ref = t @ w
        mag = t.abs() @ w.abs()
    elif e[0] == "bwd":
        _, m, w, g, zp = e
        ref = (m @ w.T) * (zp > 0)
        mag = m.abs() @ w.abs().T
        z = g
    else:
        _, h, m, z = e
        ref = h.T @ m
        mag = h.abs().T @ m.abs()
    err = float(((z - ref).abs() / (mag + 1e-30)).max())
    print(e[0], tuple(z.shape), f"max err/mag {err:.2e}", flush=True)
# 3. the float64 reference chain (scipy), with its own relu masks and with
#    the GPU's (a relu mask flips where z is within rounding of 0)
import scipy.sparse as sp  # noqa: E402
n = a.n_rows
m_ = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(n, n))
mt = m_.T.tocsr()
fw = [e for e in log if e[0] == "fwd"]
wg = [e for e in log if e[0] == "wgrad"][::-1]          # layer order 0..L-1
ws = [e[2].numpy() for e in fw]
zs_gpu = [e[3].numpy() for e in fw]
xs = x.astype(np.float64)
for use_gpu_masks in (False, True):
    hs, zs = [xs], []
    for l, w in enumerate(ws):
        z = mt @ (hs[-1] @ w)
        zs.append(z)
        if l < len(ws) - 1:
            msk = (zs_gpu[l] > 0) if use_gpu_masks else (z > 0)
            flips = int(((z > 0) != (zs_gpu[l] > 0)).sum())
            near = float(np.abs(z[(z > 0) != (zs_gpu[l] > 0)]).max()) if flips else 0.0
            if not use_gpu_masks:
                print(f"layer {l}: relu mask flips {flips} of {z.size} (max |z| there {near:.2e})")
            hs.append(z * msk)
        else:
            hs.append(z)
    lg = hs[-1]
    sh = lg - lg.max(1, keepdims=True)
    e = np.exp(sh)
    g = e / e.sum(1, keepdims=True)
    g[np.arange(n), yl] -= 1
    g /= n
    for l in range(len(ws) - 1, -1, -1):
        mm = m_ @ g
        yr = hs[l].T @ mm
        mag = np.abs(hs[l]).T @ (abs(m_) @ np.abs(g))
        yg = wg[l][3].numpy()
        print(f"gpu_masks={use_gpu_masks} Y_{l}: max err/mag {np.max(np.abs(yg - yr) / mag):.2e}",
              flush=True)
        if l > 0:
            msk = (zs_gpu[l - 1] > 0) if use_gpu_masks else (zs[l - 1] > 0)
            g = (mm @ ws[l].T) * msk
