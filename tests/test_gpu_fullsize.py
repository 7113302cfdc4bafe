"""Parity at BASELINE.json's full size (config 2, Reddit-shaped: 232,965
vertices, 115M stored nonzeros, f=602 and 16) through size-independent
properties -- the oracle's np.add.at would need ~554 GB of temporaries:

  * column checksum: sum_i Z[i,:] == sum_j (sum_i A^T[i,j]) H[j,:]  (fp64 host)
  * 2,000 sampled rows against an exact fp64 host product of those rows
  * 1D aware == oblivious bitwise on 4 emulated ranks, with the exact
    exchanged volume (aware elements <= oblivious)
"""

import os
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_04673_b200 as P  # noqa: E402
from paper_2504_04673_b200.engine import pad4  # noqa: E402
from paper_2504_04673_b200.plan import build_variant_plan  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def reddit():
    import bench
    a = bench.make_graph("reddit")
    return a


@pytest.mark.parametrize("f", [602, 16])
def test_full_size_checksum_and_sampled_rows(reddit, f):
    a = reddit
    n = a.n_rows
    rng = np.random.default_rng(f)
    h = rng.standard_normal((n, f), dtype=np.float32)
    hd = torch.zeros((n, pad4(f)), device="cuda")
    hd[:, :f] = torch.from_numpy(h).cuda()
    at = P.transpose_csr(a)                       # symmetric: at == a
    z = P.local_spmm(at, hd)[:, :f]               # CUDA tensor in -> CUDA tensor out
    zc = z.double().sum(0).cpu().numpy()
    colsum_at = np.bincount(at.col_idx, weights=at.values, minlength=n)   # sum_i A^T[i, j]
    ref = colsum_at @ h.astype(np.float64)
    mag = np.abs(colsum_at) @ np.abs(h.astype(np.float64))
    assert np.all(np.abs(zc - ref) <= 1e-6 * mag + 1e-9), float(np.abs(zc - ref).max())
    rows = rng.choice(n, size=2000, replace=False)
    zs = z[torch.from_numpy(rows).cuda(), :f].double().cpu().numpy()
    for k, r in enumerate(rows):
        lo, hi = at.row_ptr[r], at.row_ptr[r + 1]
        terms = at.values[lo:hi, None] * h[at.col_idx[lo:hi]].astype(np.float64)
        exact = terms.sum(0)
        bound = 1e-5 * np.abs(terms).sum(0) + 1e-30
        assert np.all(np.abs(zs[k] - exact) <= bound), r


def test_full_size_aware_equals_oblivious_bitwise(reddit):
    a = reddit
    n = a.n_rows
    f = 16
    h = np.random.default_rng(7).standard_normal((n, f), dtype=np.float32)
    za = P.run_spmm(a, torch.from_numpy(h).cuda(), 4, 1, "1d-sparse")
    zo = P.run_spmm(a, torch.from_numpy(h).cuda(), 4, 1, "1d-oblivious")
    assert torch.equal(za.z, zo.z)
    assert za.ledger.total_bytes_sent("data") <= zo.ledger.total_bytes_sent("data")
    grid = P.ProcessGrid(4, 1)
    vp = build_variant_plan(za.dm.fwd, grid, "1d-sparse", [])
    assert za.ledger.total_bytes_sent("data") == 8 * vp.elements(f)
