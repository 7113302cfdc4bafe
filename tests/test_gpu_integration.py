"""The INTEGRATION.md section-2 binding, executed: the unmodified reference
(`distgcn` from baseline/_ref) trains config 1 with its own runtime, ledger
and loop, its `local_spmm` swapped for the C-ABI kernel
(integration/distgcn_binding.py).  Losses must match the reference's own
NumPy run within rtol 1e-5 and the ledger must be identical (the binding
changes arithmetic, never communication)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "distgcn")),
                                 reason="baseline/_ref (the reference install) is absent")]


def test_binding_inside_reference_train_config1():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import distgcn as D
    assert os.path.abspath(D.__file__).startswith(os.path.abspath(REF))
    from paper_2504_04673_b200.graphgen import rmat
    import paper_2504_04673_b200 as P
    a = P.gcn_normalize(rmat(14, 16, 0))
    a.values = a.values.astype(np.float32).astype(np.float64)
    ra = D.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr.astype(np.int64),
                     a.col_idx.astype(np.int64), a.values)
    n = a.n_rows
    x = np.random.default_rng(1).standard_normal((n, 16)).astype(np.float32).astype(np.float64)
    y = np.random.default_rng(2).integers(0, 16, n)
    mask = np.ones(n, bool)
    cfg = D.TrainConfig(layers=3, hidden=16, lr=0.01, epochs=3, seed=1, variant="1d-sparse")
    ref = D.train(ra, x, y, mask, cfg, p=4)
    import distgcn_binding
    saved = {m: m.local_spmm for m in (D, D.sparse, D.spmm, D.gcn)}
    calls = {"n": 0}
    orig = distgcn_binding.local_spmm

    def counted(a_, h_):
        calls["n"] += 1
        return orig(a_, h_)

    distgcn_binding.local_spmm = counted
    try:
        distgcn_binding.install(D)
        got = D.train(ra, x, y, mask, cfg, p=4)
    finally:
        for m, fn in saved.items():
            m.local_spmm = fn
        distgcn_binding.local_spmm = orig
    # every block multiply of every phase went through the C ABI:
    # 3 epochs x 4 phases x 4 ranks x 4 source blocks (1d-sparse, spmm.py:188-190)
    assert calls["n"] == 3 * 4 * 4 * 4
    rl = np.array([h["loss"] for h in ref.history])
    gl = np.array([h["loss"] for h in got.history])
    assert np.allclose(gl, rl, rtol=1e-5, atol=0), (gl, rl)
    assert got.ledger.to_dict() == ref.ledger.to_dict()
    for wg, wr in zip(got.weights, ref.weights):
        assert np.max(np.abs(wg - wr)) <= 1e-5 * np.max(np.abs(wr))
