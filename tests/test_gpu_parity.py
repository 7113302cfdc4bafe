"""CUDA path vs the reference (golden vectors from the real package) and
vs the CPU oracle, through the public API (which calls the C ABI).

Tolerance: |gpu - ref| <= 1e-5 * (|A| |H|)_ij + 1e-30,
the sound form of "rtol 1e-5 allowing reduction-order differences" for
fp32 storage; the SpMM accumulates in fp64, so in practice the error is a
single fp32 rounding of the output.  Volumes / ledgers: exact."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P
from paper_2504_04673_b200 import _lib

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def _part(g, key, n, k):
    asg = g[key + "__assign"] if k > 1 else np.zeros(n, np.int64)
    sizes = np.bincount(asg, minlength=k)
    bounds, pos = [], 0
    for s in sizes:
        bounds.append((pos, pos + int(s)))
        pos += int(s)
    return P.Partition(n, k, asg, g[key + "__perm"], bounds)


def _close(z, ref, mag):
    err = np.abs(z - ref)
    assert np.all(err <= RTOL * mag + 1e-30), float((err / (mag + 1e-300)).max())


def test_library_is_the_cuda_path():
    before = _lib.launch_count()
    a = P.csr_from_dense(np.eye(4))
    P.local_spmm(a, np.ones((4, 3)))
    assert _lib.launch_count() > before


def test_run_spmm_matches_reference_all_variants(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        a = g.csr(key + "__a", P.CsrMatrix)
        p, c, vi = (int(x) for x in g[key + "__cfg"])
        variant = P.VARIANTS[vi]
        part = _part(g, key, a.n_rows, p // c)
        run = P.run_spmm(a, g[key + "__h"], p, c, variant, partition=part)
        _close(run.z, g[key + "__z"], g[key + "__absz"])
        for (prim, name), ref in g.ledger_fields(key).items():
            assert np.array_equal(run.ledger.counters[prim][name], ref), (key, prim, name)


def test_aware_equals_oblivious_bitwise(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        a = g.csr(key + "__a", P.CsrMatrix)
        p, c, _ = (int(x) for x in g[key + "__cfg"])
        h = g[key + "__h"]
        fam = ("1d", "15d") if c == 1 else ("15d",)
        for f in fam:
            z1 = P.run_spmm(a, h, p, c, f"{f}-oblivious").z
            z2 = P.run_spmm(a, h, p, c, f"{f}-sparse").z
            assert np.array_equal(z1, z2), (key, f)


def test_c1_15d_equals_1d_bitwise_and_by_volume(spmm_golden):
    g = spmm_golden
    a = g.csr("c7__a", P.CsrMatrix)
    h = g["c7__h"]
    for flavor in ("oblivious", "sparse"):
        r1 = P.run_spmm(a, h, 4, 1, f"1d-{flavor}")
        r2 = P.run_spmm(a, h, 4, 1, f"15d-{flavor}")
        assert np.array_equal(r1.z, r2.z)
        for r in range(4):
            assert r1.ledger.rank_bytes_sent(r, "data") == r2.ledger.rank_bytes_sent(r, "data")


def test_zero_communication_on_clique_blocks(spmm_golden):
    g = spmm_golden
    a = g.csr("clique__a", P.CsrMatrix)
    run = P.run_spmm(a, g["clique__h"], 4, 1, "1d-sparse")
    assert run.ledger.total_bytes_sent() == 0.0
    import distgcn_oracle as O
    ref = O.serial_reference(O.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values),
                             g["clique__h"])
    np.testing.assert_allclose(run.z, ref, rtol=1e-6, atol=0)
    obl = P.run_spmm(a, g["clique__h"], 4, 1, "1d-oblivious")
    assert [obl.ledger.rank_bytes_sent(r, "data") for r in range(4)] == [3 * 6 * 2 * 8.0] * 4


def _rmat_case(scale, f, seed=1):
    import distgcn_oracle as O
    from paper_2504_04673_b200.graphgen import rmat
    a = P.gcn_normalize(rmat(scale, 16, 0))
    a.values = a.values.astype(np.float32).astype(np.float64)
    h = np.random.default_rng(seed).standard_normal((a.n_rows, f)).astype(np.float32)
    oa = O.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)
    return a, h.astype(np.float64), oa


@pytest.mark.parametrize("f", [1, 16, 41, 100])
def test_local_spmm_rmat_vs_oracle(f):
    """R-MAT-14 (config 1 graph) at several widths, one GPU, vs oracle."""
    import distgcn_oracle as O
    a, h, oa = _rmat_case(14, f)
    ref = O.local_spmm(oa, h)
    mag = O.local_spmm(O.Csr(oa.n_rows, oa.n_cols, oa.row_ptr, oa.col_idx, np.abs(oa.values)),
                       np.abs(h))
    z = P.local_spmm(a, h)
    _close(z, ref, mag)


def test_long_rows_split_deterministically():
    """A star (one row with every column) exercises the chunk split +
    fixup path; repeated runs are bitwise identical."""
    import distgcn_oracle as O
    n = 5000
    rows = np.concatenate([np.zeros(n - 1, np.int64), np.arange(1, n)])
    cols = np.concatenate([np.arange(1, n), np.zeros(n - 1, np.int64)])
    a = P.gcn_normalize(P.csr_from_coo(n, n, rows, cols, np.ones(rows.size)))
    a.values = a.values.astype(np.float32).astype(np.float64)
    h = np.random.default_rng(0).standard_normal((n, 24)).astype(np.float32).astype(np.float64)
    z1 = P.local_spmm(a, h)
    z2 = P.local_spmm(a, h)
    assert np.array_equal(z1, z2)
    oa = O.Csr(n, n, a.row_ptr, a.col_idx, a.values)
    mag = O.local_spmm(O.Csr(n, n, a.row_ptr, a.col_idx, np.abs(a.values)), np.abs(h))
    _close(z1, O.local_spmm(oa, h), mag)


def test_rmat14_distributed_volumes_and_values():
    """Config 1 (R-MAT-14, f=16, p=4) through run_spmm: values vs oracle,
    aware volume = 25,161 rows, 1.5D p=8 c=2 and p=16 c=4."""
    import distgcn_oracle as O
    a, h, oa = _rmat_case(14, 16)
    ref = O.serial_reference(oa, h)
    mag = O.serial_reference(O.Csr(oa.n_rows, oa.n_cols, oa.row_ptr, oa.col_idx,
                                   np.abs(oa.values)), np.abs(h))
    run = P.run_spmm(a, h, 4, 1, "1d-sparse")
    _close(run.z, ref, mag)
    assert run.ledger.total_bytes_sent("data") == 3_220_608
    for p, c in [(8, 2), (16, 4)]:
        r = P.run_spmm(a, h, p, c, "15d-sparse")
        _close(r.z, ref, mag)


def test_gcn_train_matches_reference(gcn_golden):
    g = gcn_golden
    for key in g.cases():
        a = g.csr(key + "__a", P.CsrMatrix)
        p, c, layers, hidden, epochs, seed, vi = (int(x) for x in g[key + "__cfg"])
        variant = (P.VARIANTS + ("serial",))[vi]
        cfg = P.TrainConfig(layers=layers, hidden=hidden, lr=float(g[key + "__lr"][0]),
                            epochs=epochs, seed=seed, variant=variant)
        part = None if variant == "serial" or p // c == 1 else _part(g, key, a.n_rows, p // c)
        res = P.train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"], cfg, p=p, c=c,
                      partition=part)
        np.testing.assert_allclose(res.losses, g[key + "__loss"], rtol=RTOL, atol=0)
        for li, w in enumerate(res.weights):
            ref = g[f"{key}__w{li}"]
            np.testing.assert_allclose(w, ref, rtol=RTOL, atol=RTOL * np.abs(ref).max())
        if res.ledger is not None:
            for (prim, name), ref in g.ledger_fields(key).items():
                assert np.array_equal(res.ledger.counters[prim][name], ref), (key, prim, name)
            for prim in ("p2p", "alltoallv", "broadcast", "allreduce"):
                hist = [row[f"{prim}_bytes"] for row in res.history]
                assert np.array_equal(hist, g[f"{key}__hist__{prim}"]), (key, prim)
            # replication invariant: bitwise-identical weights on every rank
            for per_rank in res.weights_per_rank[1:]:
                for w0, wr in zip(res.weights_per_rank[0], per_rank):
                    assert np.array_equal(w0, wr)


def test_training_is_deterministic(gcn_golden):
    g = gcn_golden
    key = "g0"
    a = g.csr(key + "__a", P.CsrMatrix)
    cfg = P.TrainConfig(layers=3, hidden=8, lr=0.05, epochs=4, seed=3, variant="15d-sparse")
    r1 = P.train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"], cfg, p=4, c=2)
    r2 = P.train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"], cfg, p=4, c=2)
    assert r1.history == r2.history
    for w1, w2 in zip(r1.weights, r2.weights):
        assert np.array_equal(w1, w2)


def test_softmax_xent_and_serial_gcn_api():
    import distgcn_oracle as O
    rng = np.random.default_rng(0)
    logits = rng.normal(size=(10, 4)).astype(np.float32).astype(np.float64)
    labels = rng.integers(4, size=10)
    mask = rng.random(10) < 0.6
    mask[0] = True
    loss, grad = P.softmax_xent(logits, labels, mask)
    l2, g2, _ = O.xent_parts(logits, labels, mask, int(mask.sum()))
    assert abs(loss - l2 / mask.sum()) < 1e-6
    np.testing.assert_allclose(grad, g2, atol=1e-7)
    with pytest.raises(ValueError, match="labels"):
        P.softmax_xent(np.zeros((2, 3)), np.array([0, 3]), np.ones(2, dtype=bool))
    net = P.SerialGcn(P.gcn_normalize(P.csr_from_dense(np.zeros((1, 1)))),
                      [np.eye(2), 0.5 * np.eye(2)])
    out = net.forward(np.array([[2.0, -3.0]]))
    np.testing.assert_allclose(out, [[1.0, 0.0]], atol=1e-7)
    with pytest.raises(RuntimeError, match="before forward"):
        P.SerialGcn(P.csr_from_dense(np.eye(2)), [np.eye(2)]).backward(np.zeros((2, 2)))


def test_transform_first_order_same_function(gcn_golden):
    """Extension: A^T (H W) instead of (A^T H) W -- same losses / weights as
    the reference within fp32 tolerance; lower forward volume."""
    g = gcn_golden
    for key in ("g0", "g2", "g4"):
        a = g.csr(key + "__a", P.CsrMatrix)
        p, c, layers, hidden, epochs, seed, vi = (int(x) for x in g[key + "__cfg"])
        variant = (P.VARIANTS + ("serial",))[vi]
        part = None if p // c == 1 else _part(g, key, a.n_rows, p // c)
        base = dict(layers=layers, hidden=hidden, lr=float(g[key + "__lr"][0]), epochs=epochs,
                    seed=seed, variant=variant)
        res = P.train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"],
                      P.TrainConfig(order="transform-first", **base), p=p, c=c, partition=part)
        np.testing.assert_allclose(res.losses, g[key + "__loss"], rtol=RTOL, atol=0)
        for li, w in enumerate(res.weights):
            ref = g[f"{key}__w{li}"]
            np.testing.assert_allclose(w, ref, rtol=RTOL, atol=RTOL * np.abs(ref).max())


def test_reduce_after_transform_same_function(gcn_golden):
    """Extension: 1.5D replica reduction after the transform --
    same losses / weights as the reference, smaller all-reduce volume."""
    g = gcn_golden
    for key in ("g2", "g3"):                       # 15d-sparse p=4 c=2; 15d-oblivious p=8 c=2
        a = g.csr(key + "__a", P.CsrMatrix)
        p, c, layers, hidden, epochs, seed, vi = (int(x) for x in g[key + "__cfg"])
        variant = P.VARIANTS[vi]
        part = _part(g, key, a.n_rows, p // c)
        base = dict(layers=layers, hidden=hidden, lr=float(g[key + "__lr"][0]), epochs=epochs,
                    seed=seed, variant=variant)
        ref = P.train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"],
                      P.TrainConfig(**base), p=p, c=c, partition=part)
        res = P.train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"],
                      P.TrainConfig(reduce_after_transform=True, **base), p=p, c=c,
                      partition=part)
        np.testing.assert_allclose(res.losses, g[key + "__loss"], rtol=RTOL, atol=0)
        for li, w in enumerate(res.weights):
            r = g[f"{key}__w{li}"]
            np.testing.assert_allclose(w, r, rtol=RTOL, atol=RTOL * np.abs(r).max())
        for per_rank in res.weights_per_rank[1:]:
            for w0, wr in zip(res.weights_per_rank[0], per_rank):
                assert np.array_equal(w0, wr)
        assert (res.ledger.total_bytes_sent("data") <= ref.ledger.total_bytes_sent("data"))
