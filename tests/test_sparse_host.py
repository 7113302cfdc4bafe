"""Host-side sparse helpers of the drop-in (sparse.py of the reference:
canonical CSR, builders, gcn_normalize, transpose_csr, nnz_cols) against
closed forms and dense scans -- the behaviours the reference's own
test_sparse.py pins, restated here."""

import numpy as np
import pytest

import paper_2504_04673_b200 as P


def _dense(a):
    d = np.zeros(a.shape)
    for r in range(a.n_rows):
        for k in range(a.row_ptr[r], a.row_ptr[r + 1]):
            d[r, a.col_idx[k]] += a.values[k]
    return d


def test_from_edges_empty_graph():
    a = P.csr_from_edges([], 5)
    assert a.shape == (5, 5) and a.nnz == 0
    assert np.array_equal(a.row_ptr, np.zeros(6, np.int64))


def test_from_edges_symmetrize_and_accumulate():
    edges = [(0, 1, 1.0), (1, 2, 2.0), (0, 1, 0.5), (3, 3, 4.0)]
    a = P.csr_from_edges(edges, 4, symmetrize=True)
    d = _dense(a)
    assert np.array_equal(d, d.T)
    assert d[0, 1] == 1.5 and d[1, 2] == 2.0 and d[3, 3] > 0
    rng = np.random.default_rng(0)
    b = P.csr_from_edges([edges[i] for i in rng.permutation(len(edges))], 4, symmetrize=True)
    assert P.csr_equal(a, b)                      # independent of edge order


def test_from_edges_rejects_out_of_range_and_drops_zero_sums():
    with pytest.raises(ValueError):
        P.csr_from_edges([(0, 7, 1.0)], 4)
    a = P.csr_from_edges([(0, 1, 1.0), (0, 1, -1.0), (2, 3, 1.0)], 4)
    assert a.nnz == 1 and _dense(a)[2, 3] == 1.0


@pytest.mark.parametrize("n,rp,ci,msg", [
    (3, [0, 2, 1, 2], [0, 1], "non-decreasing"),
    (2, [0, 2, 2], [1, 0], "strictly increasing"),
    (2, [0, 1, 2], [0, 5], "out of range"),
    (2, [0, 1], [0], "length"),
    (2, [0, 1, 1], [0, 1], "end at nnz"),
])
def test_canonical_form_validation(n, rp, ci, msg):
    with pytest.raises(ValueError, match=msg):
        P.CsrMatrix(n, 3, rp, ci, np.ones(len(ci)))


def test_normalize_isolated_and_two_vertex():
    a = P.gcn_normalize(P.csr_from_edges([], 1))
    assert a.nnz == 1 and a.values[0] == 1.0
    b = P.gcn_normalize(P.csr_from_edges([(0, 1, 1.0)], 2, symmetrize=True))
    assert np.allclose(_dense(b), np.full((2, 2), 0.5))


def test_normalize_matches_dense_formula_and_rejects_non_square():
    rng = np.random.default_rng(3)
    m = (rng.random((30, 30)) < 0.15) * rng.uniform(0.5, 2.0, (30, 30))
    m = np.triu(m, 1)
    m = m + m.T
    a = P.gcn_normalize(P.csr_from_dense(m))
    ai = m + np.eye(30)
    dinv = 1.0 / np.sqrt(ai.sum(1))
    assert np.allclose(_dense(a), dinv[:, None] * ai * dinv[None, :], rtol=1e-14, atol=0)
    with pytest.raises(ValueError):
        P.gcn_normalize(P.csr_from_dense(np.ones((2, 3))))


@pytest.mark.parametrize("seed", range(4))
def test_transpose_involution_and_rectangular(seed):
    rng = np.random.default_rng(seed)
    m = (rng.random((17, 23)) < 0.2) * rng.standard_normal((17, 23))
    a = P.csr_from_dense(m)
    t = P.transpose_csr(a)
    assert t.shape == (23, 17) and np.array_equal(_dense(t), m.T)
    assert P.csr_equal(P.transpose_csr(t), a)
    s = P.csr_from_dense(m[:17, :17] + m[:17, :17].T)
    assert P.csr_equal(P.transpose_csr(s), s)     # symmetric fixed point


def test_nnz_cols_matches_dense_scan():
    rng = np.random.default_rng(5)
    m = (rng.random((40, 40)) < 0.08) * 1.0
    m[3, 7] = 0.0
    a = P.csr_from_dense(m)
    bounds = [(0, 13), (13, 27), (27, 40)]
    for i, (r0, r1) in enumerate(bounds):
        for j, (c0, c1) in enumerate(bounds):
            got = P.nnz_cols(a, (i, j), bounds).indices
            want = np.flatnonzero((m[r0:r1, c0:c1] != 0).any(axis=0))
            assert np.array_equal(got, want), (i, j)


def test_nnz_cols_diagonal_and_dense_blocks():
    a = P.csr_from_dense(np.eye(8))
    bounds = [(0, 4), (4, 8)]
    assert len(P.nnz_cols(a, (0, 1), bounds)) == 0
    assert np.array_equal(P.nnz_cols(a, (1, 1), bounds).indices, np.arange(4))
    d = P.csr_from_dense(np.ones((8, 8)))
    assert np.array_equal(P.nnz_cols(d, (0, 1), bounds).indices, np.arange(4))


def test_nnz_cols_counts_structural_zeros():
    a = P.CsrMatrix(4, 4, [0, 1, 2, 2, 2], [1, 3], [0.0, 2.0])   # a stored zero at (0, 1)
    bounds = [(0, 2), (2, 4)]
    assert np.array_equal(P.nnz_cols(a, (0, 0), bounds).indices, [1])
    assert np.array_equal(P.nnz_cols(a, (0, 1), bounds).indices, [1])
    assert len(P.nnz_cols(a, (1, 0), bounds)) == 0
