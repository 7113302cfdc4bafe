"""HBM-resident sharded path (sharded.py, config 5) vs the host plan
builder and the host GcnRun: plans bit-equal (halo layout, remapped
columns, values, NnzCols send lists), SpMM and GCN results bitwise equal,
and the sharded generator's output equal to the reference's
`gcn_normalize` (sparse.py:184-205) of its own pattern."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P
from paper_2504_04673_b200 import graphgen, sharded
from paper_2504_04673_b200.engine import DevicePlan, pad4, to_device
from paper_2504_04673_b200.plan import DistOperand, build_variant_plan
from paper_2504_04673_b200.runtime import ProcessGrid

pytestmark = pytest.mark.gpu


def _graph(scale=11, seed=3):
    a = P.gcn_normalize(graphgen.rmat(scale, 8, seed))
    a.values = a.values.astype(np.float32).astype(np.float64)
    return a


def _cpu(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.mark.parametrize("p", [1, 3, 4])
@pytest.mark.parametrize("variant", ["1d-sparse", "1d-oblivious"])
def test_sharded_plan_equals_host_plan(p, variant):
    a = _graph()
    grid = ProcessGrid(p, 1)
    bounds, _ = sharded.block_bounds(a.n_rows, p)
    host = build_variant_plan(DistOperand(P.transpose_csr(a), bounds), grid, variant)
    op = sharded.ShardedOperand(sharded.ShardedGraph.from_csr(a, p))
    dev = build_variant_plan(op, grid, variant)
    for r in range(p):
        h, d = host.ranks[r], dev.ranks[r]
        assert (h.n_rows, h.halo_rows, h.halo_off) == (d.n_rows, d.halo_rows, d.halo_off)
        assert np.array_equal(h.row_ptr, d.row_ptr)
        assert np.array_equal(h.col_ext, _cpu(d.col_ext))
        assert np.array_equal(h.val, _cpu(d.val))
    hs = {(s.src, s.dst): s for s in host.segments}
    ds = {(s.src, s.dst): s for s in dev.segments}
    assert hs.keys() == ds.keys()
    for k, s in hs.items():
        t = ds[k]
        assert (s.q, s.count, s.dst_row0) == (t.q, t.count, t.dst_row0), k
        if s.idx is None:
            assert t.idx is None
        else:
            assert np.array_equal(s.idx, _cpu(t.idx)), k
    for f in (1, 16, 41):
        assert host.elements(f) == dev.elements(f)


@pytest.mark.parametrize("p", [2, 4])
def test_sharded_spmm_bitwise_equals_host(p):
    a = _graph()
    grid = ProcessGrid(p, 1)
    bounds, _ = sharded.block_bounds(a.n_rows, p)
    f = 41
    ld = pad4(f)
    h = np.random.default_rng(0).standard_normal((a.n_rows, f)).astype(np.float32)
    hd = to_device(h, ld)
    hs = {r: hd[bounds[r][0]:bounds[r][1]] for r in range(p)}
    z_host = DevicePlan(build_variant_plan(DistOperand(P.transpose_csr(a), bounds), grid,
                                           "1d-sparse")).run(hs, f, ld)
    op = sharded.ShardedOperand(sharded.ShardedGraph.from_csr(a, p))
    z_dev = DevicePlan(build_variant_plan(op, grid, "1d-sparse")).run(hs, f, ld)
    for r in range(p):
        assert torch.equal(z_host[r], z_dev[r])


def test_sharded_gcn_equals_host_gcn():
    a = _graph(10, 5)
    p, f_in, classes = 4, 24, 7
    cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=3, seed=2, variant="1d-sparse")
    g = sharded.ShardedGraph.from_csr(a, p)
    x, y = sharded.sharded_inputs(g, f_in, classes, seed=4)
    xf = torch.cat([x[i] for i in range(p)])[:, :f_in].cpu().numpy()
    yf = torch.cat([y[i] for i in range(p)]).cpu().numpy()
    ref = P.train(a, xf, yf, np.ones(a.n_rows, bool), cfg, p=p)
    gr = sharded.sharded_gcn_run(g, x, y, f_in, classes, cfg)
    res = gr.result(gr.run())
    gr.close()
    assert np.array_equal(res.losses, ref.losses)
    for w1, w2 in zip(res.weights, ref.weights):
        assert np.array_equal(w1, w2)
    # the ledger's element counts are the host plan's (exact volumes)
    for prim in ref.ledger.counters:
        for name, v in ref.ledger.counters[prim].items():
            assert np.array_equal(res.ledger.counters[prim][name], v), (prim, name)


def test_chung_lu_sharded_is_normalised_symmetric():
    n, pairs, p = 20_000, 150_000, 3
    g = sharded.chung_lu_sharded(n, pairs, p, alpha=0.7, max_weight=900, seed=7)
    rp, off, cols, vals = [np.zeros(1, np.int64)], 0, [], []
    for i in range(p):
        brp, col, val = g.blocks[i]
        rp.append(brp[1:] + off)
        off += int(brp[-1])
        cols.append(col.cpu().numpy())
        vals.append(val.cpu().numpy())
    col = np.concatenate(cols).astype(np.int64)
    val = np.concatenate(vals)
    full = P.CsrMatrix(n, n, np.concatenate(rp), col, val.astype(np.float64))
    assert full.nnz == g.nnz_total
    assert pairs <= (full.nnz - n) // 2 <= pairs * 1.05
    rows = full.row_of_nnz()
    od = rows != col
    ref = P.gcn_normalize(P.csr_from_coo(n, n, rows[od], col[od], np.ones(int(od.sum()))))
    assert np.array_equal(ref.row_ptr, full.row_ptr)
    assert np.array_equal(ref.col_idx, full.col_idx)
    assert np.array_equal(ref.values.astype(np.float32), val)
    assert P.csr_equal(P.transpose_csr(full), full)
