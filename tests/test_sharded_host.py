"""Host logic of the sharded (HBM-resident) plan builder, run with the CPU
standing in for the device: the halo layout, remapped columns, values and
NnzCols send lists must equal the host plan builder's (plan.py, which
follows spmm.py:80-130) bit for bit, for both 1D variants and ragged p."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P
from paper_2504_04673_b200 import graphgen, sharded
from paper_2504_04673_b200.plan import DistOperand, build_variant_plan
from paper_2504_04673_b200.runtime import ProcessGrid


class _OneProc:
    multi = False
    size, proc = 1, 0

    def all_gather_object(self, obj):
        return [obj]

    def local_ranks(self, p):
        return list(range(p))

    def init(self):
        return self


@pytest.fixture
def cpu_dev(monkeypatch):
    monkeypatch.setattr(sharded, "_dev", lambda: torch.device("cpu"))


def _graph(scale, seed):
    a = P.gcn_normalize(graphgen.rmat(scale, 8, seed))
    a.values = a.values.astype(np.float32).astype(np.float64)
    return a


def _shard(a, p):
    bounds, _ = sharded.block_bounds(a.n_rows, p)
    blocks = {}
    for i, (r0, r1) in enumerate(bounds):
        lo, hi = int(a.row_ptr[r0]), int(a.row_ptr[r1])
        blocks[i] = ((a.row_ptr[r0:r1 + 1] - lo).astype(np.int64),
                     torch.from_numpy(a.col_idx[lo:hi].astype(np.int32)),
                     torch.from_numpy(a.values[lo:hi].astype(np.float32)))
    return sharded.ShardedGraph(a.n_rows, p, blocks, a.nnz, _OneProc())


@pytest.mark.parametrize("p", [1, 2, 3, 5])
@pytest.mark.parametrize("variant", ["1d-sparse", "1d-oblivious"])
def test_sharded_plan_equals_host_plan_cpu(cpu_dev, p, variant):
    a = _graph(9, p)
    grid = ProcessGrid(p, 1)
    bounds, _ = sharded.block_bounds(a.n_rows, p)
    assert bounds == P.block_partition(a.n_rows, p).boundaries
    host_op = DistOperand(P.transpose_csr(a), bounds)
    host = build_variant_plan(host_op, grid, variant)
    op = sharded.ShardedOperand(_shard(a, p))
    dev = build_variant_plan(op, grid, variant)
    for r in range(p):
        h, d = host.ranks[r], dev.ranks[r]
        assert (h.n_rows, h.halo_rows, h.halo_off) == (d.n_rows, d.halo_rows, d.halo_off)
        assert np.array_equal(h.row_ptr, d.row_ptr)
        assert np.array_equal(h.col_ext, d.col_ext.numpy())
        assert np.array_equal(h.val, d.val.numpy())
    ds = {(s.src, s.dst): s for s in dev.segments}
    assert {(s.src, s.dst) for s in host.segments} == set(ds)
    for s in host.segments:
        t = ds[(s.src, s.dst)]
        assert (s.q, s.count, s.dst_row0) == (t.q, t.count, t.dst_row0)
        if s.idx is None:
            assert t.idx is None
        else:
            assert np.array_equal(s.idx, t.idx.numpy())
    for (i, q), lst in host_op.nnz_cols.items():
        assert op.nnz_cols[(i, q)].size == (lst.size if i != q else 0) or i == q


def test_sharded_operand_rejects_asymmetric(cpu_dev):
    a = P.csr_from_dense(np.triu(np.ones((6, 6))))
    with pytest.raises(ValueError, match="symmetric"):
        sharded.ShardedOperand(_shard(a, 2))


def test_sharded_rejects_15d(cpu_dev):
    a = _graph(7, 1)
    op = sharded.ShardedOperand(_shard(a, 4))
    with pytest.raises(ValueError, match="1D"):
        build_variant_plan(op, ProcessGrid(4, 2), "15d-sparse")


@pytest.mark.parametrize("p", [1, 3])
def test_chung_lu_sharded_normalised_symmetric_cpu(cpu_dev, p):
    n, pairs = 3000, 20_000
    g = sharded.chung_lu_sharded(n, pairs, p, alpha=0.7, max_weight=300, seed=7,
                                 world=_OneProc())
    rp, off, cols, vals = [np.zeros(1, np.int64)], 0, [], []
    for i in range(p):
        brp, col, val = g.blocks[i]
        rp.append(brp[1:] + off)
        off += int(brp[-1])
        cols.append(col.numpy())
        vals.append(val.numpy())
    col = np.concatenate(cols).astype(np.int64)
    val = np.concatenate(vals)
    full = P.CsrMatrix(n, n, np.concatenate(rp), col, val.astype(np.float64))
    assert full.nnz == g.nnz_total
    assert pairs <= (full.nnz - n) // 2 <= pairs * 1.2
    rows = full.row_of_nnz()
    od = rows != col
    ref = P.gcn_normalize(P.csr_from_coo(n, n, rows[od], col[od], np.ones(int(od.sum()))))
    assert np.array_equal(ref.row_ptr, full.row_ptr)
    assert np.array_equal(ref.col_idx, full.col_idx)
    assert np.array_equal(ref.values.astype(np.float32), val)
    assert P.csr_equal(P.transpose_csr(full), full)


class _Shared:
    def __init__(self, size):
        import threading
        self.size, self.bar, self.slots = size, threading.Barrier(size), [None] * size


class _ProcView:
    """One simulated process of a `size`-process world (threads stand in
    for processes; all_gather_object through a barrier)."""

    multi = True

    def __init__(self, sh, proc):
        self.sh, self.proc, self.size = sh, proc, sh.size

    def all_gather_object(self, obj):
        self.sh.bar.wait()
        self.sh.slots[self.proc] = obj
        self.sh.bar.wait()
        out = list(self.sh.slots)
        self.sh.bar.wait()
        return out

    def proc_of(self, r, p):
        return (r * self.size) // p

    def local_ranks(self, p):
        return [r for r in range(p) if self.proc_of(r, p) == self.proc]

    def init(self):
        return self


@pytest.mark.parametrize("size,p", [(2, 4), (3, 3)])
def test_chung_lu_sharded_multiprocess_same_graph(cpu_dev, size, p):
    """Every process draws the same graph (counter-based generator) and
    keeps only its rows; the union equals the one-process graph, and the
    sharded operands pass the sender/receiver cross-check."""
    import threading
    n, pairs = 2500, 15_000
    one = sharded.chung_lu_sharded(n, pairs, p, alpha=0.7, max_weight=300, seed=3,
                                   world=_OneProc())
    sh = _Shared(size)
    res, errs = [None] * size, []

    def run(q):
        try:
            g = sharded.chung_lu_sharded(n, pairs, p, alpha=0.7, max_weight=300, seed=3,
                                         world=_ProcView(sh, q))
            res[q] = (g, sharded.ShardedOperand(g))
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    ts = [threading.Thread(target=run, args=(q,)) for q in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    got = {}
    for g, _ in res:
        got.update(g.blocks)
        assert g.nnz_total == one.nnz_total
    assert sorted(got) == list(range(p))
    for i in range(p):
        assert np.array_equal(got[i][0], one.blocks[i][0])
        assert torch.equal(got[i][1], one.blocks[i][1])
        assert torch.equal(got[i][2], one.blocks[i][2])
    op1 = sharded.ShardedOperand(one)
    for _, op in res:
        assert np.array_equal(op.counts, op1.counts)
