"""HBM-resident sharded graphs: the path for graphs too large to stage
through host memory (config 5, ogbn-papers100M-shaped: 111M vertices,
3.3B stored nonzeros).

The reference builds everything on the host: the generator / loader, then
`gcn_normalize` (sparse.py:184-205), `apply_partition` (partition.py:231-254)
and `build_dist_matrices` / `_extract_operand` (spmm.py:80-117) with its
`np.unique` NnzCols lists (spmm.py:103).  At papers scale those host arrays
alone are ~80 GB per process.  Here every process builds only the block rows
it hosts, on its own GPU, with the same definitions:

* block partition, sizes differing by at most one (partition.py:154-161);
* Â = D^-1/2 (A + I) D^-1/2 with degrees after the self-loops and the two
  scale factors grouped (sparse.py:196-204), values rounded once to fp32;
* NnzCols(i, q) = sorted distinct columns of block row i inside block q
  (spmm.py:103), and the rows block s sends to d are NnzCols(d, s) -- by
  the symmetry of Â these are the rows of block s with an entry in block d,
  so a sender derives its own lists from its own block row; the receivers'
  and senders' counts are cross-checked (p x p, all-gathered).

The result plugs into the same `DevicePlan` / `GcnRun` machinery as the
host-built plans (`ShardedOperand.build_variant_plan` returns a
`plan.VariantPlan` whose hosted operands are CUDA tensors) and is checked
against the host plan builder bit for bit (tests/test_gpu_sharded.py).
1D variants only (c = 1), as config 5 specifies.
"""

from __future__ import annotations

import numpy as np
import torch

from .plan import RankOperand, Segment, VariantPlan, validate_variant_grid
from .runtime import ProcessGrid

__all__ = ["ShardedGraph", "ShardedOperand", "ShardedDistMatrices", "chung_lu_sharded",
           "papers_shaped_sharded", "block_bounds", "sharded_gcn_run", "sharded_inputs"]

_CHUNK = 1 << 27          # pairs drawn per generator call


def _dev():
    """The current CUDA device (the tests' host-logic check substitutes the
    CPU here; the compute path itself always runs in the CUDA library)."""
    return torch.device("cuda", torch.cuda.current_device())


def block_bounds(n, k):
    """partition.py:154-161: the first n mod k parts take the extra vertex."""
    base, rem = divmod(int(n), int(k))
    sizes = [base + 1] * rem + [base] * (k - rem)
    starts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return [(int(starts[i]), int(starts[i + 1])) for i in range(k)], starts


class ShardedGraph:
    """Â split into p block rows; this process holds the CSR of the block
    rows it hosts, in HBM: blocks[i] = (row_ptr int64 host, col int32 CUDA
    (global ids, ascending per row), val fp32 CUDA)."""

    def __init__(self, n, p, blocks, nnz_total, world):
        self.n, self.p = int(n), int(p)
        self.boundaries, self.starts = block_bounds(n, p)
        self.blocks = blocks
        self.nnz_total = int(nnz_total)
        self.world = world

    @classmethod
    def from_csr(cls, a, p, world=None):
        """Shard a host CsrMatrix (tests; small graphs): the hosted block
        rows of `a`, uploaded as they are (no normalisation)."""
        from .dist import world as _world
        w = world or _world().init()
        dev = _dev()
        bounds, _ = block_bounds(a.n_rows, p)
        hosted = w.local_ranks(p) if w.multi else range(p)
        blocks = {}
        for i in hosted:
            r0, r1 = bounds[i]
            lo, hi = int(a.row_ptr[r0]), int(a.row_ptr[r1])
            rp = (a.row_ptr[r0:r1 + 1] - lo).astype(np.int64)
            col = torch.from_numpy(a.col_idx[lo:hi].astype(np.int32)).to(dev)
            val = torch.from_numpy(a.values[lo:hi].astype(np.float32)).to(dev)
            blocks[i] = (rp, col, val)
        return cls(a.n_rows, p, blocks, a.nnz, w)

    def release(self):
        """Drop the block CSR (after the device plans hold their copies)."""
        self.blocks = {i: None for i in self.blocks}


def _s64(c):
    return c - (1 << 64) if c >= (1 << 63) else c


_GOLD, _MIX1, _MIX2 = _s64(0x9E3779B97F4A7C15), _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB)


def _splitmix64(x):
    """splitmix64 finaliser on int64 tensors (two's-complement wraparound;
    logical shifts by masking): a counter-based generator whose output is a
    pure function of the index -- identical on every device and process,
    whatever the chunking."""
    z = x * _GOLD + _GOLD
    z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * _MIX1
    z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * _MIX2
    return z ^ ((z >> 31) & ((1 << 33) - 1))


def _uniform(seed, stream, start, m, dev):
    """m uniform doubles in [0, 1): draws start .. start+m-1 of `stream`."""
    k = torch.arange(start, start + m, device=dev, dtype=torch.int64)
    z = _splitmix64(_splitmix64(k * 4 + stream) ^ int(seed))
    return ((z >> 11) & ((1 << 53) - 1)).to(torch.float64) * (2.0 ** -53)


def _all_gather_np(w, arr):
    return [np.asarray(x) for x in w.all_gather_object(arr)]


def chung_lu_sharded(n, pairs, p, alpha=0.6, max_weight=None, seed=0, world=None,
                     log=None) -> ShardedGraph:
    """Power-law (Chung-Lu) symmetric graph with ~`pairs` undirected edges,
    GCN-normalised (sparse.py:184-205) and split into p block rows; each
    process materialises only its hosted rows (on its GPU).

    Same model as graphgen.chung_lu_device (expected degree of the vertex of
    rank k ~ (k+1)^-alpha, capped, seeded relabel), drawn in fixed-size
    chunks so every process consumes the identical random stream and keeps
    the pairs touching its rows.  Draw rounds continue until the global
    number of distinct pairs reaches `pairs` (it ends within a fraction of
    a percent above; the exact nnz is reported)."""
    from .dist import world as _world
    w = world or _world().init()
    dev = _dev()
    say = log or (lambda *a: None)
    n, pairs = int(n), int(pairs)
    bounds, starts = block_bounds(n, p)
    hosted = w.local_ranks(p) if w.multi else list(range(p))
    R0, R1 = bounds[hosted[0]][0], bounds[hosted[-1]][1]
    # degree weights and their CDF on the host: a sequential (numpy) sum is
    # bit-identical in every process, a parallel GPU scan is not (its
    # association order depends on timing), and a draw landing on a CDF
    # boundary would then pick different vertices in different processes
    wt = (np.arange(n, dtype=np.float64) + 1.0) ** (-alpha)
    wt = wt / wt.sum() * (2.0 * pairs)
    if max_weight is not None:
        for _ in range(8):
            wt = np.minimum(wt, float(max_weight))
            wt = wt / wt.sum() * (2.0 * pairs)
    # seeded relabel (hubs scattered): a permutation from sorting hashed ids
    perm = torch.argsort(_splitmix64(torch.arange(n, device=dev) * 4 + 3) ^ int(seed))
    wt = wt[perm.cpu().numpy()]
    del perm
    cdf = np.cumsum(wt)
    cdf = torch.from_numpy(cdf / cdf[-1]).to(dev)
    del wt
    keys = torch.zeros(0, dtype=torch.int64, device=dev)
    draw = pairs                   # duplicates / self-pairs are topped up below
    total = 0
    drawn = 0                      # draws consumed so far (counter of the generator)
    while True:
        kept = [keys]
        todo = draw
        while todo > 0:
            m = min(_CHUNK, todo)
            todo -= m
            u = torch.searchsorted(cdf, _uniform(seed, 0, drawn, m, dev))
            v = torch.searchsorted(cdf, _uniform(seed, 1, drawn, m, dev))
            drawn += m
            u.clamp_(max=n - 1)
            v.clamp_(max=n - 1)
            lo, hi = torch.minimum(u, v), torch.maximum(u, v)
            del u, v
            sel = (lo != hi) & (((lo >= R0) & (lo < R1)) | ((hi >= R0) & (hi < R1)))
            kept.append(lo[sel] * n + hi[sel])
            del lo, hi, sel
        keys = torch.unique(torch.cat(kept))
        del kept
        owned = int(((keys >= R0 * n) & (keys < R1 * n)).sum())
        total = sum(w.all_gather_object(owned))
        if w.multi:
            _check_cross_pairs(w, keys, n, p, bounds)
        say(f"[sharded] distinct pairs {total:,} of {pairs:,}")
        if total >= pairs:
            break
        draw = int((pairs - total) * 1.05) + 1024
    del cdf
    # ---- block rows: entries (lo, hi) for lo in the block, (hi, lo) for hi
    blocks, deg_local = {}, {}
    for i in hosted:
        r0, r1 = bounds[i]
        a0 = int(torch.searchsorted(keys, torch.tensor(r0 * n, device=dev)))
        a1 = int(torch.searchsorted(keys, torch.tensor(r1 * n, device=dev)))
        rows_a = keys[a0:a1] // n
        cols_a = keys[a0:a1] % n
        parts_r, parts_c = [rows_a, torch.arange(r0, r1, device=dev)], \
            [cols_a, torch.arange(r0, r1, device=dev)]
        for c0 in range(0, keys.numel(), _CHUNK):
            kc = keys[c0:c0 + _CHUNK]
            hi = kc % n
            sel = (hi >= r0) & (hi < r1)
            parts_r.append(hi[sel])
            parts_c.append(kc[sel] // n)
            del hi, sel, kc
        rows = torch.cat(parts_r)
        cols = torch.cat(parts_c)
        del parts_r, parts_c, rows_a, cols_a
        key2, _ = torch.sort((rows - r0) * n + cols)
        del rows, cols
        rl = key2 // n
        col = (key2 % n).to(torch.int32)
        del key2
        cnt = torch.bincount(rl, minlength=r1 - r0)
        del rl
        rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        rp[1:] = torch.cumsum(cnt, 0).cpu().numpy()
        deg_local[i] = cnt.to(torch.int32)            # unit weights + self-loop
        blocks[i] = [rp, col, None]
        say(f"[sharded] block {i}: rows {r1 - r0:,} nnz {col.numel():,}")
    del keys
    # ---- global degrees (each process knows its rows'), then normalise
    mine = torch.cat([deg_local[i] for i in hosted]).cpu().numpy()
    deg = torch.from_numpy(np.concatenate(_all_gather_np(w, mine))).to(dev)
    dinv = deg.to(torch.float64) ** -0.5
    del deg
    nnz_local = 0
    for i in hosted:
        rp, col, _ = blocks[i]
        r0, r1 = bounds[i]
        lens = torch.from_numpy(np.diff(rp)).to(dev)
        rowg = torch.repeat_interleave(torch.arange(r0, r1, device=dev), lens)
        val = (dinv[rowg] * dinv[col.long()]).to(torch.float32)   # sparse.py:204
        del rowg, lens
        blocks[i][2] = val
        blocks[i] = tuple(blocks[i])
        nnz_local += col.numel()
    del dinv, deg_local
    nnz_total = sum(w.all_gather_object(nnz_local))
    torch.cuda.empty_cache()
    return ShardedGraph(n, p, blocks, nnz_total, w)


def _check_cross_pairs(w, keys, n, p, bounds):
    """Every pair joining two processes' rows is held by both: the number of
    (lo in A, hi in B) pairs each process holds must agree (a cheap guard
    against the processes drawing different graphs)."""
    size = w.size
    edges = torch.tensor([bounds[r][0] for r in range(p) if w.proc_of(r, p) != w.proc_of(r - 1, p)
                          or r == 0] + [n], device=keys.device, dtype=torch.int64)
    cnt = torch.zeros(size * size, dtype=torch.int64, device=keys.device)
    hsum = torch.zeros(size * size, dtype=torch.int64, device=keys.device)
    for c0 in range(0, keys.numel(), _CHUNK):
        kc = keys[c0:c0 + _CHUNK]
        a = torch.searchsorted(edges, kc // n, right=True) - 1
        b = torch.searchsorted(edges, kc % n, right=True) - 1
        ab = a * size + b
        cnt += torch.bincount(ab, minlength=size * size)
        # order-independent checksum of the pair set (wrapping int64 sum of hashes)
        hsum.index_add_(0, ab, _splitmix64(kc))
    mine = (cnt.cpu().numpy().reshape(size, size), hsum.cpu().numpy().reshape(size, size))
    allc = w.all_gather_object(mine)
    me = w.proc
    for q in range(size):
        if q == me:
            continue
        a, b = min(me, q), max(me, q)
        if allc[me][0][a, b] != allc[q][0][a, b] or allc[me][1][a, b] != allc[q][1][a, b]:
            raise RuntimeError(f"processes {me} and {q} drew different graphs "
                               f"({allc[me][0][a, b]} vs {allc[q][0][a, b]} shared pairs)")


def papers_shaped_sharded(p, seed=0, n=111_059_956, nnz=3_231_371_744, world=None, log=None):
    """Config 5: ogbn-papers100M-shaped power-law graph (111,059,956
    vertices, ~3.23B stored off-diagonal nonzeros + self-loops,
    PAPER.md:550), sharded into p block rows."""
    return chung_lu_sharded(n, nnz // 2, p, alpha=0.7, max_weight=30_000, seed=seed,
                            world=world, log=log)


class _Count:
    """Stands in for an NnzCols list where only its length is needed (the
    ledger's index charges, plan.index_setup_charges)."""

    __slots__ = ("size",)

    def __init__(self, size):
        self.size = int(size)


class ShardedOperand:
    """`plan.DistOperand` counterpart over a ShardedGraph (symmetric Â, so
    the forward and backward operands alias, spmm.py:116)."""

    parities = 1            # single halo buffer per rank (halos fill HBM at this scale)

    def __init__(self, graph: ShardedGraph):
        self.graph = graph
        self.boundaries = list(graph.boundaries)
        self.widths = [e - s for s, e in self.boundaries]
        self.starts = graph.starts
        self._device = {}
        w, p = graph.world, graph.p
        dev = _dev()
        self._starts_dev = torch.from_numpy(self.starts).to(dev)
        self._starts32 = torch.from_numpy(self.starts.astype(np.int32)).to(dev)
        self._split = {}      # hosted i -> occupancy prefix at each block start
        self._send = {}       # hosted s -> {d: sorted int32 local rows of s needed by d}
        recv = np.zeros((p, p), dtype=np.int64)
        send = np.zeros((p, p), dtype=np.int64)
        for i, blk in graph.blocks.items():
            _, col, _ = blk
            occ = torch.zeros(graph.n, dtype=torch.bool, device=dev)
            occ[col.long()] = True
            cs = torch.cumsum(occ, 0)
            del occ
            split = torch.zeros(p + 1, dtype=torch.int64, device=dev)
            split[1:] = cs[self._starts_dev[1:] - 1]
            del cs
            self._split[i] = split
            sp = split.cpu().numpy()
            recv[i] = np.diff(sp)
            recv[i, i] = 0
            self._send[i] = self._send_lists(i)
            for d, idx in self._send[i].items():
                send[i, d] = idx.numel()
        recv = np.sum(_all_gather_np(w, recv), axis=0)
        send = np.sum(_all_gather_np(w, send), axis=0)
        # receiver d's NnzCols(d, s) and sender s's list must have the same size
        if not np.array_equal(recv, send.T):
            raise ValueError("sharded operand is not structurally symmetric: "
                             "sender and receiver row lists disagree")
        self.counts = recv                       # counts[i, q] = |NnzCols(i, q)|
        self.nnz_cols = {(i, q): _Count(recv[i, q]) for i in range(p) for q in range(p)}

    @property
    def n_blocks(self):
        return len(self.boundaries)

    def _send_lists(self, s):
        rp, col, _ = self.graph.blocks[s]
        p = self.graph.p
        n_s = len(rp) - 1
        dev = col.device
        lens = torch.from_numpy(np.diff(rp)).to(dev)
        rows = torch.repeat_interleave(torch.arange(n_s, device=dev), lens)
        owner = torch.searchsorted(self._starts32[1:], col, right=True, out_int32=True)
        flag = torch.zeros(n_s * p, dtype=torch.bool, device=dev)
        flag[rows * p + owner] = True
        del rows, owner, lens
        flag = flag.view(n_s, p)
        out = {}
        for d in range(p):
            if d != s:
                out[d] = torch.nonzero(flag[:, d]).flatten().to(torch.int32)
        return out

    def _ext(self, i, aware, halo_off):
        rp, col, _ = self.graph.blocks[i]
        r0 = self.boundaries[i][0]
        n_i = self.widths[i]
        dev = col.device
        st = self._starts_dev
        owner = torch.searchsorted(self._starts32[1:], col, right=True).long()
        base = torch.zeros(self.n_blocks, dtype=torch.int64, device=dev)
        for q, o in halo_off.items():
            base[q] = n_i + o
        c64 = col.long()
        if aware:
            occ = torch.zeros(self.graph.n, dtype=torch.bool, device=dev)
            occ[c64] = True
            rank_in_u = torch.cumsum(occ, 0) - 1
            del occ
            ext = base[owner] + rank_in_u[c64] - self._split[i][owner]
            del rank_in_u
        else:
            ext = base[owner] + c64 - st[owner]
        ext = torch.where(owner == i, c64 - r0, ext).to(torch.int32)
        return ext

    def build_variant_plan(self, grid: ProcessGrid, variant: str, local_ranks=None):
        """plan.build_variant_plan for the 1D variants (spmm.py:172-191)."""
        validate_variant_grid(variant, grid.p, grid.c)
        if not variant.startswith("1d") or grid.p != self.graph.p:
            raise ValueError("sharded operands support the 1D variants on their own p")
        hosted = set(self.graph.blocks) if local_ranks is None else set(local_ranks)
        aware = variant.endswith("sparse")
        p, widths = grid.p, self.widths
        ranks = []
        for r in range(p):
            halo_off, off = {}, 0
            for q in range(p):
                if q == r:
                    continue
                halo_off[q] = off
                off += int(self.counts[r, q]) if aware else widths[q]
            if r not in hosted or self.graph.blocks.get(r) is None:
                ranks.append(RankOperand(r, r, 0, widths[r], widths[r], None, None, None, off,
                                         halo_off))
                continue
            rp, _, val = self.graph.blocks[r]
            ranks.append(RankOperand(r, r, 0, widths[r], widths[r], rp,
                                     self._ext(r, aware, halo_off), val, off, halo_off))
        segments = []
        for s in range(p):
            for d in range(p):
                if d == s:
                    continue
                if aware:
                    cnt = int(self.counts[d, s])
                    idx = self._send[s][d] if s in self._send else None
                    if idx is None:
                        idx = _Count(cnt)          # not hosted here: count only
                else:
                    idx, cnt = None, widths[s]
                segments.append(Segment(s, d, s, idx, cnt, ranks[d].halo_off[s]))
        return VariantPlan(grid, variant, ranks, segments, widths, self.nnz_cols)

    def release_device(self):
        for dp in self._device.values():
            dp.close()
        self._device.clear()


class ShardedDistMatrices:
    """`plan.DistMatrices` over a ShardedOperand (fwd and bwd alias)."""

    def __init__(self, op: ShardedOperand, grid: ProcessGrid):
        self.grid = grid
        self.boundaries = op.boundaries
        self.fwd = self.bwd = op
        self.n = op.graph.n

    @property
    def symmetric(self):
        return True

    def release_device(self):
        self.fwd.release_device()


def _sharded_run_class():
    from .gcn import GcnRun

    class ShardedGcnRun(GcnRun):
        """`gcn.GcnRun` over a ShardedGraph: the same epoch loop
        (gcn.py:258-286); the features, labels and mask exist only as the
        hosted block rows, generated on the device (x[i], labels[i], mask[i])."""

        def __init__(self, graph: ShardedGraph, x: dict, labels: dict, f_in: int, f_out: int,
                     cfg, denom: int = None):
            from .dist import world
            from .engine import pad4
            from .gcn import _dev, init_weights
            from .partition import block_partition
            from .spmm import device_plan
            validate_variant_grid(cfg.variant, graph.p, 1)
            world().init()
            self.cfg = cfg
            self.grid = grid = ProcessGrid(graph.p, 1)
            self.part = None
            self.device = dev = _dev()
            self.graph = graph
            op = ShardedOperand(graph)
            self.dm = ShardedDistMatrices(op, grid)
            self.f_in = int(f_in)
            self.x = x
            self.f_out = int(f_out)
            self.denom = int(graph.n if denom is None else denom)
            self.dims = cfg.layer_dims(self.f_in, self.f_out)
            self.lds = [pad4(d) for d in self.dims]
            self.w0 = []
            for l, w in enumerate(init_weights(cfg, self.f_in, self.f_out)):
                wp = torch.zeros((self.lds[l], self.lds[l + 1]), dtype=torch.float32,
                                 device=dev)
                wp[:w.shape[0], :w.shape[1]] = torch.from_numpy(w.astype(np.float32))
                self.w0.append(wp)
            self.labels = labels
            self.mask = {i: torch.ones(t.numel(), dtype=torch.uint8, device=dev)
                         for i, t in labels.items()}
            self.xent, self.dense, self.ctx, self.timer = {}, {}, {}, None
            device_plan(op, grid, cfg.variant, max_ld=max(self.lds))
            graph.release()                      # the plans hold the entries now
            torch.cuda.empty_cache()
            self.part = block_partition(graph.n, graph.p)

        def _inputs(self, i):
            return self.x[i], self.labels[i], self.mask[i]

    return ShardedGcnRun


def sharded_gcn_run(graph, x, labels, f_in, f_out, cfg, denom=None):
    """Build a GcnRun over a ShardedGraph (see ShardedGcnRun)."""
    return _sharded_run_class()(graph, x, labels, f_in, f_out, cfg, denom)


def sharded_inputs(graph: ShardedGraph, f_in: int, classes: int, seed=1):
    """Synthetic inputs for the hosted block rows, generated on the device:
    features N(0, 1) (padded to the row pitch), labels uniform in
    [0, classes); seeded per block so they do not depend on the process
    count."""
    from .engine import pad4
    dev = _dev()
    ld = pad4(f_in)
    x, y = {}, {}
    for i in graph.blocks:
        r0, r1 = graph.boundaries[i]
        g = torch.Generator(device=dev)
        g.manual_seed(int(seed) * 1_000_003 + i)
        t = torch.zeros((r1 - r0, ld), dtype=torch.float32, device=dev)
        t[:, :f_in] = torch.randn((r1 - r0, f_in), generator=g, device=dev)
        x[i] = t
        y[i] = torch.randint(0, classes, (r1 - r0,), generator=g, device=dev)
    return x, y
