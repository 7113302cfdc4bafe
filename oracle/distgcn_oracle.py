"""CPU oracle for the distributed-SpMM / full-graph-GCN hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in `paper_2504_04673_b200/` imports,
calls or links this module; only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may use it, and there
only as the checker (or as the timed stand-in for the reference's own CPU
path), never as the thing measured or shipped.

What it is: a plain NumPy restatement of the reference package `distgcn`
0.1.0 (pure Python/NumPy, /root/reference/pkg/src/distgcn) for exactly the
functions on the hot path.  Every function cites the reference file:line it
follows.  Sequential (no threads): the reference's bulk-synchronous runtime
is schedule-independent (runtime.py:1-20), so replaying every rank in
ascending order with the same accounting rules gives the same results and
the same ledger.

Pinning: the restatement is checked against golden vectors produced by
importing the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`, checked by
`tests/test_oracle_golden.py`).  Parity is therefore pinned, not assumed.

Arithmetic is float64 throughout, like the reference (sparse.py:46-48).
"""

from __future__ import annotations

import numpy as np

PRIMITIVES = ("p2p", "alltoallv", "broadcast", "allreduce")
_SENT = ("bytes_sent", "data_bytes_sent", "index_bytes_sent",
         "msgs_sent", "data_msgs_sent", "index_msgs_sent")
_RECV = ("bytes_received", "data_bytes_received", "index_bytes_received",
         "msgs_received", "data_msgs_received", "index_msgs_received")
VARIANTS = ("1d-oblivious", "1d-sparse", "15d-oblivious", "15d-sparse")


# --------------------------------------------------------------------------
# CSR helpers (sparse.py)
# --------------------------------------------------------------------------

class Csr:
    """Canonical CSR, int64 indices / float64 values (sparse.py:30-48)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.col_idx.size)

    def row_of_nnz(self):
        # sparse.py:74-76
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_ptr))

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        out[self.row_of_nnz(), self.col_idx] = self.values
        return out


def csr_from_coo(n_rows, n_cols, rows, cols, vals, drop_zeros=True):
    """sparse.py:110-137: lexsort by (row, col, val), sum duplicates with
    add.reduceat, drop exact zeros."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size:
        o = np.lexsort((vals, cols, rows))
        rows, cols, vals = rows[o], cols[o], vals[o]
        first = np.ones(rows.size, dtype=bool)
        first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        st = np.flatnonzero(first)
        vals = np.add.reduceat(vals, st)
        rows, cols = rows[st], cols[st]
        if drop_zeros:
            k = vals != 0.0
            rows, cols, vals = rows[k], cols[k], vals[k]
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    if rows.size:
        np.cumsum(np.bincount(rows, minlength=n_rows), out=rp[1:])
    return Csr(n_rows, n_cols, rp, cols, vals)


def csr_from_dense(d):
    """sparse.py:168-173."""
    d = np.asarray(d, dtype=np.float64)
    r, c = np.nonzero(d)
    return csr_from_coo(d.shape[0], d.shape[1], r, c, d[r, c])


def transpose_csr(a: Csr) -> Csr:
    """sparse.py:237-247: stable argsort of columns (a pure permutation)."""
    order = np.argsort(a.col_idx, kind="stable")
    rp = np.zeros(a.n_cols + 1, dtype=np.int64)
    if a.nnz:
        np.cumsum(np.bincount(a.col_idx, minlength=a.n_cols), out=rp[1:])
    return Csr(a.n_cols, a.n_rows, rp, a.row_of_nnz()[order], a.values[order])


def csr_equal(a: Csr, b: Csr) -> bool:
    """sparse.py:176-181."""
    return ((a.n_rows, a.n_cols) == (b.n_rows, b.n_cols)
            and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(a.values, b.values))


def gcn_normalize(a: Csr) -> Csr:
    """sparse.py:184-205: D^-1/2 (A + I) D^-1/2 with the two scale factors
    grouped (dinv[r] * dinv[c]) before multiplying the value."""
    n = a.n_rows
    diag = np.arange(n, dtype=np.int64)
    wl = csr_from_coo(n, n, np.concatenate([a.row_of_nnz(), diag]),
                      np.concatenate([a.col_idx, diag]),
                      np.concatenate([a.values, np.ones(n)]))
    deg = np.bincount(wl.row_of_nnz(), weights=wl.values, minlength=n)
    dinv = deg ** -0.5
    vals = wl.values * (dinv[wl.row_of_nnz()] * dinv[wl.col_idx])
    return Csr(n, n, wl.row_ptr, wl.col_idx, vals)


def local_spmm(a: Csr, h) -> np.ndarray:
    """sparse.py:208-223: out = A @ h accumulated in storage order with
    np.add.at over an nnz x f temporary (the reference's hot loop)."""
    h = np.asarray(h, dtype=np.float64)
    out = np.zeros((a.n_rows, h.shape[1]))
    if a.nnz:
        np.add.at(out, a.row_of_nnz(), a.values[:, None] * h[a.col_idx])
    return out


def local_spmm_fast(a: Csr, h) -> np.ndarray:
    """The same product as `local_spmm` in float64 through scipy.sparse
    (checker acceleration for large or long runs: the summation order
    differs from np.add.at's by rounding at 1e-16, five orders below the
    fp32 contract).  Used only by tests at BASELINE sizes."""
    import scipy.sparse as sp
    h = np.asarray(h, dtype=np.float64)
    m = sp.csr_matrix((np.asarray(a.values, np.float64), np.asarray(a.col_idx, np.int64),
                       np.asarray(a.row_ptr, np.int64)), shape=(a.n_rows, a.n_cols))
    return np.asarray(m @ h)


def serial_reference(a: Csr, h) -> np.ndarray:
    """spmm.py:249-252."""
    return local_spmm(transpose_csr(a), h)


# --------------------------------------------------------------------------
# partition layout (partition.py)
# --------------------------------------------------------------------------

def block_boundaries(n, k):
    """partition.py:154-161: first n mod k parts take one extra vertex."""
    base, rem = divmod(n, k)
    sizes = [base + 1] * rem + [base] * (k - rem)
    b, pos = [], 0
    for s in sizes:
        b.append((pos, pos + s))
        pos += s
    return b


def perm_from_assignment(assignment, k):
    """partition.py:55-65: stable sort by part -> perm (old id -> new id)
    and the variable boundaries."""
    assignment = np.asarray(assignment, dtype=np.int64)
    order = np.argsort(assignment, kind="stable")
    perm = np.empty(assignment.size, dtype=np.int64)
    perm[order] = np.arange(assignment.size)
    sizes = np.bincount(assignment, minlength=k)
    b, pos = [], 0
    for s in sizes:
        b.append((pos, pos + int(s)))
        pos += int(s)
    return perm, b


def apply_partition(a: Csr, h, perm):
    """partition.py:231-254: P A P^T via lexsort of (new col, new row) and
    h[inv_perm]."""
    nr = perm[a.row_of_nnz()]
    nc = perm[a.col_idx]
    order = np.lexsort((nc, nr))
    rp = np.zeros(a.n_rows + 1, dtype=np.int64)
    if a.nnz:
        np.cumsum(np.bincount(nr, minlength=a.n_rows), out=rp[1:])
    a2 = Csr(a.n_rows, a.n_cols, rp, nc[order], a.values[order])
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    h2 = None if h is None else np.asarray(h, dtype=np.float64)[inv]
    return a2, h2, inv


def comm_send_rows(a: Csr, assignment, k):
    """partition.py:201-228 (vectorised): per-part send rows and pair rows.
    pair_rows[foreign, own] counts vertices of part `own` with at least one
    out-neighbour in part `foreign`."""
    assignment = np.asarray(assignment, dtype=np.int64)
    rows = a.row_of_nnz()
    key = np.unique(rows * k + assignment[a.col_idx])
    v, t = key // k, key % k
    own = assignment[v]
    f = t != own
    pair = np.zeros((k, k), dtype=np.int64)
    np.add.at(pair, (t[f], own[f]), 1)
    send = pair.sum(axis=0)
    return send, pair


# --------------------------------------------------------------------------
# block layout (spmm.py:80-117)
# --------------------------------------------------------------------------

def extract_operand(mat: Csr, boundaries):
    """spmm.py:80-105: blocks[i][j] with block-local columns and
    nnz_cols[(i, j)] = np.unique(sub_cols)."""
    nb = len(boundaries)
    widths = [e - s for s, e in boundaries]
    starts = np.array([s for s, _ in boundaries] + [mat.n_cols], dtype=np.int64)
    row_all = mat.row_of_nnz()
    blocks, cache = [], {}
    for i, (r0, r1) in enumerate(boundaries):
        lo, hi = mat.row_ptr[r0], mat.row_ptr[r1]
        rows = row_all[lo:hi] - r0
        cols = mat.col_idx[lo:hi]
        vals = mat.values[lo:hi]
        owner = np.searchsorted(starts, cols, side="right") - 1
        rb = []
        for j in range(nb):
            sel = owner == j
            sr, sc = rows[sel], cols[sel] - starts[j]
            rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
            if sr.size:
                np.cumsum(np.bincount(sr, minlength=r1 - r0), out=rp[1:])
            rb.append(Csr(r1 - r0, widths[j], rp, sc, vals[sel]))
            cache[(i, j)] = np.unique(sc)
        blocks.append(rb)
    return {"blocks": blocks, "nnz_cols": cache, "widths": widths}


def build_dist_matrices(a: Csr, boundaries):
    """spmm.py:108-117: fwd = blocks of A^T, bwd aliases fwd if symmetric."""
    at = transpose_csr(a)
    fwd = extract_operand(at, boundaries)
    bwd = fwd if csr_equal(at, a) else extract_operand(a, boundaries)
    return fwd, bwd


# --------------------------------------------------------------------------
# ledger (runtime.py:112-219) -- same counters and charging conventions
# --------------------------------------------------------------------------

class Ledger:
    def __init__(self, p):
        self.p = p
        self.counters = {}
        for prim in PRIMITIVES:
            d = {n: np.zeros(p, np.int64 if n.startswith("msgs") else np.float64)
                 for n in _SENT + _RECV}
            d["calls"] = np.zeros(p, np.int64)
            self.counters[prim] = d
        self.pair_max_bytes = {}
        self.pair_max_data_bytes = {}
        self.marks = {}

    def send(self, prim, r, nbytes, kind, msgs=1):           # runtime.py:139-144
        c = self.counters[prim]
        c["bytes_sent"][r] += nbytes
        c[kind + "_bytes_sent"][r] += nbytes
        c["msgs_sent"][r] += msgs
        c[kind + "_msgs_sent"][r] += msgs

    def recv(self, prim, r, nbytes, kind, msgs=1):           # runtime.py:146-151
        c = self.counters[prim]
        c["bytes_received"][r] += nbytes
        c[kind + "_bytes_received"][r] += nbytes
        c["msgs_received"][r] += msgs
        c[kind + "_msgs_received"][r] += msgs

    def pair(self, s, d, nbytes, kind):                       # runtime.py:153-158
        k = (s, d)
        if nbytes > self.pair_max_bytes.get(k, 0):
            self.pair_max_bytes[k] = nbytes
        if kind == "data" and nbytes > self.pair_max_data_bytes.get(k, 0):
            self.pair_max_data_bytes[k] = nbytes

    def p2p(self, s, d, elems, kind):
        """Comm.isend + matching recv (runtime.py:311-344)."""
        if s == d:
            return
        nb = 8 * elems
        self.send("p2p", s, nb, kind)
        self.pair(s, d, nb, kind)
        self.recv("p2p", d, nb, kind)

    def alltoallv(self, elems):
        """Comm.all_to_allv (runtime.py:379-406); elems[s][d] element counts."""
        p = self.p
        for r in range(p):
            self.counters["alltoallv"]["calls"][r] += 1
        for s in range(p):
            for d in range(p):
                e = elems[s][d]
                if s == d or e == 0:
                    continue
                self.send("alltoallv", s, 8 * e, "data")
                self.recv("alltoallv", d, 8 * e, "data")
                self.pair(s, d, 8 * e, "data")

    def broadcast(self, root, elems):
        """Comm.broadcast (runtime.py:408-435): linear at the root."""
        p = self.p
        nb = 8 * elems
        for r in range(p):
            self.counters["broadcast"]["calls"][r] += 1
            if r != root:
                self.recv("broadcast", r, nb, "data")
                self.pair(root, r, nb, "data")
        if p > 1:
            self.send("broadcast", root, nb * (p - 1), "data", msgs=p - 1)

    def allreduce(self, group, elems):
        """Comm.all_reduce_sum (runtime.py:437-466): ring 2(g-1)/g."""
        g = len(group)
        nb = 8 * elems
        wire = 2.0 * (g - 1) / g * nb if g > 1 else 0.0
        for r in group:
            self.counters["allreduce"]["calls"][r] += 1
            if g > 1:
                self.send("allreduce", r, wire, "data", msgs=2 * (g - 1))
                self.recv("allreduce", r, wire, "data", msgs=2 * (g - 1))

    def snapshot(self):                                       # runtime.py:193-203
        return {prim: {"bytes_sent": float(c["bytes_sent"].sum()),
                       "data_bytes_sent": float(c["data_bytes_sent"].sum()),
                       "index_bytes_sent": float(c["index_bytes_sent"].sum()),
                       "msgs_sent": int(c["msgs_sent"].sum())}
                for prim, c in self.counters.items()}


# --------------------------------------------------------------------------
# the four variants (spmm.py:133-246), replayed rank by rank
# --------------------------------------------------------------------------

def grid_coords(rank, c):
    return divmod(rank, c)                                    # runtime.py:85-89


def exchange_index_lists(led: Ledger, op, p, c, variant):
    """spmm.py:133-163: one-time index announcements (int64 payloads)."""
    if variant.endswith("oblivious"):
        return
    nnzc = op["nnz_cols"]
    if variant == "1d-sparse":
        for r in range(p):
            for dst in range(p):
                if dst != r and nnzc[(r, dst)].size:
                    led.p2p(r, dst, nnzc[(r, dst)].size, "index")
        return
    s = p // (c * c)
    for r in range(p):
        i, j = grid_coords(r, c)
        for k in range(s):
            q = j * s + k
            if q != i and nnzc[(i, q)].size:
                led.p2p(r, q * c + j, nnzc[(i, q)].size, "index")


def _scatter(idx, payload, width, f):                         # spmm.py:166-169
    buf = np.zeros((width, f))
    buf[idx] = payload
    return buf


def spmm_all_ranks(led: Ledger, op, hblocks, p, c, variant):
    """spmm.py:172-227 for every rank; hblocks[i] is block row i of H.
    Returns per-rank results z[rank]."""
    blocks, nnzc, widths = op["blocks"], op["nnz_cols"], op["widths"]
    f = hblocks[0].shape[1]
    out = [None] * p
    if variant == "1d-oblivious":                             # spmm.py:172-179
        z = [np.zeros((blocks[r][r].n_rows, f)) for r in range(p)]
        for j in range(p):
            led.broadcast(j, hblocks[j].size)
            for r in range(p):
                z[r] += local_spmm(blocks[r][j], hblocks[j])
        return z
    if variant == "1d-sparse":                                # spmm.py:182-191
        elems = [[hblocks[s][nnzc[(d, s)]].size for d in range(p)] for s in range(p)]
        led.alltoallv(elems)
        for r in range(p):
            z = np.zeros((blocks[r][r].n_rows, f))
            for j in range(p):
                hj = _scatter(nnzc[(r, j)], hblocks[j][nnzc[(r, j)]], widths[j], f)
                z += local_spmm(blocks[r][j], hj)
            out[r] = z
        return out
    sparse = variant == "15d-sparse"                          # spmm.py:194-227
    s = p // (c * c)
    nrows = p // c
    partial = [None] * p
    for r in range(p):
        i, j = grid_coords(r, c)
        z = np.zeros((blocks[i][i].n_rows, f))
        for k in range(s):
            q = j * s + k
            if q == i:
                for l in range(nrows):
                    if l == i:
                        continue
                    if sparse:
                        idx = nnzc[(l, q)]
                        if idx.size == 0:
                            continue
                        led.p2p(r, l * c + j, hblocks[q][idx].size, "data")
                    else:
                        led.p2p(r, l * c + j, hblocks[q].size, "data")
                hq = (_scatter(nnzc[(i, q)], hblocks[q][nnzc[(i, q)]], widths[q], f)
                      if sparse else hblocks[q])
            elif sparse:
                idx = nnzc[(i, q)]
                hq = (_scatter(idx, hblocks[q][idx], widths[q], f) if idx.size
                      else np.zeros((widths[q], f)))
            else:
                hq = hblocks[q]
            z += local_spmm(blocks[i][q], hq)
        partial[r] = z
    for i in range(nrows):                                    # runtime.py:437-466
        group = [i * c + jj for jj in range(c)]
        total = partial[group[0]].copy()
        for r in group[1:]:
            total = total + partial[r]
        led.allreduce(group, total.size)
        for r in group:
            out[r] = total.copy()
    return out


def run_spmm(a: Csr, h, p, c, variant, assignment=None, index_setup=True):
    """spmm.py:264-294: permute, distribute, run, gather in original order.
    `assignment` (vertex -> part) defaults to the block partition."""
    h = np.asarray(h, dtype=np.float64)
    nrows = p // c
    if assignment is None:
        bounds = block_boundaries(a.n_rows, nrows)
        assignment = np.repeat(np.arange(nrows), [e - s for s, e in bounds])
    perm, bounds = perm_from_assignment(assignment, nrows)
    a2, h2, _ = apply_partition(a, h, perm)
    fwd, _ = build_dist_matrices(a2, bounds)
    led = Ledger(p)
    if index_setup:
        exchange_index_lists(led, fwd, p, c, variant)
    hb = [h2[s:e] for s, e in bounds]
    z = spmm_all_ranks(led, fwd, hb, p, c, variant)
    z2 = np.vstack([z[i * c] for i in range(nrows)])
    return z2[perm], led, fwd, bounds, perm


# --------------------------------------------------------------------------
# GCN (gcn.py)
# --------------------------------------------------------------------------

def layer_dims(layers, hidden, f_in, f_out):
    return [f_in] + [hidden] * (layers - 2) + [f_out]          # gcn.py:72-73


def init_weights(seed, layers, hidden, f_in, f_out):
    """gcn.py:85-95: uniform(-sqrt(6/(fi+fo)), +) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    dims = layer_dims(layers, hidden, f_in, f_out)
    return [rng.uniform(-np.sqrt(6.0 / (fi + fo)), np.sqrt(6.0 / (fi + fo)), size=(fi, fo))
            for fi, fo in zip(dims[:-1], dims[1:])]


def xent_parts(logits, labels, mask, denom):
    """gcn.py:98-120: (loss sum, grad / denom, correct argmax count)."""
    shift = logits - logits.max(axis=1, keepdims=True)
    log_norm = np.log(np.exp(shift).sum(axis=1))
    grad = np.zeros_like(logits)
    loss_sum, correct = 0.0, 0
    if mask.any():
        rows = np.flatnonzero(mask)
        sel = labels[rows]
        loss_sum = float((log_norm[rows] - shift[rows, sel]).sum())
        sm = np.exp(shift[rows]) / np.exp(shift[rows]).sum(axis=1, keepdims=True)
        sm[np.arange(rows.size), sel] -= 1.0
        grad[rows] = sm / denom
        correct = int((logits[rows].argmax(axis=1) == sel).sum())
    return loss_sum, grad, correct


def serial_train(a_hat: Csr, features, labels, mask, layers, hidden, lr, epochs, seed,
                 f_out=None, weights=None, spmm=None):
    """gcn.py:135-172 + 211-227: full-batch GD on the undistributed matrix.
    Returns (history [(loss, acc)], final weights).  `spmm` (default
    `local_spmm`) may be `local_spmm_fast` for long checker runs."""
    local_spmm_ = local_spmm if spmm is None else spmm
    features = np.asarray(features, dtype=np.float64)
    labels = np.asarray(labels, dtype=np.int64)
    mask = np.asarray(mask, dtype=bool)
    f_out = f_out if f_out is not None else int(labels.max()) + 1
    ws = ([np.array(w, dtype=np.float64) for w in weights] if weights is not None
          else init_weights(seed, layers, hidden, features.shape[1], f_out))
    at = transpose_csr(a_hat)
    fwd = a_hat if csr_equal(at, a_hat) else at
    denom = int(mask.sum())
    hist = []
    last = len(ws) - 1
    for _ in range(epochs):
        hs, zs = [features], []
        for l, w in enumerate(ws):
            z = local_spmm_(fwd, hs[-1]) @ w
            zs.append(z)
            hs.append(np.maximum(z, 0.0) if l < last else z)
        loss_sum, g, correct = xent_parts(hs[-1], labels, mask, denom)
        ys = [None] * len(ws)
        for l in range(last, -1, -1):
            m = local_spmm_(a_hat, g)
            ys[l] = hs[l].T @ m
            if l > 0:
                g = (m @ ws[l].T) * (zs[l - 1] > 0.0)
        for w, y in zip(ws, ys):
            w -= lr * y
        hist.append((loss_sum / denom, correct / denom))
    return hist, ws


def train_ledger(fwd, bwd, p, c, variant, epochs, dims):
    """Ledger of gcn.py:258-286 for `epochs` epochs: index setup, then per
    epoch 2(L-1) multiply phases and L-1 col-group weight all-reduces, with
    a mark after every epoch.  Data volumes depend only on the plan."""
    led = Ledger(p)
    exchange_index_lists(led, fwd, p, c, variant)
    if bwd is not fwd:
        exchange_index_lists(led, bwd, p, c, variant)
    nw = len(dims) - 1
    n_blocks = p // c
    widths = fwd["widths"]

    def phase(op, f):
        hb = [np.zeros((widths[i], f)) for i in range(n_blocks)]
        # volume only; reuse the variant replay on zero blocks
        spmm_all_ranks(led, op, hb, p, c, variant)

    for e in range(epochs):
        for l in range(nw):
            phase(fwd, dims[l])
        for l in range(nw - 1, -1, -1):
            phase(bwd, dims[l + 1])
            for j in range(c):
                led.allreduce(list(range(j, p, c)), dims[l] * dims[l + 1])
        led.marks[("epoch", e)] = led.snapshot()
    return led
