"""Locality-preserving SpMM schedules: the order in which a rank's rows are
processed by `dg_spmm_run`.

The order changes no number -- every row is still summed in its CSR storage
order -- it only decides which rows are in flight together, and therefore
which rows of H the GPU gathers at the same time.  On a graph with
community structure (ogbn-products: co-purchase clusters) processing rows
community by community keeps the gathered H rows L2-resident; in row order
(or after a random relabel) every window of rows gathers from the whole
table.

The communities are derived from the graph itself by label propagation on
the rank's own diagonal block (columns in [0, n_local): the rows whose
gathers stay on this GPU).  No external labels (no generator knowledge):
this is the B200 counterpart of the paper's METIS / GVB reordering step,
done per rank on the device in a few sort passes instead of on the host.
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["label_propagation", "community_order", "rank_row_order", "lpa_partition", "ORDERS"]

ORDERS = (None, "lpa")


def _edges(row_ptr, col, n_local, device):
    """(rows, cols) int64 device tensors of the entries whose column lies in
    the own block [0, n_local)."""
    rp = torch.as_tensor(np.asarray(row_ptr, dtype=np.int64), device=device)
    cols = (col if isinstance(col, torch.Tensor)
            else torch.from_numpy(np.ascontiguousarray(col))).to(device=device,
                                                                    dtype=torch.int64)
    n_rows = rp.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n_rows, device=device), rp[1:] - rp[:-1])
    keep = cols < n_local
    return rows[keep], cols[keep]


def label_propagation(rows, cols, n, iters=12, seed=0):
    """Label propagation over the edges (rows[k] -> cols[k]) of an n-vertex
    graph (both endpoints < n).  Every vertex adopts the most frequent label
    among its neighbours (ties: a seeded hash of the label, so no label
    wins ties everywhere); the two halves of the vertex set (by hash) update
    on alternate iterations, which stops the two-cycle oscillation of
    synchronous updates.  Deterministic for a given input.  Returns int64
    labels (on rows.device)."""
    dev = rows.device
    lab = torch.arange(n, device=dev, dtype=torch.int64)
    if rows.numel() == 0:
        return lab
    vid = torch.arange(n, device=dev, dtype=torch.int64)
    half = ((vid * 0x9E3779B1 + seed) >> 7) & 1
    for it in range(iters):
        key, _ = torch.sort(rows * n + lab[cols])
        uk, cnt = torch.unique_consecutive(key, return_counts=True)
        r, lb = uk // n, uk % n
        h = (lb * 0x85EBCA77 + (it + 1) * 0xC2B2AE3D + seed) & 0x7FFFFFFF
        score = (cnt.to(torch.int64) << 31) | h
        best = torch.full((n,), -1, dtype=torch.int64, device=dev)
        best.scatter_reduce_(0, r, score, reduce="amax")
        win = score == best[r]
        new = lab.clone()
        new[r[win]] = lb[win]
        upd = half == (it & 1)
        new = torch.where(upd, new, lab)
        changed = int((new != lab).sum())
        lab = new
        if changed <= n // 1000 and it >= 3:
            break
    return lab


def community_order(labels):
    """Rows grouped by label (groups in order of their first row), row order
    kept inside a group: int32 permutation."""
    n = labels.numel()
    dev = labels.device
    first = torch.full((n,), n, dtype=torch.int64, device=dev)
    first.scatter_reduce_(0, labels, torch.arange(n, device=dev), reduce="amin")
    key = first[labels] * n + torch.arange(n, device=dev)
    return torch.argsort(key).to(torch.int32).cpu().numpy()


def rank_row_order(ro, policy, device=None):
    """Processing order of one rank operand's rows under `policy`
    (None: row order, returns None; "lpa": label-propagation communities of
    the own diagonal block)."""
    if policy is None:
        return None
    if policy not in ORDERS:
        raise ValueError(f"row order must be one of {ORDERS}, got {policy!r}")
    n = int(ro.n_rows)
    if n == 0 or int(ro.n_local) != n:
        return None
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    rows, cols = _edges(ro.row_ptr, ro.col_ext, n, dev)
    lab = label_propagation(rows, cols, n)
    del rows, cols
    return community_order(lab)


def lpa_partition(a, k, device=None):
    """k-way partition of the graph `a` (CsrMatrix) from its own structure:
    label-propagation communities of the whole graph, packed onto k parts
    (largest first onto the part with the fewest nonzeros; a community
    heavier than a whole part is cut into row-order pieces first),
    vertices ordered by (part, community, id) so every part is community-
    ordered.  A graph-derived stand-in for the paper's METIS step that
    needs no host pass over the edges.  Returns a `Partition`."""
    from .partition import Partition
    n = int(a.n_rows)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    rows, cols = _edges(a.row_ptr, a.col_idx, n, dev)
    lab = label_propagation(rows, cols, n)
    del rows, cols
    lab = lab.cpu().numpy()
    deg = np.diff(np.asarray(a.row_ptr, dtype=np.int64)) + 1
    # dense community ids in order of first vertex
    _, first_idx, comm = np.unique(lab, return_index=True, return_inverse=True)
    rank_of = np.empty(first_idx.size, dtype=np.int64)
    rank_of[np.argsort(first_idx, kind="stable")] = np.arange(first_idx.size)
    comm = rank_of[comm]
    # cut oversized communities into pieces (row order inside a community)
    cap = max(1, -(-int(deg.sum()) // k))
    order = np.lexsort((np.arange(n), comm))
    w_sorted = deg[order]
    c_sorted = comm[order]
    cw = np.cumsum(w_sorted) - w_sorted                # weight before each vertex
    starts = np.flatnonzero(np.r_[True, c_sorted[1:] != c_sorted[:-1]])
    base = np.repeat(cw[starts], np.diff(np.r_[starts, n]))
    sub = (cw - base) // cap                           # piece inside the community
    _, piece_sorted = np.unique(c_sorted * (n + 1) + sub, return_inverse=True)
    piece = np.empty(n, dtype=np.int64)
    piece[order] = piece_sorted
    pid = int(piece_sorted.max()) if n else -1
    weights = np.bincount(piece, weights=deg, minlength=pid + 1)
    load = np.zeros(k, dtype=np.float64)
    part_of = np.zeros(pid + 1, dtype=np.int64)
    for pc in np.argsort(-weights, kind="stable"):
        t = int(np.argmin(load))
        part_of[pc] = t
        load[t] += weights[pc]
    asg = part_of[piece]
    vorder = np.lexsort((np.arange(n), piece, asg))
    perm = np.empty(n, dtype=np.int64)
    perm[vorder] = np.arange(n)
    sizes = np.bincount(asg, minlength=k)
    bounds, pos = [], 0
    for sz in sizes:
        bounds.append((pos, pos + int(sz)))
        pos += int(sz)
    return Partition(n, k, asg, perm, bounds)
