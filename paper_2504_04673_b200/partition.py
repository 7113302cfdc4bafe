"""K-way vertex partitions: layout, permutation and send-volume metrics.

Mirrors the partition API the hot path consumes (partition.py:19-30):
`Partition`, `block_partition`, `random_partition`, `apply_partition`,
`comm_metrics`, `edgecut`, `imbalance_pct`, `CommMetrics`.  Host
preprocessing, vectorised (O(nnz)) instead of the reference's per-vertex
Python loops.  The reference's partitioners (`greedy_tv_partition`,
`volume_balanced_refine`, partition.py:257-428) are one-time host
preprocessing outside the hot path; they run natively (csrc/partition.cu,
identical assignments) so the volume-balanced configurations are feasible
at millions of vertices.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import CsrMatrix

__all__ = ["CommMetrics", "Partition", "apply_partition", "block_partition", "comm_metrics",
           "edgecut", "greedy_tv_partition", "imbalance_pct", "random_partition", "read_partition",
           "volume_balanced_refine", "write_partition"]

import logging

log = logging.getLogger(__name__)


def _bounds(sizes):
    out, pos = [], 0
    for s in sizes:
        out.append((pos, pos + int(s)))
        pos += int(s)
    return out


@dataclass
class Partition:
    """k-way partition with its row layout (partition.py:35-102)."""

    n: int
    k: int
    assignment: np.ndarray
    perm: np.ndarray
    boundaries: list

    def __post_init__(self):
        self.assignment = np.asarray(self.assignment, dtype=np.int64)
        self.perm = np.asarray(self.perm, dtype=np.int64)
        self.validate()

    @classmethod
    def from_assignment(cls, assignment, k) -> "Partition":
        """Canonical layout: parts ascending, original order kept inside a
        part (stable sort, partition.py:55-65)."""
        assignment = np.asarray(assignment, dtype=np.int64)
        n = assignment.size
        order = np.argsort(assignment, kind="stable")
        perm = np.empty(n, dtype=np.int64)
        perm[order] = np.arange(n)
        return cls(n, k, assignment, perm, _bounds(np.bincount(assignment, minlength=k)))

    def validate(self):
        if self.k < 1:
            raise ValueError("k must be at least 1")
        if self.assignment.shape != (self.n,):
            raise ValueError("assignment must have one entry per vertex")
        if self.assignment.size and (self.assignment.min() < 0 or self.assignment.max() >= self.k):
            raise ValueError("part ids must lie in [0, k)")
        if self.perm.shape != (self.n,) or (self.n and not np.array_equal(
                np.bincount(self.perm, minlength=self.n), np.ones(self.n, np.int64))):
            raise ValueError("perm must be a bijection on [0, n)")
        if len(self.boundaries) != self.k:
            raise ValueError("need one boundary range per part")
        pos = 0
        for s, e in self.boundaries:
            if s != pos or e < s:
                raise ValueError("boundaries must be consecutive and cover [0, n)")
            pos = e
        if pos != self.n:
            raise ValueError("boundaries must cover [0, n)")
        widths = np.array([e - s for s, e in self.boundaries])
        if not np.array_equal(np.bincount(self.assignment, minlength=self.k), widths):
            raise ValueError("boundary widths must match part sizes")
        new_to_part = self.assignment[self.inv_perm]
        if self.n and np.any(np.diff(new_to_part) < 0):
            raise ValueError("parts must occupy contiguous ascending new-id ranges")

    @property
    def inv_perm(self) -> np.ndarray:
        inv = np.empty(self.n, dtype=np.int64)
        inv[self.perm] = np.arange(self.n)
        return inv

    @property
    def part_sizes(self) -> np.ndarray:
        return np.bincount(self.assignment, minlength=self.k)

    @property
    def is_identity(self) -> bool:
        return bool(np.array_equal(self.perm, np.arange(self.n)))


@dataclass
class CommMetrics:
    """Send volume of one partition in dense rows (partition.py:105-141)."""

    per_part_send_rows: np.ndarray
    total_rows: int
    max_rows: float
    avg_rows: float
    imbalance_pct: float
    cut_p: int
    f: int = 1
    pair_rows: np.ndarray = None

    def to_dict(self) -> dict:
        return {
            "per_part_send_rows": [int(x) for x in self.per_part_send_rows],
            "total_rows": int(self.total_rows),
            "max_rows": float(self.max_rows),
            "avg_rows": float(self.avg_rows),
            "imbalance_pct": float(self.imbalance_pct),
            "cut_p": int(self.cut_p),
            "f": int(self.f),
            "total_bytes": float(self.total_rows * self.f * 8),
            "max_bytes": float(self.max_rows * self.f * 8),
        }


def imbalance_pct(avg, mx) -> float:
    if avg <= 0:
        return 0.0
    return 100.0 * (mx - avg) / avg


def _check_kn(n, k):
    if k < 1:
        raise ValueError("k must be at least 1")
    if k > n:
        raise ValueError(f"cannot split {n} vertices into {k} parts")


def block_partition(n, k) -> Partition:
    """Contiguous blocks, first n mod k parts one larger (partition.py:154-161)."""
    _check_kn(n, k)
    base, rem = divmod(n, k)
    sizes = [base + 1] * rem + [base] * (k - rem)
    return Partition.from_assignment(np.repeat(np.arange(k, dtype=np.int64), sizes), k)


def random_partition(n, k, seed) -> Partition:
    """Seeded random relabel then even split (partition.py:164-171); the
    same draw as the reference, so the same partition."""
    _check_kn(n, k)
    perm = np.random.default_rng(seed).permutation(n).astype(np.int64)
    base, rem = divmod(n, k)
    sizes = [base + 1] * rem + [base] * (k - rem)
    part_of_new = np.repeat(np.arange(k, dtype=np.int64), sizes)
    return Partition(n, k, part_of_new[perm], perm, _bounds(sizes))


def edgecut(a: CsrMatrix, part: Partition) -> int:
    """Undirected edges crossing parts (partition.py:190-198)."""
    r, c = a.row_of_nnz(), a.col_idx
    keep = r != c
    r, c = r[keep], c[keep]
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    key = np.unique(lo * a.n_rows + hi)
    lo, hi = key // a.n_rows, key % a.n_rows
    return int(np.count_nonzero(part.assignment[lo] != part.assignment[hi]))


def comm_metrics(a: CsrMatrix, part: Partition, f=1) -> CommMetrics:
    """Per-part send rows of one aware multiply (partition.py:201-228):
    vertex v of part s ships one row to every foreign part holding an
    out-neighbour of v.  Vectorised over (vertex, part) pairs."""
    if a.n_rows != a.n_cols or a.n_rows != part.n:
        raise ValueError("partition does not match the matrix")
    k = part.k
    asg = part.assignment
    rows = a.row_of_nnz()
    key = np.unique(rows * k + asg[a.col_idx])
    v, t = key // k, key % k
    own = asg[v]
    foreign = t != own
    pair = np.zeros((k, k), dtype=np.int64)
    np.add.at(pair, (t[foreign], own[foreign]), 1)
    send = pair.sum(axis=0)
    total = int(send.sum())
    mx = float(send.max()) if k else 0.0
    avg = total / k
    off = pair[~np.eye(k, dtype=bool)]
    cut_p = int(off.max()) if off.size else 0
    return CommMetrics(send, total, mx, avg, imbalance_pct(avg, mx), cut_p, f, pair)


def apply_partition(a: CsrMatrix, h, part: Partition):
    """(P A P^T, h[inv_perm]) (partition.py:231-254).  Identity partitions
    (the block default) return the inputs without the O(nnz log nnz) sort."""
    if a.n_rows != a.n_cols:
        raise ValueError("symmetric permutation requires a square matrix")
    if a.n_rows != part.n:
        raise ValueError("partition does not match the matrix")
    if h is not None:
        if h.shape[0] != a.n_rows:
            raise ValueError("row count of h must match the matrix")
    if part.is_identity:
        return a, h
    from . import _lib as L
    perm = np.ascontiguousarray(part.perm, dtype=np.int64)
    rp = np.zeros(a.n_rows + 1, dtype=np.int64)
    ci = np.empty(a.nnz, dtype=np.int64)
    va = np.empty(a.nnz, dtype=np.float64)
    src = [np.ascontiguousarray(x) for x in (a.row_ptr, a.col_idx, a.values)]
    rc = L.host_lib().dg_host_permute(a.n_rows, src[0].ctypes.data, src[1].ctypes.data,
                                      src[2].ctypes.data, perm.ctypes.data, rp.ctypes.data,
                                      ci.ctypes.data, va.ctypes.data)
    if rc != 0:
        raise ValueError(L.host_lib().dg_last_error().decode())
    a2 = CsrMatrix(a.n_rows, a.n_cols, rp, ci, va, check=False)
    h2 = None if h is None else h[part.inv_perm]
    return a2, h2


def read_partition(path, k=None) -> Partition:
    """Reference on-disk format: line i = part of vertex i (io.py:217-238)."""
    asg = np.loadtxt(path, dtype=np.int64, ndmin=1)
    return Partition.from_assignment(asg, int(asg.max()) + 1 if k is None else k)


def write_partition(path, part: Partition):
    np.savetxt(path, part.assignment, fmt="%d")


def _sym_pattern(a: CsrMatrix) -> CsrMatrix:
    """Undirected pattern of a (union with its transpose), diagonal removed
    (partition.py:174-183)."""
    from .sparse import transpose_csr
    at = transpose_csr(a)
    rows = a.row_of_nnz()
    if np.array_equal(at.row_ptr, a.row_ptr) and np.array_equal(at.col_idx, a.col_idx):
        keep = rows != a.col_idx                          # structurally symmetric
        r, c = rows[keep], a.col_idx[keep]
    else:
        r = np.concatenate([rows, a.col_idx])
        c = np.concatenate([a.col_idx, rows])
        keep = r != c
        key = np.unique(r[keep] * a.n_rows + c[keep])
        r, c = key // a.n_rows, key % a.n_rows
    rp = np.zeros(a.n_rows + 1, dtype=np.int64)
    if r.size:
        np.cumsum(np.bincount(r, minlength=a.n_rows), out=rp[1:])
    return CsrMatrix(a.n_rows, a.n_cols, rp, c, np.ones(c.size), check=False)


def greedy_tv_partition(a: CsrMatrix, k, epsilon=0.10, max_passes=10) -> Partition:
    """BFS-grown parts refined by greedy edgecut-reducing moves
    (partition.py:257-289), run natively with the reference's orders and
    tie-breaks."""
    from . import _lib as L
    if a.n_rows != a.n_cols:
        raise ValueError("partitioning requires a square matrix")
    n = a.n_rows
    _check_kn(n, k)
    pat = _sym_pattern(a)
    asg = np.empty(n, dtype=np.int64)
    relaxed = np.zeros(1, dtype=np.int32)
    rc = L.host_lib().dg_host_greedy_tv(n, pat.row_ptr.ctypes.data, pat.col_idx.ctypes.data, k,
                                        float(epsilon), int(max_passes), asg.ctypes.data,
                                        relaxed.ctypes.data)
    if rc != 0:
        raise ValueError(L.host_lib().dg_last_error().decode())
    if relaxed[0]:
        w = np.maximum(np.diff(pat.row_ptr), 1)
        log.warning("a single vertex carries %d nonzeros, above the balance cap %.1f; "
                    "relaxing the constraint to row granularity", int(w.max()),
                    (1.0 + epsilon) * w.sum() / k)
    return Partition.from_assignment(asg, k)


def volume_balanced_refine(a: CsrMatrix, part: Partition, lambda_max=None, epsilon=0.10,
                           max_passes=10) -> Partition:
    """Boundary refinement of total and bottleneck send volume
    (partition.py:342-428), run natively with the reference's orders and
    tie-breaks."""
    from . import _lib as L
    from .sparse import transpose_csr
    if a.n_rows != a.n_cols or a.n_rows != part.n:
        raise ValueError("partition does not match the matrix")
    n, k = part.n, part.k
    lam = float(k) if lambda_max is None else float(lambda_max)
    at = transpose_csr(a)
    pat = _sym_pattern(a)
    asg = part.assignment.astype(np.int64).copy()
    arrs = [np.ascontiguousarray(x, dtype=np.int64) for x in
            (a.row_ptr, a.col_idx, at.row_ptr, at.col_idx, pat.row_ptr)]
    rc = L.host_lib().dg_host_gvb(n, *[x.ctypes.data for x in arrs], k, lam, float(epsilon),
                                  int(max_passes), asg.ctypes.data)
    if rc != 0:
        raise ValueError(L.host_lib().dg_last_error().decode())
    return Partition.from_assignment(asg, k)
