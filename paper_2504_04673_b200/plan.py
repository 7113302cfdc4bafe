"""Host plan builder: block layout, NnzCols lists, per-rank remapped CSR,
exchange segments and the analytic ledger charges of every variant.

Follows spmm.py:80-130 (`_extract_operand`, `build_dist_matrices`,
`validate_variant_grid`) for the layout and the per-peer row lists, and
spmm.py:133-227 for which rows each variant moves where.  Runs once per
operand (the sparse pattern is fixed for a whole run, spmm.py:140-141);
O(nnz + p*n) with occupancy masks instead of per-block sorts.

Device layout produced here:
  rank (i, j) owns block row i of the operand restricted to the column
  blocks it multiplies (all blocks in 1D; the stage band q in
  [j*s, (j+1)*s) in 1.5D).  Its columns are renumbered into an extended
  space [own block i | halo segment of source q0 | q1 | ...] (ascending q).
  Entries keep the reference's storage order (ascending global column),
  so the summation order -- and therefore the result -- does not depend
  on the variant.  The received rows land directly in the halo segments:
  the reference's `_scatter` (spmm.py:166-169) disappears.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .runtime import CommLedger, ProcessGrid
from .sparse import CsrMatrix, csr_equal, transpose_csr

VARIANTS = ("1d-oblivious", "1d-sparse", "15d-oblivious", "15d-sparse")


def validate_variant_grid(variant, p, c):
    """spmm.py:120-130, same messages."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    if variant.startswith("1d") and c != 1:
        raise ValueError(f"variant {variant} requires c == 1 (got c={c})")
    if p % c != 0:
        raise ValueError(f"c must divide p (p={p}, c={c})")
    if variant.startswith("15d") and p % (c * c) != 0:
        raise ValueError(f"variant {variant} requires c*c to divide p (p={p}, c={c})")


class DistOperand:
    """One sparse operand split into a grid of blocks (spmm.py:40-54).

    `nnz_cols[(i, j)]` holds the sorted occupied local columns of block
    (i, j) -- exactly the reference's `np.unique(sub_cols)` list -- and
    `widths` the block widths.  `blocks[i][j]` (block-local CSR) is built
    lazily: the device path never needs it.
    """

    def __init__(self, mat: CsrMatrix, boundaries):
        self.mat = mat
        self.boundaries = [tuple(b) for b in boundaries]
        self.widths = [e - s for s, e in self.boundaries]
        nb = len(self.boundaries)
        n = mat.n_cols
        self.starts = np.array([s for s, _ in self.boundaries] + [n], dtype=np.int64)
        part_of = np.repeat(np.arange(nb, dtype=np.int32), self.widths)
        self.nnz_cols = {}
        self._owner = []      # per block row: owner block of each entry (int32)
        self._pos = []        # per block row: position inside nnz_cols[(i, owner)] (int32)
        occ = np.zeros(n, dtype=bool)
        for i, (r0, r1) in enumerate(self.boundaries):
            lo, hi = int(mat.row_ptr[r0]), int(mat.row_ptr[r1])
            cols = mat.col_idx[lo:hi]
            owner = part_of[cols] if cols.size else np.zeros(0, np.int32)
            occ[:] = False
            occ[cols] = True
            uniq = np.flatnonzero(occ)
            rank_in_u = np.cumsum(occ, dtype=np.int64) - 1
            split = np.searchsorted(uniq, self.starts)
            for j in range(nb):
                self.nnz_cols[(i, j)] = uniq[split[j]:split[j + 1]] - self.starts[j]
            pos = (rank_in_u[cols] - split[owner]).astype(np.int32) if cols.size else \
                np.zeros(0, np.int32)
            self._owner.append(owner)
            self._pos.append(pos)
        self._blocks = None
        self._device = {}     # (variant, device key) -> device plan

    @property
    def n_blocks(self) -> int:
        return len(self.boundaries)

    def release_device(self):
        """Free the cached device plans (collective under torchrun)."""
        for dp in self._device.values():
            dp.close()
        self._device.clear()

    @property
    def blocks(self):
        if self._blocks is None:
            self._blocks = [[self.block(i, j) for j in range(self.n_blocks)]
                            for i in range(self.n_blocks)]
        return self._blocks

    def block(self, i, j) -> CsrMatrix:
        """Block (i, j) with block-local columns (spmm.py:93-101)."""
        r0, r1 = self.boundaries[i]
        lo, hi = int(self.mat.row_ptr[r0]), int(self.mat.row_ptr[r1])
        sel = self._owner[i] == j
        rows = self.mat.row_of_nnz()[lo:hi][sel] - r0
        rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        if rows.size:
            np.cumsum(np.bincount(rows, minlength=r1 - r0), out=rp[1:])
        return CsrMatrix(r1 - r0, self.widths[j], rp,
                         self.mat.col_idx[lo:hi][sel] - self.starts[j],
                         self.mat.values[lo:hi][sel], check=False)


@dataclass
class DistMatrices:
    """Operands on a grid (spmm.py:57-77): fwd = blocks of A^T, bwd = blocks
    of A, aliased when A is symmetric."""

    grid: ProcessGrid
    boundaries: list
    fwd: DistOperand
    bwd: DistOperand
    n: int

    @property
    def symmetric(self) -> bool:
        return self.bwd is self.fwd

    def release_device(self):
        self.fwd.release_device()
        if self.bwd is not self.fwd:
            self.bwd.release_device()


def build_dist_matrices(a: CsrMatrix, boundaries, grid: ProcessGrid) -> DistMatrices:
    """spmm.py:108-117."""
    bounds = list(getattr(boundaries, "boundaries", boundaries))
    if len(bounds) != grid.n_rows:
        raise ValueError(f"need {grid.n_rows} block rows for this grid, got {len(bounds)}")
    at = transpose_csr(a)
    fwd = DistOperand(at, bounds)
    bwd = fwd if csr_equal(at, a) else DistOperand(a, bounds)
    return DistMatrices(grid, bounds, fwd, bwd, a.n_rows)


# ---------------------------------------------------------------------------
# per-variant plan
# ---------------------------------------------------------------------------

@dataclass
class RankOperand:
    rank: int
    i: int
    j: int
    n_rows: int
    n_local: int
    row_ptr: np.ndarray      # int64
    col_ext: np.ndarray      # int32, extended column space
    val: np.ndarray          # float32
    halo_rows: int
    halo_off: dict           # source block q -> first halo row


@dataclass
class Segment:
    src: int                 # sending rank
    dst: int                 # receiving rank
    q: int                   # source block row
    idx: object              # int32 local rows of H_q, or None (whole block)
    count: int
    dst_row0: int


@dataclass
class VariantPlan:
    grid: ProcessGrid
    variant: str
    ranks: list              # RankOperand per rank
    segments: list
    widths: list
    nnz_cols: dict = field(repr=False, default=None)

    def charge(self, ledger: CommLedger, f: int, reduce_f: int = None):
        """Ledger charges of one multiply phase of width f -- exactly what
        the reference's collectives charge for the same phase.  `reduce_f`
        (extension): the width of the 1.5D row-group reduction when it runs
        after the transform (n_i x f_out instead of n_i x f_in)."""
        p, c = self.grid.p, self.grid.c
        allr = tuple(range(p))
        if self.variant == "1d-oblivious":
            for j in range(p):                                   # spmm.py:176-177
                ledger.broadcast(j, allr, self.widths[j] * f)
        elif self.variant == "1d-sparse":                         # spmm.py:185-186
            ledger.alltoallv(allr, {(s.src, s.dst): s.count * f for s in self.segments})
        else:                                                     # spmm.py:203-227
            for s in self.segments:
                ledger.p2p(s.src, s.dst, s.count * f)
            rf = f if reduce_f is None else reduce_f
            for i in range(self.grid.n_rows):
                ledger.allreduce(self.grid.row_group(i), self.widths[i] * rf)

    def elements(self, f: int) -> int:
        """Exchanged data elements of one phase (excluding the 1.5D reduction)."""
        if self.variant == "1d-oblivious":
            return sum(self.widths) * (self.grid.p - 1) * f
        return sum(s.count for s in self.segments) * f


def stage_band(grid: ProcessGrid, j):
    s = grid.stage_count()
    return list(range(j * s, (j + 1) * s))


def build_variant_plan(op: DistOperand, grid: ProcessGrid, variant: str,
                       local_ranks=None) -> VariantPlan:
    """Plan of `variant` on `grid`.  The halo layout and exchange segments
    are computed for every rank (every process needs its peers' offsets);
    the remapped CSR only for `local_ranks` (default: all)."""
    if hasattr(op, "build_variant_plan"):          # HBM-resident operand (sharded.py)
        return op.build_variant_plan(grid, variant, local_ranks)
    validate_variant_grid(variant, grid.p, grid.c)
    hosted = set(range(grid.p)) if local_ranks is None else set(local_ranks)
    aware = variant.endswith("sparse")
    one_d = variant.startswith("1d")
    nb = op.n_blocks
    widths = op.widths
    mat = op.mat
    row_all = mat.row_of_nnz()
    ranks = []
    for r in range(grid.p):
        i, j = grid.coords(r)
        sources = list(range(nb)) if one_d else stage_band(grid, j)
        r0, r1 = op.boundaries[i]
        lo, hi = int(mat.row_ptr[r0]), int(mat.row_ptr[r1])
        owner = op._owner[i]
        # halo segments, ascending source block
        halo_off, off = {}, 0
        for q in sources:
            if q == i:
                continue
            cnt = op.nnz_cols[(i, q)].size if aware else widths[q]
            if not one_d and aware and cnt == 0:
                continue
            halo_off[q] = off
            off += cnt
        if r not in hosted:
            ranks.append(RankOperand(r, i, j, r1 - r0, r1 - r0, None, None, None, off, halo_off))
            continue
        local_rows = row_all[lo:hi] - r0
        cols = mat.col_idx[lo:hi]
        vals = mat.values[lo:hi]
        if one_d:
            keep = slice(None)
        else:
            keep = (owner >= sources[0]) & (owner <= sources[-1])
        cols, vals, own, rows = cols[keep], vals[keep], owner[keep], local_rows[keep]
        pos = op._pos[i][keep]
        base = np.zeros(nb, dtype=np.int64)
        for q, o in halo_off.items():
            base[q] = r1 - r0 + o
        if aware:
            ext = base[own] + pos
        else:
            ext = base[own] + (cols - op.starts[own])
        is_local = own == i
        ext = np.where(is_local, cols - r0, ext).astype(np.int32)
        rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        if rows.size:
            np.cumsum(np.bincount(rows, minlength=r1 - r0), out=rp[1:])
        ranks.append(RankOperand(r, i, j, r1 - r0, r1 - r0, rp, ext,
                                 vals.astype(np.float32), off, halo_off))
    segments = []
    if one_d:
        for s in range(grid.p):                                  # sender = block s
            for d in range(grid.p):
                if d == s:
                    continue
                if aware:
                    idx = op.nnz_cols[(d, s)].astype(np.int32)
                    cnt = idx.size
                else:
                    idx, cnt = None, widths[s]
                segments.append(Segment(s, d, s, idx, cnt, ranks[d].halo_off.get(s, 0)))
    else:
        s_stage = grid.stage_count()
        for q in range(nb):                                      # band owner (q, q // s)
            jq = q // s_stage
            src = grid.rank_of(q, jq)
            for l in range(nb):
                if l == q:
                    continue
                dst = grid.rank_of(l, jq)
                if aware:
                    idx = op.nnz_cols[(l, q)].astype(np.int32)
                    if idx.size == 0:
                        continue
                    cnt = idx.size
                else:
                    idx, cnt = None, widths[q]
                segments.append(Segment(src, dst, q, idx, cnt, ranks[dst].halo_off[q]))
    return VariantPlan(grid, variant, ranks, segments, widths, op.nnz_cols)


def index_setup_charges(ledger: CommLedger, op: DistOperand, grid: ProcessGrid, variant: str):
    """Ledger of `exchange_index_lists` (spmm.py:133-163): one int64 list per
    (receiver -> owner) pair, charged as index traffic.  The lists never
    cross to the device at run time (the plan is built on every host)."""
    if variant.endswith("oblivious"):
        return
    if variant == "1d-sparse":
        for r in range(grid.p):
            for dst in range(grid.p):
                if dst != r and op.nnz_cols[(r, dst)].size:
                    ledger.p2p(r, dst, op.nnz_cols[(r, dst)].size, "index", wire=0)
        return
    s = grid.stage_count()
    for r in range(grid.p):
        i, j = grid.coords(r)
        for k in range(s):
            q = j * s + k
            if q != i and op.nnz_cols[(i, q)].size:
                ledger.p2p(r, grid.rank_of(q, j), op.nnz_cols[(i, q)].size, "index", wire=0)
