"""Distributed SpMM entry points -- the drop-in for `distgcn.spmm`.

Same names, arguments, return types and errors as the reference
(spmm.py:25-37): `VARIANTS`, `DistOperand`, `DistMatrices`,
`build_dist_matrices`, `exchange_index_lists`, `spmm_kernel`, `run_spmm`,
`serial_reference`, `validate_variant_grid`, `SpmmRun`.

`spmm_kernel(comm, op, h_block, variant)` is called from inside a rank
program exactly like the reference's; it is a collective over the ranks of
the process, and the last rank to arrive launches the batched device phase
(exchange -> SpMM -> 1.5D group reduction) for all of them.  The ledger is
charged from the plan with the reference's conventions, so volumes match
the reference bit-exactly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import DevicePlan, pad4, to_device
from .partition import Partition, apply_partition, block_partition
from .plan import (VARIANTS, DistMatrices, DistOperand, build_dist_matrices, build_variant_plan,
                   index_setup_charges, validate_variant_grid)
from .runtime import Comm, ProcessGrid, RunResult, run_program
from .sparse import CsrMatrix, local_spmm, transpose_csr

__all__ = ["DistMatrices", "DistOperand", "VARIANTS", "build_dist_matrices",
           "exchange_index_lists", "run_spmm", "serial_reference", "spmm_kernel",
           "validate_variant_grid", "SpmmRun", "device_plan", "spmm_phase", "row_group_reduce"]


def exchange_index_lists(comm: Comm, op: DistOperand, variant: str):
    """One-time NnzCols announcements (spmm.py:133-163).  The lists are
    already known to every host (the plan is deterministic), so nothing
    moves on the device; the reference's index traffic is charged once,
    by whichever rank arrives last."""
    grid = comm.grid
    ledger = comm.ledger

    def complete(arr):
        index_setup_charges(ledger, op, grid, variant)
        return {r: None for r in arr}

    comm._collective(("idx", id(op), variant), tuple(range(comm.p)), None, complete)


def device_plan(op: DistOperand, grid: ProcessGrid, variant: str, max_ld=None):
    """Device plan of `op` for `variant` covering the ranks this process
    hosts (all of them in a single-process run), built once and cached on
    the operand.  Multi-process plans register fixed-size IPC buffers, so
    they need the widest row pitch of the run (`max_ld`) up front."""
    from .dist import world
    w = world().init()
    local = w.local_ranks(grid.p) if w.multi else None
    key = (variant, grid.p, grid.c, torch.cuda.current_device())
    dp = op._device.get(key)
    if dp is not None and w.multi and max_ld is not None and max_ld > dp.max_ld:
        raise ValueError(f"row pitch {max_ld} exceeds this plan's registered {dp.max_ld}")
    if dp is None:
        dp = DevicePlan(build_variant_plan(op, grid, variant, local), local, max_ld=max_ld,
                        parities=getattr(op, "parities", 2),
                        row_order=getattr(op, "row_order", None))
        op._device[key] = dp
    return dp


def spmm_phase(comm: Comm, op: DistOperand, h_pad: torch.Tensor, f: int, variant: str,
               reduce: bool = True, reduce_f: int = None, out: torch.Tensor = None,
               fuse=None):
    """Device form of `spmm_kernel`: h_pad is a contiguous fp32 CUDA tensor
    (n_i, pad4(f)) with zero padding; returns the padded (n_i, pad4(f))
    product.  A collective over the ranks of this process: the last rank to
    arrive launches exchange -> SpMM -> (1.5D) group reduction for all.
    reduce=False (1.5D, extension): return each replica's partial product;
    the caller reduces after its transform and `reduce_f` is the width the
    ledger charges for that reduction.  `out` (optional): this rank's
    (n_i, pad4(f)) output buffer (the GCN loop's activation arena).
    `fuse` (optional, see `DevicePlan.run_fused`): (w, n_out, z, h) -- the
    layer's transform and ReLU fused into the SpMM epilogue; every rank
    passes its (bitwise identical) replica of w and its own z / h buffers;
    returns z.  The phase and its ledger charges are unchanged."""
    grid = comm.grid
    ledger = comm.ledger
    ld = pad4(f)

    def complete(arr):
        dp = device_plan(op, grid, variant, max_ld=ld)
        hs, outs = {}, {}
        for r, (h, o, _) in arr.items():
            hs[r] = h if (isinstance(h, torch.Tensor) and h.dtype == torch.float32
                          and h.is_cuda and h.is_contiguous() and h.shape[1] == ld) \
                else to_device(h[:, :f], ld)
            outs[r] = o
        if fuse is not None:
            fz = {r: fu for r, (_, _, fu) in arr.items()}
            w, n_out = fz[min(fz)][0], fz[min(fz)][1]
            z = {r: v[2] for r, v in fz.items()}
            hh = {r: v[3] for r, v in fz.items()}
            res = dp.run_fused(hs, f, ld, w, n_out, int(z[min(z)].shape[1]), z,
                               hh if all(v is not None for v in hh.values()) else None)
        else:
            given = all(o is not None for o in outs.values())
            res = dp.run(hs, f, ld, out=outs if given else None, reduce=reduce)
        dp.vplan.charge(ledger, f, None if reduce else reduce_f)
        return res

    return comm._collective(("spmm", id(op), variant, reduce, fuse is not None),
                            tuple(range(comm.p)), (h_pad, out, fuse), complete)


def row_group_reduce(comm: Comm, u: torch.Tensor, dm: DistMatrices, variant: str):
    """Row-group sum of a replica-partial (n_i x ld) tensor (the reduction
    that `spmm_phase(reduce=False)` deferred), bit-identical on the
    replicas.  Collective over the ranks of this process."""
    from .engine import RowGroupReducer
    rt = comm._rt
    ld = int(u.shape[1])

    def complete(arr):
        key = ("rowgroup", ld, id(dm))
        red = rt.ctx.get(key)
        if red is None:
            red = rt.ctx[key] = RowGroupReducer(comm.grid, device_plan(
                dm.fwd, comm.grid, variant).vplan, ld)
        return red(dict(arr))

    return comm._collective(("rowgroup", ld), tuple(range(comm.p)), u, complete)


def spmm_kernel(comm: Comm, op: DistOperand, h_block, variant: str):
    """One distributed multiply phase from inside a rank program
    (spmm.py:230-246).  h_block: this rank's block row of H (NumPy array or
    CUDA tensor, replicated over the row group when c > 1).  Returns the
    block row of the product: a CUDA tensor (n_i, f) for tensor input, a
    float64 NumPy array for NumPy input."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    numpy_in = not isinstance(h_block, torch.Tensor)
    f = int(h_block.shape[1])
    z = spmm_phase(comm, op, to_device(h_block, pad4(f)), f, variant)
    if numpy_in:
        return z[:, :f].double().cpu().numpy()
    return z if z.shape[1] == f else z[:, :f]


def serial_reference(a: CsrMatrix, h) -> np.ndarray:
    """transpose(a) @ h on one GPU (spmm.py:249-252)."""
    return local_spmm(transpose_csr(a), h)


@dataclass
class SpmmRun:
    z: np.ndarray
    ledger: object
    dm: DistMatrices
    partition: Partition
    grid: ProcessGrid


def run_spmm(a: CsrMatrix, h, p, c, variant, partition=None, index_setup=True) -> SpmmRun:
    """One distributed multiply end to end (spmm.py:264-294): permute by the
    partition (block by default), distribute on the (p/c) x c grid, run the
    variant on the GPU, gather back in the original order."""
    validate_variant_grid(variant, p, c)
    if a.n_rows != a.n_cols:
        raise ValueError("distributed multiply requires a square matrix")
    from .dist import world
    world().init()
    numpy_in = not isinstance(h, torch.Tensor)
    if numpy_in:
        h = np.asarray(h, dtype=np.float64)
    grid = ProcessGrid(p, c)
    part = partition if partition is not None else block_partition(a.n_rows, grid.n_rows)
    if part.k != grid.n_rows:
        raise ValueError(f"partition has {part.k} parts but the grid needs {grid.n_rows}")
    a2, h2 = apply_partition(a, h, part)
    dm = build_dist_matrices(a2, part.boundaries, grid)
    f = int(h2.shape[1])
    hd = to_device(h2, pad4(f))

    def program(comm):
        i, _ = comm.coords
        r0, r1 = dm.boundaries[i]
        if index_setup:
            exchange_index_lists(comm, dm.fwd, variant)
        return spmm_phase(comm, dm.fwd, hd[r0:r1], f, variant)

    run: RunResult = run_program(p, c, program)
    dev = hd.device
    z2 = torch.cat([run.results[grid.rank_of(i, 0)].to(dev) for i in range(grid.n_rows)],
                   0)[:, :f]
    dm.release_device()
    if not part.is_identity:
        z2 = z2[torch.from_numpy(part.perm).to(z2.device)]
    z = z2.double().cpu().numpy() if numpy_in else z2
    return SpmmRun(z, run.ledger, dm, part, grid)
