"""Full-batch GCN training on the GPU -- the drop-in for `distgcn.gcn`.

Same API (gcn.py:27-37): `TrainConfig`, `TrainResult`, `SerialGcn`,
`init_weights`, `relu`, `relu_grad`, `softmax_xent`, `serial_train`,
`train`.  The epoch loop is the reference's (gcn.py:258-286), step for
step: per weight layer a forward multiply `spmm_kernel(fwd)` then `T W`
and ReLU; masked softmax cross-entropy; per layer (reversed) a backward
multiply `spmm_kernel(bwd)`, the weight gradient `H^T M` all-reduced over
the column group, `G = (M W^T) * 1[Z > 0]` with W before its update, and
SGD.  Every rank's data stays on the GPU for the whole run; loss and
accuracy are accumulated on the device and read back once at the end.

Numerics: fp32 storage; SpMM sums in fp32 windows folded into a second fp32
(rows >= 32 floats) or fp64 (narrower rows) accumulator; GEMMs fp32
with TF32 off.  Widths are padded to multiples of 4 (zero padding, also in
the weights) so every activation is a 16-byte-aligned row-major tensor.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .engine import _no_tf32, pad4, to_device
from .partition import Partition, apply_partition, block_partition
from .plan import build_dist_matrices, validate_variant_grid
from .runtime import ProcessGrid, run_program
from .sparse import CsrMatrix, csr_equal, local_spmm, transpose_csr
from .spmm import exchange_index_lists, row_group_reduce, spmm_phase

__all__ = ["SerialGcn", "TrainConfig", "TrainResult", "init_weights", "relu", "relu_grad",
           "serial_train", "softmax_xent", "train"]


@dataclass
class TrainConfig:
    """gcn.py:40-73.  `layers` counts representation levels: layers=3 trains
    two weight matrices."""

    layers: int = 3
    hidden: int = 16
    lr: float = 0.01
    epochs: int = 100
    activation: str = "relu"
    seed: int = 0
    variant: str = "1d-sparse"
    f_in: int = None
    f_out: int = None
    # extension (not in the reference): "transform-first" computes
    # A^T (H W) instead of (A^T H) W for layers that shrink the width --
    # the same function, with the forward multiply (and its exchange) at the
    # narrower width; the backward pass is unchanged.  Default: the
    # reference's aggregate-first order (gcn.py:273-274), exact volumes.
    order: str = "aggregate-first"
    # extension: in the 1.5D variants, reduce the c replica
    # partials after the transform (n_i x f_out) instead of before it
    # (n_i x f_in), since (sum_j T_j) W = sum_j (T_j W).  Off by default:
    # the reference reduces before (spmm.py:227).
    reduce_after_transform: bool = False

    def __post_init__(self):
        if self.layers < 2:
            raise ValueError("need at least 2 layers (one weight matrix)")
        if self.hidden < 1:
            raise ValueError("hidden width must be at least 1")
        if self.lr < 0:
            raise ValueError("learning rate must be non-negative")
        if self.epochs < 0:
            raise ValueError("epochs must be non-negative")
        if self.activation != "relu":
            raise ValueError(f"unsupported activation {self.activation!r}")
        if self.order not in ("aggregate-first", "transform-first"):
            raise ValueError(f"unknown order {self.order!r}")

    def layer_dims(self, f_in, f_out):
        return [f_in] + [self.hidden] * (self.layers - 2) + [f_out]


def _dev():
    L.lib()
    return torch.device("cuda", torch.cuda.current_device())


def relu(z):
    """max(z, 0) on the GPU (gcn.py:76-77)."""
    t = z if isinstance(z, torch.Tensor) else torch.from_numpy(np.asarray(z, dtype=np.float64))
    out = torch.clamp_min(t.to(_dev()), 0.0)
    return out if isinstance(z, torch.Tensor) else out.cpu().numpy()


def relu_grad(z):
    """1[z > 0] (gcn.py:80-82), 0 at exactly 0."""
    t = z if isinstance(z, torch.Tensor) else torch.from_numpy(np.asarray(z, dtype=np.float64))
    out = (t.to(_dev()) > 0).to(t.dtype)
    return out if isinstance(z, torch.Tensor) else out.cpu().numpy()


def init_weights(cfg: TrainConfig, f_in, f_out):
    """Seeded symmetric-uniform init (gcn.py:85-95), identical draws."""
    rng = np.random.default_rng(cfg.seed)
    dims = cfg.layer_dims(f_in, f_out)
    out = []
    for fi, fo in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fi + fo))
        out.append(rng.uniform(-lim, lim, size=(fi, fo)))
    return out


class _Xent:
    """Device masked softmax cross-entropy (dg_xent) with its scratch."""

    def __init__(self, n, device):
        blocks = (max(n, 1) + 7) // 8
        self.scratch = torch.zeros(2 * blocks + 2, dtype=torch.float64, device=device)
        self.counter = torch.zeros(1, dtype=torch.int32, device=device)

    def __call__(self, logits, C, labels, mask_u8, denom, grad, stats):
        n = logits.shape[0]
        if n == 0:
            return
        L.check(L.lib().dg_xent(logits.data_ptr(), n, C, logits.stride(0), labels.data_ptr(),
                                mask_u8.data_ptr(), float(denom), grad.data_ptr(),
                                grad.stride(0), self.scratch.data_ptr(),
                                self.counter.data_ptr(), stats.data_ptr(), L.stream_ptr()))


def softmax_xent(logits, labels, mask):
    """Mean masked cross-entropy and its gradient (gcn.py:123-132)."""
    logits_np = np.asarray(logits, dtype=np.float64)
    labels = np.asarray(labels)
    mask = np.asarray(mask, dtype=bool)
    count = int(mask.sum())
    if count == 0:
        raise ValueError("softmax_xent needs at least one masked row")
    C = logits_np.shape[1]
    sel = labels[mask]
    if sel.min() < 0 or sel.max() >= C:
        raise ValueError(f"labels must lie in [0, {C}) on masked rows")
    dev = _dev()
    ld = pad4(C)
    x = to_device(logits_np, ld)
    grad = torch.zeros_like(x)
    stats = torch.zeros(2, dtype=torch.float64, device=dev)
    _Xent(x.shape[0], dev)(x, C, torch.from_numpy(labels.astype(np.int64)).to(dev),
                           torch.from_numpy(mask.astype(np.uint8)).to(dev), count, grad, stats)
    st = stats.cpu().numpy()
    return float(st[0] / count), grad[:, :C].double().cpu().numpy()


class SerialGcn:
    """Forward/backward on the undistributed matrix (gcn.py:135-172), on the
    GPU; NumPy in / NumPy out like the reference."""

    def __init__(self, a_hat: CsrMatrix, weights):
        self.a = a_hat
        at = transpose_csr(a_hat)
        self.at = a_hat if csr_equal(at, a_hat) else at
        self.weights = weights
        self._cache = None

    def forward(self, h0):
        dev = _dev()
        hs = [torch.as_tensor(np.asarray(h0, dtype=np.float64), device=dev).float()]
        zs = []
        last = len(self.weights) - 1
        with _no_tf32():
            for l, w in enumerate(self.weights):
                t = local_spmm(self.at, hs[-1])
                z = t @ torch.as_tensor(np.asarray(w), device=dev).float()
                zs.append(z)
                hs.append(torch.clamp_min(z, 0.0) if l < last else z)
        self._cache = (hs, zs)
        return hs[-1].double().cpu().numpy()

    def backward(self, g_out):
        if self._cache is None:
            raise RuntimeError("backward called before forward")
        hs, zs = self._cache
        dev = _dev()
        g = torch.as_tensor(np.asarray(g_out, dtype=np.float64), device=dev).float()
        ys = [None] * len(self.weights)
        with _no_tf32():
            for l in range(len(self.weights) - 1, -1, -1):
                m = local_spmm(self.a, g)
                ys[l] = (hs[l].T @ m).double().cpu().numpy()
                if l > 0:
                    w = torch.as_tensor(np.asarray(self.weights[l]), device=dev).float()
                    g = (m @ w.T) * (zs[l - 1] > 0)
        return ys


@dataclass
class TrainResult:
    """gcn.py:175-197."""

    history: list
    weights: list
    ledger: object = None
    partition: Partition = None
    weights_per_rank: list = field(default_factory=list)

    @property
    def losses(self):
        return np.array([row["loss"] for row in self.history])

    @property
    def final_accuracy(self):
        return self.history[-1]["train_acc"] if self.history else None


def _check_train_inputs(features, labels, train_mask):
    n_f = features.shape[0]
    labels = np.asarray(labels, dtype=np.int64)
    mask = np.asarray(train_mask, dtype=bool)
    if not (n_f == labels.shape[0] == mask.shape[0]):
        raise ValueError("features, labels and train_mask must agree on the vertex count")
    if int(mask.sum()) == 0:
        raise ValueError("train_mask must select at least one vertex")
    return labels, mask


class _Arena:
    """Per-rank activation buffers reused across epochs (one flat buffer per
    slot, grown only when a larger view is requested).  At papers scale the
    epoch's four ~20 GB activations would otherwise be fresh caching-allocator
    requests every epoch -- occasionally several seconds of allocator
    recovery.  Slot lifetimes (gcn.py:270-285): "t" the forward SpMM output
    (consumed by that layer's transform), "l" the logits (until the loss),
    then the backward SpMM outputs (the logits are dead by then), "g" the
    loss gradient."""

    def __init__(self, device):
        self.device = device
        self.bufs = {}

    def get(self, slot, rows, ld):
        need = rows * ld
        buf = self.bufs.get(slot)
        if buf is None or buf.numel() < need:
            self.bufs[slot] = buf = None
            buf = self.bufs[slot] = torch.empty(max(need, 4), dtype=torch.float32,
                                                device=self.device)
        return buf[:need].view(rows, ld)


class _Dense:
    """The GCN step's dense transforms on the library's kernels
    (dg_dense_rows / dg_dense_tn); cuBLAS (torch.mm, TF32 off) only for
    shapes outside their range."""

    def __init__(self, device):
        self.device = device
        self.work = torch.zeros(1, dtype=torch.float64, device=device)

    @staticmethod
    def _rows_ok(K, N):
        return N <= 64 and K * 16 * ((N + 15) // 16) <= 16384

    def fwd(self, t, w, f_in, f_out, relu, z=None):
        """z = t @ w (padded), h = relu(z) if requested (gcn.py:274-276);
        `z` optionally preallocated (n x ld_out)."""
        n, ldo = t.shape[0], w.shape[1]
        if not self._rows_ok(f_in, f_out):
            z = torch.mm(t, w) if z is None else torch.mm(t, w, out=z)
            return z, (torch.clamp_min(z, 0.0) if relu else None)
        if z is None:
            z = torch.empty((n, ldo), dtype=torch.float32, device=self.device)
        h = torch.empty_like(z) if relu else None
        L.check(L.lib().dg_dense_rows(t.data_ptr(), t.stride(0), n, f_in, w.data_ptr(),
                                      w.stride(0), f_out, 0, z.data_ptr(), ldo,
                                      0 if h is None else h.data_ptr(), 0, 0, L.stream_ptr()))
        return z, h

    def bwd(self, m, w, f_in, f_out, zprev):
        """g = (m @ w^T) * 1[zprev > 0] (gcn.py:282); w is f_in x f_out."""
        n, ldi = m.shape[0], w.shape[0]
        if not self._rows_ok(f_out, f_in):
            g = torch.mm(m, w.T)
            L.check(L.lib().dg_relu_grad_mul(g.data_ptr(), g.stride(0), zprev.data_ptr(),
                                             zprev.stride(0), n, f_in, L.stream_ptr()))
            return g
        g = torch.empty((n, ldi), dtype=torch.float32, device=self.device)
        L.check(L.lib().dg_dense_rows(m.data_ptr(), m.stride(0), n, f_out, w.data_ptr(),
                                      w.stride(0), f_in, 1, g.data_ptr(), ldi, 0,
                                      zprev.data_ptr(), zprev.stride(0), L.stream_ptr()))
        return g

    def wgrad(self, h, m, f_in, f_out, ld_in, ld_out):
        """y = h^T m as an (ld_in x ld_out) zero-padded matrix (gcn.py:280)."""
        n = h.shape[0]
        # N > 64 (papers-shaped C=172): cuBLAS measured faster (12.6 vs 21 ms)
        if f_out > 64 or ld_out > 16 * ((f_out + 15) // 16):
            return torch.mm(h.T, m)
        lib = L.lib()
        need = int(lib.dg_dense_tn_work(n, ld_in, f_out))
        if self.work.numel() < need:
            self.work = torch.empty(need, dtype=torch.float64, device=self.device)
        y = torch.empty((ld_in, ld_out), dtype=torch.float32, device=self.device)
        L.check(lib.dg_dense_tn(h.data_ptr(), h.stride(0), n, ld_in, m.data_ptr(), m.stride(0),
                                f_out, y.data_ptr(), ld_out, self.work.data_ptr(),
                                self.work.numel(), L.stream_ptr()))
        return y


class PhaseTimer:
    """Optional CUDA-event marks between the steps of an epoch (bench
    breakdown).  `mark(name)` records an event on the current stream; the
    time attributed to `name` is the gap since the previous mark."""

    def __init__(self):
        self.events = []

    def mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.append((name, e))

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for (_, e0), (name, e1) in zip(self.events[:-1], self.events[1:]):
            out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
        return out


class GcnRun:
    """Device state of one training run (shared by every hosted rank).

    Split from `train` so the benchmark can time epochs of a prepared run
    (setup -- partition, plans, uploads -- happens once, as in the
    reference where it precedes the epoch loop)."""

    def __init__(self, a_hat: CsrMatrix, features, labels, train_mask, cfg: TrainConfig, p=1,
                 c=1, partition=None, row_order=None, fuse=True):
        validate_variant_grid(cfg.variant, p, c)
        from .dist import world
        world().init()
        labels, mask = _check_train_inputs(features, labels, train_mask)
        if a_hat.n_rows != features.shape[0]:
            raise ValueError("feature rows must match the matrix")
        f_out = cfg.f_out if cfg.f_out is not None else int(labels.max()) + 1
        sel = labels[mask]
        if sel.min() < 0 or sel.max() >= f_out:
            raise ValueError(f"labels must lie in [0, {f_out}) on masked rows")
        self.cfg = cfg
        self.grid = grid = ProcessGrid(p, c)
        part = partition if partition is not None else block_partition(a_hat.n_rows,
                                                                         grid.n_rows)
        if part.k != grid.n_rows:
            raise ValueError(f"partition has {part.k} parts but the grid needs {grid.n_rows}")
        self.part = part
        dev = _dev()
        self.device = dev
        is_t = isinstance(features, torch.Tensor)
        a2, feats2 = apply_partition(a_hat, features if is_t else np.asarray(features), part)
        inv = part.inv_perm
        self.dm = build_dist_matrices(a2, part.boundaries, grid)
        self.f_in = int(features.shape[1])
        self.f_out = f_out
        self.denom = int(mask.sum())
        self.dims = cfg.layer_dims(self.f_in, f_out)
        self.lds = [pad4(d) for d in self.dims]
        w0 = init_weights(cfg, self.f_in, f_out)
        self.w0 = []
        for l, w in enumerate(w0):
            wp = torch.zeros((self.lds[l], self.lds[l + 1]), dtype=torch.float32, device=dev)
            wp[:w.shape[0], :w.shape[1]] = torch.from_numpy(w.astype(np.float32))
            self.w0.append(wp)
        self.x = to_device(feats2, self.lds[0])
        lab2 = labels if part.is_identity else labels[inv]
        msk2 = mask if part.is_identity else mask[inv]
        self.labels = torch.from_numpy(lab2.astype(np.int64)).to(dev)
        self.mask = torch.from_numpy(msk2.astype(np.uint8)).to(dev)
        self.xent = {}
        self.dense = {}
        self.fuse = bool(fuse)        # fused SpMM + transform + ReLU where it applies
        self.ctx = {}                 # device state reused across runs (reduction slots)
        self.timer = None             # PhaseTimer for a breakdown run (bench)
        # register the device plans up front (multi-process: fixed IPC
        # buffers sized for the widest layer)
        # row_order (locality.py): processing order of every rank's rows in
        # the SpMM -- "lpa" groups rows by graph community; results unchanged
        from .spmm import device_plan
        for op in {id(self.dm.fwd): self.dm.fwd, id(self.dm.bwd): self.dm.bwd}.values():
            op.row_order = row_order
            device_plan(op, grid, cfg.variant, max_ld=max(self.lds))

    def _fusable(self, l):
        """Layer l's forward transform (+ReLU) runs in the SpMM epilogue
        (DevicePlan.run_fused): aggregate-first order, 1D or c=1, a
        single-pass phase, 13..16-float inputs, <= 64 outputs.
        Same numbers as SpMM -> dense_rows: T is summed identically and
        z = t W accumulates in ascending k in fp32 in both."""
        from .spmm import device_plan
        cfg = self.cfg
        if not getattr(self, "fuse", True) or cfg.order != "aggregate-first":
            return False
        if cfg.reduce_after_transform and self.grid.c > 1:
            return False
        if not cfg.variant.startswith("1d") and self.grid.c > 1:
            return False
        if not (13 <= self.dims[l] <= 16 and self.dims[l + 1] <= 64):
            return False
        return device_plan(self.dm.fwd, self.grid, cfg.variant).can_fuse(self.dims[l],
                                                                         self.dims[l + 1])

    def _inputs(self, i):
        """Block row i of the features, labels and mask (device views)."""
        r0, r1 = self.dm.boundaries[i]
        return self.x[r0:r1], self.labels[r0:r1], self.mask[r0:r1]

    def program(self, comm, epochs, stats, weights_out=None):
        """The per-rank epoch loop (gcn.py:258-286)."""
        cfg, dm = self.cfg, self.dm
        i, j = comm.coords
        r0, r1 = dm.boundaries[i]
        h0, yb, mb = self._inputs(i)
        ws = [w.clone() for w in self.w0] if weights_out is None else weights_out
        xent = self.xent.setdefault(comm.rank, _Xent(r1 - r0, self.device))
        dense = self.dense.setdefault(comm.rank, _Dense(self.device))
        if not hasattr(self, "arena"):
            self.arena = {}
        arena = self.arena.setdefault(comm.rank, _Arena(self.device))
        n_i = r1 - r0
        exchange_index_lists(comm, dm.fwd, cfg.variant)
        if dm.bwd is not dm.fwd:
            exchange_index_lists(comm, dm.bwd, cfg.variant)
        col_group = comm.grid.col_group(j)
        last = len(ws) - 1
        lib = L.lib()
        st = L.stream_ptr()
        dims, lds = self.dims, self.lds
        post_reduce = (cfg.reduce_after_transform and cfg.variant.startswith("15d")
                       and comm.grid.c > 1)
        tm = self.timer if comm.rank == min(comm._rt.local) else None
        mark = tm.mark if tm is not None else (lambda name: None)
        with _no_tf32():
            for epoch in range(epochs):
                mark("epoch_start")
                hs, zs = [h0], []
                for l, w in enumerate(ws):
                    if cfg.order == "transform-first" and dims[l + 1] < dims[l]:
                        u, _ = dense.fwd(hs[-1], w, dims[l], dims[l + 1], False)
                        z = spmm_phase(comm, dm.fwd, u, dims[l + 1], cfg.variant)
                        mark(f"fwd_spmm_f{dims[l + 1]}_tf")
                        h = None
                        if l < last:
                            h = torch.empty_like(z)
                            L.check(lib.dg_relu(z.data_ptr(), h.data_ptr(), z.shape[0],
                                                dims[l + 1], lds[l + 1], st))
                    elif post_reduce and dims[l + 1] < dims[l]:
                        parts = spmm_phase(comm, dm.fwd, hs[-1], dims[l], cfg.variant,
                                           reduce=False, reduce_f=dims[l + 1])
                        u, _ = dense.fwd(parts, w, dims[l], dims[l + 1], False)
                        z = row_group_reduce(comm, u, dm, cfg.variant)
                        mark(f"fwd_spmm_f{dims[l]}_postreduce")
                        h = None
                        if l < last:
                            h = torch.empty_like(z)
                            L.check(lib.dg_relu(z.data_ptr(), h.data_ptr(), z.shape[0],
                                                dims[l + 1], lds[l + 1], st))
                    elif self._fusable(l):
                        # fused forward epilogue: T = A H stays in registers
                        z = (arena.get("l", n_i, lds[l + 1]) if l == last else
                             torch.empty((n_i, lds[l + 1]), dtype=torch.float32,
                                         device=self.device))
                        h = torch.empty_like(z) if l < last else None
                        spmm_phase(comm, dm.fwd, hs[-1], dims[l], cfg.variant,
                                   fuse=(w, dims[l + 1], z, h))
                        mark(f"fwd_spmm_f{dims[l]}_fused")
                    else:
                        t = spmm_phase(comm, dm.fwd, hs[-1], dims[l], cfg.variant,
                                       out=arena.get("t", n_i, lds[l]))
                        mark(f"fwd_spmm_f{dims[l]}")
                        z, h = dense.fwd(t, w, dims[l], dims[l + 1], l < last,
                                         z=arena.get("l", n_i, lds[l + 1]) if l == last else None)
                    zs.append(z)
                    hs.append(h if l < last else z)
                    mark(f"fwd_dense_{l}")
                logits = hs[-1]
                t = u = parts = z = h = None      # only hs / zs stay alive (HBM at scale)
                g = arena.get("g", logits.shape[0], logits.shape[1])
                xent(logits, dims[-1], yb, mb, self.denom, g, stats[epoch])
                mark("xent")
                hs[-1] = zs[-1] = logits = None       # not needed by the backward pass
                for l in range(last, -1, -1):
                    m = spmm_phase(comm, dm.bwd, g, dims[l + 1], cfg.variant,
                                   out=arena.get("l", n_i, lds[l + 1]))   # logits are dead
                    mark(f"bwd_spmm_f{dims[l + 1]}")
                    y = comm.all_reduce_sum(dense.wgrad(hs[l], m, dims[l], dims[l + 1], lds[l],
                                                        lds[l + 1]),
                                            group=col_group, elems=dims[l] * dims[l + 1])
                    mark(f"bwd_wgrad_{l}")
                    if l > 0:
                        g = dense.bwd(m, ws[l], dims[l], dims[l + 1], zs[l - 1])
                    L.check(lib.dg_sgd(ws[l].data_ptr(), y.data_ptr(), ws[l].numel(),
                                       float(cfg.lr), st))
                    mark(f"bwd_dense_{l}")
                comm.ledger_mark(("epoch", epoch))
        return {"stats": stats, "weights": ws}

    def run(self, epochs=None, gather=True):
        """`epochs` training epochs.  gather=False (multi-process): skip the
        end-of-run host gather of every rank's results; pair with
        `global_stats` to read the loss (a device-side sum over all ranks)."""
        epochs = self.cfg.epochs if epochs is None else epochs
        p = self.grid.p
        from .dist import world
        w = world()
        hosted = w.local_ranks(p) if w.multi else range(p)
        stats = {r: torch.zeros((max(epochs, 1), 2), dtype=torch.float64, device=self.device)
                 for r in hosted}
        return run_program(p, self.grid.c,
                           lambda comm: self.program(comm, epochs, stats[comm.rank]),
                           ctx=self.ctx, gather=gather)

    def run_lockstep(self, epochs=None, gather=True, weights_out=None, stats_out=None):
        """`run` with this process's ranks driven by one host thread in lock
        step instead of one thread per rank: each multiply phase is one
        batched device call for all hosted ranks and the collectives need no
        host rendezvous (the thread-per-rank runtime costs ~60 us per
        collective and a GIL hand-off per launch at 4 hosted ranks).  Same
        kernels, same order per rank, same ledger (the reference's
        conventions); aggregate-first order only.  Results equal `run` bit
        for bit (tests/test_gpu_api.py)."""
        from .dist import world
        from .engine import GroupReducer, reduce_members
        from .plan import index_setup_charges
        from .runtime import CommLedger, RunResult, _to_host
        from .spmm import device_plan
        epochs = self.cfg.epochs if epochs is None else epochs
        cfg, dm, grid = self.cfg, self.dm, self.grid
        if cfg.order != "aggregate-first" or cfg.reduce_after_transform:
            raise ValueError("run_lockstep: aggregate-first order only")
        w = world()
        p = grid.p
        ranks = w.local_ranks(p) if w.multi else list(range(p))
        ledger = CommLedger(p, hosted=ranks if w.multi else None)
        index_setup_charges(ledger, dm.fwd, grid, cfg.variant)
        if dm.bwd is not dm.fwd:
            index_setup_charges(ledger, dm.bwd, grid, cfg.variant)
        dims, lds = self.dims, self.lds
        last = len(self.w0) - 1
        lib = L.lib()
        st = L.stream_ptr()
        if not hasattr(self, "arena"):
            self.arena = {}
        blk, n_i, xent, dense, arena, ws, stats = {}, {}, {}, {}, {}, {}, {}
        for r in ranks:
            i, _ = grid.coords(r)
            r0, r1 = dm.boundaries[i]
            blk[r] = self._inputs(i)
            n_i[r] = r1 - r0
            xent[r] = self.xent.setdefault(r, _Xent(r1 - r0, self.device))
            dense[r] = self.dense.setdefault(r, _Dense(self.device))
            arena[r] = self.arena.setdefault(r, _Arena(self.device))
            ws[r] = ([w.clone() for w in self.w0] if weights_out is None else weights_out[r])
            stats[r] = (torch.zeros((max(epochs, 1), 2), dtype=torch.float64, device=self.device)
                        if stats_out is None else stats_out[r])
        fwd = device_plan(dm.fwd, grid, cfg.variant, max_ld=max(lds))
        bwd = device_plan(dm.bwd, grid, cfg.variant, max_ld=max(lds))
        tm = self.timer
        mark = tm.mark if tm is not None else (lambda name: None)
        with _no_tf32():
            for epoch in range(epochs):
                mark("epoch_start")
                hs = {r: [blk[r][0]] for r in ranks}
                zs = {r: [] for r in ranks}
                for l in range(last + 1):
                    if self._fusable(l):                # fused forward epilogue
                        zz = {r: (arena[r].get("l", n_i[r], lds[l + 1]) if l == last else
                                  torch.empty((n_i[r], lds[l + 1]), dtype=torch.float32,
                                              device=self.device)) for r in ranks}
                        hh = ({r: torch.empty_like(zz[r]) for r in ranks} if l < last
                              else None)
                        fwd.run_fused({r: hs[r][-1] for r in ranks}, dims[l], lds[l],
                                      ws[ranks[0]][l], dims[l + 1], lds[l + 1], zz, hh)
                        fwd.vplan.charge(ledger, dims[l])
                        mark(f"fwd_spmm_f{dims[l]}_fused")
                        for r in ranks:
                            zs[r].append(zz[r])
                            hs[r].append(hh[r] if l < last else zz[r])
                        mark(f"fwd_dense_{l}")
                        continue
                    t = fwd.run({r: hs[r][-1] for r in ranks}, dims[l], lds[l],
                                out={r: arena[r].get("t", n_i[r], lds[l]) for r in ranks})
                    fwd.vplan.charge(ledger, dims[l])
                    mark(f"fwd_spmm_f{dims[l]}")
                    for r in ranks:
                        z, h = dense[r].fwd(t[r], ws[r][l], dims[l], dims[l + 1], l < last,
                                            z=(arena[r].get("l", n_i[r], lds[l + 1])
                                               if l == last else None))
                        zs[r].append(z)
                        hs[r].append(h if l < last else z)
                    mark(f"fwd_dense_{l}")
                g = {}
                for r in ranks:
                    logits = hs[r][-1]
                    g[r] = arena[r].get("g", logits.shape[0], logits.shape[1])
                    xent[r](logits, dims[-1], blk[r][1], blk[r][2], self.denom, g[r],
                            stats[r][epoch])
                    hs[r][-1] = zs[r][-1] = None
                mark("xent")
                for l in range(last, -1, -1):
                    m = bwd.run(g, dims[l + 1], lds[l + 1],
                                out={r: arena[r].get("l", n_i[r], lds[l + 1]) for r in ranks})
                    bwd.vplan.charge(ledger, dims[l + 1])
                    mark(f"bwd_spmm_f{dims[l + 1]}")
                    ys = {r: dense[r].wgrad(hs[r][l], m[r], dims[l], dims[l + 1], lds[l],
                                            lds[l + 1]) for r in ranks}
                    y = {}
                    elems = dims[l] * dims[l + 1]
                    if w.multi:                         # peer-memory group reduction
                        numel = ys[ranks[0]].numel()
                        red = self.ctx.get(("reducer", numel))
                        if red is None:
                            red = self.ctx[("reducer", numel)] = GroupReducer(p, numel)
                        groups = {r: grid.col_group(grid.coords(r)[1]) for r in ranks}
                        y = red(ys, groups)
                        for grp in sorted(set(groups.values())):
                            ledger.allreduce(grp, elems)
                    else:
                        for j in range(grid.c):         # all_reduce_sum over each column group
                            grp = grid.col_group(j)
                            for r, o in zip(grp, reduce_members([ys[r] for r in grp])):
                                y[r] = o
                            ledger.allreduce(grp, elems)
                    mark(f"bwd_wgrad_{l}")
                    for r in ranks:
                        if l > 0:
                            g[r] = dense[r].bwd(m[r], ws[r][l], dims[l], dims[l + 1],
                                                zs[r][l - 1])
                        L.check(lib.dg_sgd(ws[r][l].data_ptr(), y[r].data_ptr(),
                                           ws[r][l].numel(), float(cfg.lr), st))
                    mark(f"bwd_dense_{l}")
                ledger.marks[("epoch", epoch)] = ledger.snapshot()
        results = [None] * p
        for r in ranks:
            results[r] = {"stats": stats[r], "weights": ws[r]}
        if w.multi and gather:                          # as run_program does
            torch.cuda.synchronize()
            w.check()
            parts = w.all_gather_object((_to_host({r: results[r] for r in ranks}), ledger))
            for res, _ in parts:
                for r, v in res.items():
                    results[r] = v
            ledger = CommLedger.merged([lg for _, lg in parts])
        return RunResult(results, ledger, grid)

    def global_stats(self, run):
        """(loss sum, correct) per epoch summed over every rank, as a device
        tensor on this process: one device reduction over the row groups'
        first replicas (their rows partition the vertices), no host gather.
        Collective under torchrun."""
        from .dist import world
        w = world()
        grid = self.grid
        firsts = tuple(grid.rank_of(i, 0) for i in range(grid.n_rows))
        if not w.multi:
            tot = run.results[firsts[0]]["stats"].clone()
            for r in firsts[1:]:
                tot += run.results[r]["stats"]
            return tot
        hosted = w.local_ranks(grid.p)
        st = {r: run.results[r]["stats"].float() for r in hosted}
        # members outside the first replicas contribute zeros
        st = {r: (t if r in firsts else torch.zeros_like(t)) for r, t in st.items()}
        numel = next(iter(st.values())).numel()
        key = ("stats_reducer", numel)
        red = self.ctx.get(key)
        if red is None:
            from .engine import GroupReducer
            red = self.ctx[key] = GroupReducer(grid.p, numel)
        out = red(st, {r: tuple(range(grid.p)) for r in hosted})
        return out[hosted[0]].double()

    def run_graph(self, epochs=None):
        """`run` with the epoch captured once in a CUDA graph and replayed
        (launch-bound small graphs, e.g. config 1).  Single
        process (one rank, or several driven in lock step), aggregate-first
        order.  The replayed epochs run exactly the captured kernels on fixed
        buffers (inputs, activation arena, weights updated in place); the
        ledger -- host bookkeeping -- is extended by the captured epoch's
        charges once per replay, so the result equals `run` bit for bit
        (tests/test_gpu_api.py)."""
        import copy
        from .dist import world
        epochs = self.cfg.epochs if epochs is None else epochs
        if world().multi or self.cfg.order != "aggregate-first" or \
                self.cfg.reduce_after_transform:
            raise ValueError("run_graph: single-process, aggregate-first runs only")
        dev = self.device
        p = self.grid.p
        if getattr(self, "_graph", None) is None:
            self._gw = {r: [w.clone() for w in self.w0] for r in range(p)}
            self._gstats = {r: torch.zeros((1, 2), dtype=torch.float64, device=dev)
                            for r in range(p)}
            if p == 1:
                prog = lambda comm: self.program(comm, 1, self._gstats[0],  # noqa: E731
                                                 weights_out=self._gw[0])
                epoch = lambda: run_program(1, 1, prog, ctx=self.ctx)  # noqa: E731
                base = run_program(1, 1, lambda comm: self.program(comm, 0, self._gstats[0]),
                                   ctx=self.ctx).ledger
            else:
                epoch = lambda: self.run_lockstep(1, weights_out=self._gw,  # noqa: E731
                                                  stats_out=self._gstats)
                base = self.run_lockstep(0).ledger          # index setup only
            epoch()                                        # warm-up: plans, arena, workspaces
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream())
            n0 = L.launch_count()
            with torch.cuda.stream(side), torch.cuda.graph(g):
                one = epoch().ledger
            self._graph_launches = L.launch_count() - n0   # our kernels in one epoch
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            self._graph, self._gbase, self._gone = g, base, one
        for r in range(p):
            for w, w0 in zip(self._gw[r], self.w0):
                w.copy_(w0)
        stats = {r: torch.zeros((max(epochs, 1), 2), dtype=torch.float64, device=dev)
                 for r in range(p)}
        for e in range(epochs):
            for r in range(p):
                self._gstats[r].zero_()                   # the loss kernel accumulates
            self._graph.replay()
            for r in range(p):
                stats[r][e].copy_(self._gstats[r][0])
        # ledger: index setup + epochs x the captured epoch's charges
        led = copy.deepcopy(self._gbase)
        base, one = self._gbase, self._gone
        for e in range(epochs):
            for prim, c in one.counters.items():
                for k, arr in c.items():
                    led.counters[prim][k] += arr - base.counters[prim][k]
            led.wire_bytes_sent += one.wire_bytes_sent - base.wire_bytes_sent
            led.marks[("epoch", e)] = led.snapshot()
        led.pair_max_bytes = dict(one.pair_max_bytes)
        led.pair_max_data_bytes = dict(one.pair_max_data_bytes)
        from .runtime import RunResult
        return RunResult([{"stats": stats[r], "weights": [w.clone() for w in self._gw[r]]}
                          for r in range(p)], led, self.grid)

    def close(self):
        """Release the run's device state (collective under torchrun)."""
        for obj in self.ctx.values():
            if hasattr(obj, "close"):
                obj.close()
        self.ctx.clear()
        self.dm.release_device()

    def result(self, run, epochs=None) -> TrainResult:
        epochs = self.cfg.epochs if epochs is None else epochs
        grid = self.grid
        per_epoch = np.zeros((epochs, 2))
        for i in range(grid.n_rows):
            per_epoch += run.results[grid.rank_of(i, 0)]["stats"][:epochs].cpu().numpy()
        history = []
        for epoch in range(epochs):
            row = {"epoch": epoch, "loss": float(per_epoch[epoch, 0] / self.denom),
                   "train_acc": float(per_epoch[epoch, 1] / self.denom)}
            snap = run.ledger.marks.get(("epoch", epoch), {})
            for prim, vals in snap.items():
                row[f"{prim}_bytes"] = vals["bytes_sent"]
            history.append(row)
        wpr = []
        for r in range(grid.p):
            ws = run.results[r]["weights"]
            wpr.append([w[:a, :b].double().cpu().numpy()
                        for w, a, b in zip(ws, self.dims[:-1], self.dims[1:])])
        return TrainResult(history, wpr[0], run.ledger, self.part, wpr)


def train(a_hat: CsrMatrix, features, labels, train_mask, cfg: TrainConfig, p=1, c=1,
          partition=None) -> TrainResult:
    """Train over the selected distributed multiply variant (gcn.py:230-302),
    every rank on the GPU.  cfg.variant == "serial" runs the undistributed
    path (one rank, no ledger)."""
    if cfg.variant == "serial":
        return serial_train(a_hat, features, labels, train_mask, cfg)
    gr = GcnRun(a_hat, features, labels, train_mask, cfg, p, c, partition)
    run = gr.run()
    res = gr.result(run)
    gr.close()
    return res


def serial_train(a_hat: CsrMatrix, features, labels, train_mask, cfg: TrainConfig) -> TrainResult:
    """Full-batch GD on one rank (gcn.py:211-227)."""
    from dataclasses import replace
    c2 = replace(cfg, variant="1d-sparse")
    gr = GcnRun(a_hat, features, labels, train_mask, c2, 1, 1, None)
    res = gr.result(gr.run())
    gr.close()
    for row in res.history:
        for k in [k for k in row if k.endswith("_bytes")]:
            del row[k]
    return TrainResult(res.history, res.weights)
