"""Device engine: per-process state of a variant plan and the calls that
run one distributed multiply phase on the GPU.

One `DevicePlan` covers every rank this process hosts (all p ranks in a
single-process run -- "emulated" ranks sharing one GPU -- or the ranks of
one GPU under torchrun).  A phase is three launches, whatever the number
of hosted ranks:

  1. dg_xchg_run   fused gather of the rows each peer needs (NnzCols lists,
                   or whole blocks for the oblivious forms) stored straight
                   into the receivers' halo buffers (local or peer GPU);
  2. dg_spmm_run   the local SpMM of every hosted rank over
                   [own block | halo] with the remapped CSR;
  3. dg_group_reduce (1.5D only) the row-group sum of the c partial
                   products, reduced once per element in ascending member
                   order so the replicas are bitwise identical.

Buffers: H / Z / halos are torch CUDA tensors (row pitch ld = f rounded up
to 4 floats, zero padding); the sparse operand and exchange lists live in
the C plans.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L

__all__ = ["DevicePlan", "single_spmm", "device_gemm", "reduce_members", "pad4", "to_device",
           "ACC_FP64"]

ACC_FP64 = 1          # accumulate SpMM in fp64 (fp32 inputs / outputs)
MAX_CHUNK = 1024      # nonzeros per work item before a row is split


def pad4(f: int) -> int:
    return (int(f) + 3) // 4 * 4


def to_device(h, ld=None, device=None) -> torch.Tensor:
    """(n, f) array/tensor -> contiguous fp32 CUDA tensor (n, ld), zero padded."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if isinstance(h, torch.Tensor):
        t = h.to(device=dev, dtype=torch.float32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(h, dtype=np.float32))).to(dev)
    if t.dim() != 2:
        raise ValueError("dense operand must be 2-D")
    n, f = t.shape
    ld = pad4(f) if ld is None else ld
    if ld == f and t.is_contiguous():
        return t
    out = torch.zeros((n, ld), dtype=torch.float32, device=dev)
    out[:, :f] = t
    return out


def _stream():
    return L.stream_ptr()


class DevicePlan:
    """Device state of one `plan.VariantPlan` for the locally hosted ranks."""

    def __init__(self, vplan, local_ranks=None, acc=ACC_FP64, max_chunk=MAX_CHUNK):
        lib = L.lib()
        self.vplan = vplan
        self.grid = vplan.grid
        self.local = list(range(vplan.grid.p)) if local_ranks is None else list(local_ranks)
        self.li = {r: k for k, r in enumerate(self.local)}
        self.acc = acc
        self.device = torch.device("cuda", torch.cuda.current_device())
        ro = [vplan.ranks[r] for r in self.local]
        self._keep = ro
        n = len(ro)
        rp = (C.c_void_p * n)(*[x.row_ptr.ctypes.data for x in ro])
        ce = (C.c_void_p * n)(*[x.col_ext.ctypes.data for x in ro])
        va = (C.c_void_p * n)(*[x.val.ctypes.data for x in ro])
        h = C.c_void_p()
        L.check(lib.dg_spmm_plan_create(C.byref(h), n, L.i64_array([x.n_rows for x in ro]),
                                        L.i64_array([x.n_local for x in ro]),
                                        L.i64_array([x.col_ext.size for x in ro]),
                                        rp, ce, va, max_chunk))
        self._splan = h
        segs = [s for s in vplan.segments if s.src in self.li and s.count > 0]
        self._segs = segs
        idx_keep = [s.idx for s in segs]
        xh = C.c_void_p()
        L.check(lib.dg_xchg_plan_create(
            C.byref(xh), len(segs), L.i32_array([self.li[s.src] for s in segs]),
            L.i64_array([s.count for s in segs]),
            (C.c_void_p * max(len(segs), 1))(*[0 if s.idx is None else s.idx.ctypes.data
                                               for s in segs]),
            L.i64_array([0] * len(segs)), L.i32_array([s.dst for s in segs]),
            L.i64_array([s.dst_row0 for s in segs])))
        del idx_keep
        self._xplan = xh
        self.halo = {r: None for r in self.local}
        self.partial = {r: None for r in self.local}
        self.one_d = vplan.variant.startswith("1d")
        info = (C.c_int64 * 8)()
        L.check(lib.dg_spmm_plan_info(self._splan, info))
        self.info = list(info)

    def __del__(self):
        try:
            lib = L.lib()
            if getattr(self, "_splan", None):
                lib.dg_spmm_plan_destroy(self._splan)
            if getattr(self, "_xplan", None):
                lib.dg_xchg_plan_destroy(self._xplan)
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass

    def _buffer(self, store, r, rows, ld):
        need = rows * ld
        buf = store[r]
        if buf is None or buf.numel() < need:
            buf = torch.empty(max(need, 4), dtype=torch.float32, device=self.device)
            store[r] = buf
        return buf[:need].view(rows, ld)

    def run(self, hs: dict, f: int, ld: int, out: dict = None) -> dict:
        """One multiply phase.  hs[r]: (n_i, ld) fp32 CUDA tensor for every
        hosted rank r; returns {r: (n_i, ld) tensor}."""
        lib = L.lib()
        st = _stream()
        vp = self.vplan
        halos = {r: self._buffer(self.halo, r, vp.ranks[r].halo_rows, ld) for r in self.local}
        if self._segs:
            dst = [0] * self.grid.p
            for r in self.local:
                dst[r] = halos[r].data_ptr()
            L.check(lib.dg_xchg_run(self._xplan, L.ptr_array([hs[r] for r in self.local]),
                                    len(self.local), L.ptr_array(dst), len(dst), f, ld, 0, st))
        if out is None:
            out = {r: torch.empty((vp.ranks[r].n_rows, ld), dtype=torch.float32,
                                  device=self.device) for r in self.local}
        if self.one_d or self.grid.c == 1:
            z = out
        else:
            z = {r: self._buffer(self.partial, r, vp.ranks[r].n_rows, ld) for r in self.local}
        L.check(lib.dg_spmm_run(self._splan, L.ptr_array([hs[r] for r in self.local]),
                                L.ptr_array([halos[r] for r in self.local]),
                                L.ptr_array([z[r] for r in self.local]), f, ld, ld, self.acc, 0,
                                st))
        if not self.one_d and self.grid.c > 1:
            for i in range(self.grid.n_rows):
                grp = self.grid.row_group(i)
                if not all(r in self.li for r in grp):
                    raise NotImplementedError("row group split across processes")
                n = vp.ranks[grp[0]].n_rows * ld
                L.check(lib.dg_group_reduce(len(grp), L.ptr_array([z[r] for r in grp]),
                                            L.ptr_array([out[r] for r in grp]), 0, n, 0, st))
        return out


def reduce_members(tensors):
    """Element-wise sum in ascending member order, identical for every
    member (Comm.all_reduce_sum, runtime.py:437-466)."""
    lib = L.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    src = []
    for t in tensors:
        if isinstance(t, torch.Tensor):
            src.append(t.to(device=dev, dtype=torch.float32).contiguous())
        else:
            src.append(torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32)).to(dev))
    outs = [torch.empty_like(src[0]) for _ in src]
    n = src[0].numel()
    L.check(lib.dg_group_reduce(len(src), L.ptr_array(src), L.ptr_array(outs), 0, n, 0,
                                _stream()))
    res = []
    for t, o in zip(tensors, outs):
        res.append(o if isinstance(t, torch.Tensor) else o.double().cpu().numpy())
    return res


def single_spmm(a, h):
    """`local_spmm` on one GPU: one rank whose columns are all local."""
    from .plan import RankOperand
    from .runtime import ProcessGrid
    if getattr(h, "ndim", None) != 2 and not (isinstance(h, torch.Tensor) and h.dim() == 2):
        raise ValueError("dense operand must be 2-D")
    if a.n_cols != h.shape[0]:
        raise ValueError(f"dimension mismatch: {a.shape} @ {tuple(h.shape)}")
    f = int(h.shape[1])
    ld = pad4(max(f, 1))
    numpy_in = not isinstance(h, torch.Tensor)
    if f == 0 or a.n_rows == 0:
        z = np.zeros((a.n_rows, f))
        return z if numpy_in else torch.zeros((a.n_rows, f), device=h.device)
    ro = RankOperand(0, 0, 0, a.n_rows, a.n_cols, a.row_ptr,
                     a.col_idx.astype(np.int32), a.values.astype(np.float32), 0, {})

    class _VP:
        pass
    vp = _VP()
    vp.grid = ProcessGrid(1, 1)
    vp.ranks = [ro]
    vp.segments = []
    vp.variant = "1d-sparse"
    plan = DevicePlan(vp)
    hd = to_device(h, ld)
    z = plan.run({0: hd}, f, ld)[0][:, :f]
    return z.double().cpu().numpy() if numpy_in else z


def device_gemm(a, b):
    """Dense a @ b with the reference's shape checks (sparse.py:226-234);
    cuBLAS fp32 (TF32 disabled)."""
    numpy_in = not isinstance(a, torch.Tensor)
    ta = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a, dtype=np.float64))
    tb = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.asarray(b, dtype=np.float64))
    if ta.dim() != 2 or tb.dim() != 2:
        raise ValueError("gemm operands must be 2-D")
    if ta.shape[1] != tb.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(ta.shape)} @ {tuple(tb.shape)}")
    L.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    with _no_tf32():
        out = ta.to(dev, torch.float32) @ tb.to(dev, torch.float32)
    return out.double().cpu().numpy() if numpy_in else out


class _no_tf32:
    def __enter__(self):
        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False

    def __exit__(self, *exc):
        torch.backends.cuda.matmul.allow_tf32 = self.prev
