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
           "ACC_FP64", "ACC_TWO_LEVEL"]

ACC_FP64 = 1          # fp32 4-entry windows folded into fp64 accumulators
ACC_TWO_LEVEL = 2     # two-level fp32 (<= 64 ulp of sum|terms| per item; rows >= 32 floats)
MAX_CHUNK = 1024      # nonzeros per work item before a row is split
SPMM_WINDOW_NNZ = 0   # entries per length-bucketing window of a plan (0: DG_SPMM_WINDOW_NNZ)
# multi-process phases narrower than this run exchange -> barrier -> one
# SpMM pass instead of overlapping the exchange with an own-block pass and
# adding a halo pass: narrow exchanges are short, and the split costs a
# second pass over nearly every row (products-shaped N=4: every row has halo
# entries) plus a read-modify-write of Z
OVERLAP_MIN_F = 64
# CTAs of an exchange overlapped with the own-block SpMM (all segments).
# The default grid takes every SM before the SpMM starts, serialising the
# two; a capped one (two rows in flight per lane group) moves ~6 GB/s per
# CTA (products rows, 4 GPUs: 319 GB/s at 48 CTAs, 596 at 96).  The cap is
# sized so the exchange ends about when the own-block pass does: both
# scale with the row width, so cap ~ K * rows exchanged / own-block entries
# (Reddit-shaped N=4: ratio 0.024; products-shaped N=4: ~0.057).  K sweep
# at N=4 (f=602 / f=100 phase ms): 1500 -> 4.73 / 1.97, 2500 -> 4.79 /
# 2.18, 4000 -> 4.88 / 2.21 (profiles/r02/xchg_cap/)
OVERLAP_XCHG_K = 1500
OVERLAP_XCHG_MIN_CTAS = 48
# above this the exchange dominates the phase: no cap (the full grid keeps
# the most rows in flight -- papers-shaped sources stream from DRAM)
OVERLAP_XCHG_MAX_CTAS = 296
NARROW_XCHG_CTAS = 296                 # 2 per SM
NARROW_XCHG_L2_BYTES = 64 << 20


def pad4(f: int) -> int:
    """Row pitch (floats) of an f-wide dense operand: 16-byte rows for
    f <= 16; 32-byte rows for f <= 64 (the SpMM's 256-bit loads); 128-byte
    (cache-line) rows for wide layers, so a feature slab of a multiple of 32
    floats maps onto whole L2 lines."""
    f = int(f)
    if f > 64:
        return (f + 31) // 32 * 32
    if f > 16:
        return (f + 7) // 8 * 8
    return (f + 3) // 4 * 4


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


def _ptr(a):
    return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data


def _numel(a):
    return a.numel() if isinstance(a, torch.Tensor) else a.size


def _make_spmm_plan(rank_ops, max_chunk, flags=0, orders=None):
    """dg_spmm_plan over a list of RankOperand-like objects (row_ptr,
    col_ext, val, n_rows, n_local).  col_ext / val may be CUDA tensors (a
    graph built in HBM): the entries are then laid out on the device.
    orders: per operand, None or an int32 permutation of its rows (the
    processing order, locality.py)."""
    lib = L.lib()
    n = len(rank_ops)
    dev = [isinstance(x.col_ext, torch.Tensor) for x in rank_ops]
    if any(dev):
        if not all(dev):
            raise ValueError("mixed host / device operands in one plan")
        flags |= L.DG_PLAN_DEVICE_SRC
        torch.cuda.synchronize()
    rp = (C.c_void_p * n)(*[x.row_ptr.ctypes.data for x in rank_ops])
    ce = (C.c_void_p * n)(*[_ptr(x.col_ext) for x in rank_ops])
    va = (C.c_void_p * n)(*[_ptr(x.val) for x in rank_ops])
    orders = [None] * n if orders is None else list(orders)
    for o, x in zip(orders, rank_ops):
        if o is not None and (o.dtype != np.int32 or o.size != x.n_rows):
            raise ValueError("row order must be an int32 permutation of the rank's rows")
    od = (C.c_void_p * n)(*[0 if o is None else o.ctypes.data for o in orders])
    h = C.c_void_p()
    L.check(lib.dg_spmm_plan_create_ordered(
        C.byref(h), n, L.i64_array([x.n_rows for x in rank_ops]),
        L.i64_array([x.n_local for x in rank_ops]),
        L.i64_array([_numel(x.col_ext) for x in rank_ops]), rp, ce, va, max_chunk, flags,
        od if any(o is not None for o in orders) else None, SPMM_WINDOW_NNZ))
    return h


def _check_bounds(vplan, local):
    """Host-side bounds validation of everything the kernels will index
    (compute-sanitizer is unavailable on the GPU pool): extended columns
    inside [0, n_local + halo_rows), row pointers monotone and covering the
    entries, every exchange segment inside its source block and its
    destination halo."""
    for r in local:
        ro = vplan.ranks[r]
        if _numel(ro.col_ext):
            lo, hi = int(ro.col_ext.min()), int(ro.col_ext.max())
            if lo < 0 or hi >= ro.n_local + ro.halo_rows:
                raise ValueError(f"rank {r}: extended column {lo}..{hi} outside "
                                 f"[0, {ro.n_local + ro.halo_rows})")
        if ro.row_ptr[0] != 0 or ro.row_ptr[-1] != _numel(ro.col_ext) or \
                np.any(np.diff(ro.row_ptr) < 0):
            raise ValueError(f"rank {r}: malformed row pointers")
    widths = getattr(vplan, "widths", None)
    for sg in vplan.segments:
        if sg.dst_row0 < 0 or sg.dst_row0 + sg.count > vplan.ranks[sg.dst].halo_rows:
            raise ValueError(f"segment {sg.src}->{sg.dst} overflows the receiver's halo")
        if sg.src not in local:
            continue                                   # sent by another process
        if sg.idx is not None and _numel(sg.idx) != sg.count:
            raise ValueError(f"segment {sg.src}->{sg.dst}: row list length != count")
        if sg.idx is not None and _numel(sg.idx) and (int(sg.idx.min()) < 0 or
                                                      int(sg.idx.max()) >= widths[sg.q]):
            raise ValueError(f"segment {sg.src}->{sg.dst} indexes outside block {sg.q}")
        if sg.idx is None and sg.count > widths[sg.q]:
            raise ValueError(f"segment {sg.src}->{sg.dst} longer than block {sg.q}")


class _Part:
    """A rank operand restricted to its own-block (interior) or halo
    (boundary) entries, storage order kept."""

    def __init__(self, ro, boundary):
        keep = (ro.col_ext >= ro.n_local) if boundary else (ro.col_ext < ro.n_local)
        self.n_rows, self.n_local = ro.n_rows, ro.n_local
        self.row_ptr = np.zeros(ro.n_rows + 1, dtype=np.int64)
        if isinstance(ro.col_ext, torch.Tensor):       # operand resident in HBM
            lens = torch.from_numpy(np.diff(ro.row_ptr)).to(ro.col_ext.device)
            rows = torch.repeat_interleave(torch.arange(ro.n_rows, device=lens.device), lens)
            cnt = torch.bincount(rows[keep], minlength=ro.n_rows)
            del rows, lens
            self.row_ptr[1:] = torch.cumsum(cnt, 0).cpu().numpy()
            self.col_ext = ro.col_ext[keep].contiguous()
            self.val = ro.val[keep].contiguous()
            return
        rows = np.repeat(np.arange(ro.n_rows, dtype=np.int64), np.diff(ro.row_ptr))[keep]
        if rows.size:
            np.cumsum(np.bincount(rows, minlength=ro.n_rows), out=self.row_ptr[1:])
        self.col_ext = np.ascontiguousarray(ro.col_ext[keep])
        self.val = np.ascontiguousarray(ro.val[keep])


class DevicePlan:
    """Device state of one `plan.VariantPlan` for the ranks this process
    hosts.

    Single process: halo / partial buffers are torch tensors (growable); a
    phase is exchange -> SpMM -> (1.5D) group reduction on one stream.
    Multi-process: buffers are symmetric CUDA-IPC buffers (`dist.SymBuffer`),
    double-buffered by call parity so a phase never overwrites rows a slow
    peer is still reading from the previous phase.  The SpMM is split into
    an own-block (interior) pass that runs on the main stream while the
    exchange + device barrier run on a side stream, and a halo (boundary)
    pass that accumulates into Z once the barrier has passed."""

    def __init__(self, vplan, local_ranks=None, acc=ACC_TWO_LEVEL, max_chunk=MAX_CHUNK,
                 max_ld=None, standalone=False, parities=2, row_order=None):
        from .dist import world
        lib = L.lib()
        self.vplan = vplan
        self.grid = vplan.grid
        self.world = world()
        # standalone: a process-local plan (local_spmm) -- never collective
        self.multi = self.world.multi and not standalone
        self.local = list(range(vplan.grid.p)) if local_ranks is None else list(local_ranks)
        self.li = {r: k for k, r in enumerate(self.local)}
        self.acc = acc
        # halo parities (multi-process): 2 = double-buffered (one device
        # barrier per phase); 1 = single buffer, one more barrier before the
        # exchange overwrites it (halves the halo memory of graphs whose halos
        # fill HBM, e.g. the papers-shaped config)
        if parities not in (1, 2):
            raise ValueError("parities must be 1 or 2")
        self.parities = parities
        self.device = torch.device("cuda", torch.cuda.current_device())
        ro = [vplan.ranks[r] for r in self.local]
        _check_bounds(vplan, self.local)
        # processing order of every hosted rank's rows (locality.py; no
        # effect on any result)
        from .locality import rank_row_order
        self.row_order = row_order
        orders = [rank_row_order(x, row_order, self.device) for x in ro]
        self.overlap = self.multi
        self._fplan = None
        if self.overlap:
            self._splan = _make_spmm_plan([_Part(x, False) for x in ro], max_chunk,
                                          orders=orders)
            self._bplan = _make_spmm_plan([_Part(x, True) for x in ro], max_chunk,
                                          L.DG_PLAN_SKIP_EMPTY_ROWS, orders=orders)
            # single-pass plan for the narrow phases (OVERLAP_MIN_F): a second
            # copy of the entries (papers scale: +6.7 GB per GPU of 180)
            self._fplan = _make_spmm_plan(ro, max_chunk, orders=orders)
            # high priority: the exchange's blocks are dispatched ahead of the
            # own-block SpMM's (otherwise the 10^5-block SpMM grid starves it)
            self._side = torch.cuda.Stream(device=self.device, priority=-1)
        else:
            self._splan = _make_spmm_plan(ro, max_chunk, orders=orders)
            self._bplan = None
        segs = [s for s in vplan.segments if s.src in self.li and s.count > 0]
        # blocks are dispatched roughly in segment order: rotate every
        # sender's destinations by process distance so that at any moment
        # each GPU receives from one sender (no incast on one NVLink ingress)
        w, p = self.world, vplan.grid.p
        segs.sort(key=lambda sg: ((w.proc_of(sg.dst, p) - w.proc_of(sg.src, p)) % w.size,
                                  (sg.dst - sg.src) % p, sg.src))
        self._segs = segs
        self.xchg_ctas = 0                      # 0: no cap
        if self.overlap:
            me = w.proc
            own = sum(int((x.col_ext < x.n_local).sum()) for x in ro)
            out_rows = sum(s.count for s in segs if w.proc_of(s.dst, p) != me)
            in_rows = sum(s.count for s in vplan.segments
                          if s.dst in self.li and w.proc_of(s.src, p) != me)
            if own > 0:
                cap = max(OVERLAP_XCHG_MIN_CTAS,
                          round(OVERLAP_XCHG_K * max(in_rows, out_rows) / own))
                self.xchg_ctas = int(cap) if cap <= OVERLAP_XCHG_MAX_CTAS else 0
        xh = C.c_void_p()
        L.check(lib.dg_xchg_plan_create(
            C.byref(xh), len(segs), L.i32_array([self.li[s.src] for s in segs]),
            L.i64_array([s.count for s in segs]),
            (C.c_void_p * max(len(segs), 1))(*[0 if s.idx is None else _ptr(s.idx)
                                               for s in segs]),
            L.i64_array([0] * len(segs)), L.i32_array([s.dst for s in segs]),
            L.i64_array([s.dst_row0 for s in segs])))
        self._xplan = xh
        self.one_d = vplan.variant.startswith("1d")
        self.reduce = (not self.one_d) and self.grid.c > 1
        self.halo = {r: None for r in self.local}
        self.partial = {r: None for r in self.local}
        self.parity = 0
        if max_ld is not None:                 # split-row buffers: no growth in the hot call
            for h in (self._splan, self._bplan, self._fplan):
                if h:
                    L.check(lib.dg_spmm_plan_reserve(h, int(max_ld)))
        info = (C.c_int64 * 8)()
        L.check(lib.dg_spmm_plan_info(self._splan, info))
        self.info = list(info)
        for x in ro:
            if isinstance(x.col_ext, torch.Tensor):
                # HBM-resident operand: the plans hold their own copy of the
                # entries; keep only the counts (frees ~8 B per nonzero)
                x.nnz = int(x.col_ext.numel())
                occ = torch.zeros(x.n_local + x.halo_rows + 1, dtype=torch.bool,
                                  device=self.device)
                occ[x.col_ext.long()] = True
                x.u = int(occ.sum())
                del occ
                x.col_ext = x.val = None
        if self.multi:
            self._init_symmetric(max_ld)

    # ---- multi-process symmetric buffers --------------------------------
    def _init_symmetric(self, max_ld):
        from .dist import SymBuffer
        if max_ld is None:
            raise ValueError("multi-process plans need max_ld up front (IPC buffers are fixed)")
        self.max_ld = int(max_ld)
        w, p = self.world, self.grid.p
        ranks = self.vplan.ranks
        # per process: its hosted ranks' slots laid out in rank order, two
        # parities each; every process computes every offset identically
        self._hoff, self._poff = {}, {}
        hsize, psize = [0] * w.size, [0] * w.size
        for r in range(p):
            q = w.proc_of(r, p)
            self._hoff[r] = hsize[q]
            hsize[q] += self.parities * ranks[r].halo_rows * self.max_ld * 4
            self._poff[r] = psize[q]
            psize[q] += 2 * ranks[r].n_rows * self.max_ld * 4 if self.reduce else 0
        self.hsym = SymBuffer(w, max(hsize[w.proc], 16))
        self.psym = SymBuffer(w, max(psize[w.proc], 16)) if self.reduce else None

    def _halo_ptr(self, r, par):
        q = self.world.proc_of(r, self.grid.p)
        return (self.hsym.ptrs[q] + self._hoff[r]
                + (par % self.parities) * self.vplan.ranks[r].halo_rows * self.max_ld * 4)

    def _partial_ptr(self, r, par):
        q = self.world.proc_of(r, self.grid.p)
        return (self.psym.ptrs[q] + self._poff[r]
                + par * self.vplan.ranks[r].n_rows * self.max_ld * 4)

    def close(self):
        """Release device state.  Multi-process: collective (every process
        closes the same plans in the same order)."""
        if self.multi:
            for buf in (getattr(self, "hsym", None), getattr(self, "psym", None)):
                if buf is not None:
                    buf.close(self.world)
            self.hsym = self.psym = None
        self._destroy_plans()

    def _destroy_plans(self):
        lib = L.lib()
        for name in ("_splan", "_bplan", "_fplan", "_xplan"):
            h = getattr(self, name, None)
            if h:
                (lib.dg_xchg_plan_destroy if name == "_xplan" else lib.dg_spmm_plan_destroy)(h)
                setattr(self, name, None)

    def __del__(self):
        try:
            self._destroy_plans()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass

    def _buffer(self, store, r, rows, ld):
        need = rows * ld
        buf = store[r]
        if buf is None or buf.numel() < need:
            buf = torch.empty(max(need, 4), dtype=torch.float32, device=self.device)
            store[r] = buf
        return buf[:need].view(rows, ld)

    def _spmm(self, plan, hs, halo_ptrs, zp, f, ld, beta, stream):
        L.check(L.lib().dg_spmm_run(plan, L.ptr_array([hs[r] for r in self.local]),
                                    L.ptr_array(halo_ptrs), L.ptr_array(zp), f, ld, ld, self.acc,
                                    0, beta, stream))

    def _narrow_ctas(self, ld):
        """CTA cap of a narrow (single-pass) exchange: with the hosted H rows
        L2-resident, 2 CTAs per SM beat the flooding grid (products rows at
        f=16: 0.099 -> 0.06 ms); rows streamed from DRAM keep it uncapped."""
        rows = sum(self.vplan.ranks[r].n_rows for r in self.local)
        return NARROW_XCHG_CTAS if rows * ld * 4 <= NARROW_XCHG_L2_BYTES else 0

    def _xchg(self, hs, dst, f, ld, stream, ctas=0):
        if self._segs:
            L.check(L.lib().dg_xchg_run_ctas(self._xplan, L.ptr_array([hs[r] for r in self.local]),
                                             len(self.local), L.ptr_array(dst), len(dst), f, ld,
                                             1 if self.multi else 0, ctas, stream))

    def run(self, hs: dict, f: int, ld: int, out: dict = None, reduce: bool = True) -> dict:
        """One multiply phase.  hs[r]: (n_i, ld) fp32 CUDA tensor for every
        hosted rank r; returns {r: (n_i, ld) tensor}.  1.5D with
        reduce=False returns each replica's partial product (views of the
        plan's partial buffers, valid until the next phase) for a reduction
        after the transform."""
        lib = L.lib()
        st = _stream()
        vp = self.vplan
        p = self.grid.p
        if self.reduce and not reduce:
            out = {}
        elif out is None:
            out = {r: torch.empty((vp.ranks[r].n_rows, ld), dtype=torch.float32,
                                  device=self.device) for r in self.local}
        if not self.multi:
            halos = {r: self._buffer(self.halo, r, vp.ranks[r].halo_rows, ld)
                     for r in self.local}
            dst = [0] * p
            for r in self.local:
                dst[r] = halos[r].data_ptr()
            self._xchg(hs, dst, f, ld, st)
            if self.reduce:
                zp = [self._buffer(self.partial, r, vp.ranks[r].n_rows, ld).data_ptr()
                      for r in self.local]
            else:
                zp = [out[r].data_ptr() for r in self.local]
            self._spmm(self._splan, hs, [halos[r].data_ptr() for r in self.local], zp, f, ld,
                       0, st)
            if self.reduce and not reduce:
                return {r: self._buffer(self.partial, r, vp.ranks[r].n_rows, ld)
                        for r in self.local}
            if self.reduce:
                zl = dict(zip(self.local, zp))
                for i in range(self.grid.n_rows):
                    grp = self.grid.row_group(i)
                    n = vp.ranks[grp[0]].n_rows * ld
                    L.check(lib.dg_group_reduce(len(grp), L.ptr_array([zl[r] for r in grp]),
                                                len(grp), L.ptr_array([out[r] for r in grp]), 0,
                                                n, 0, st))
            return out
        # ---- multi-process: overlap the own-block SpMM with the exchange --
        if ld > self.max_ld:
            raise ValueError(f"row pitch {ld} exceeds the registered maximum {self.max_ld}")
        par = self.parity
        self.parity ^= 1
        dst = [self._halo_ptr(d, par) for d in range(p)]
        halo_ptrs = [self._halo_ptr(r, par) for r in self.local]
        zp = ([self._partial_ptr(r, par) for r in self.local] if self.reduce
              else [out[r].data_ptr() for r in self.local])
        if self._fplan is not None and f < OVERLAP_MIN_F:
            # narrow phase: exchange -> barrier -> one pass over all entries
            if self.parities == 1:
                self.world.barrier()
            self._xchg(hs, dst, f, ld, st, self._narrow_ctas(ld))
            self.world.barrier()                        # every peer's rows have landed
            self._spmm(self._fplan, hs, halo_ptrs, zp, f, ld, 0, st)
        else:
            main = torch.cuda.current_stream()
            self._side.wait_stream(main)                # H is ready
            with torch.cuda.stream(self._side):
                if self.parities == 1:
                    # every peer has finished reading its (single) halo buffer
                    # in the previous phase before anyone overwrites it
                    self.world.barrier()
                self._xchg(hs, dst, f, ld, L.stream_ptr(self._side), self.xchg_ctas)
                self.world.barrier()                    # every peer's rows have landed
            self._spmm(self._splan, hs, halo_ptrs, zp, f, ld, 0, st)   # own block
            main.wait_stream(self._side)
            self._spmm(self._bplan, hs, halo_ptrs, zp, f, ld, 1, st)   # halo rows, z +=
            for r in self.local:                        # inputs in use on the side stream
                hs[r].record_stream(self._side)
        if self.reduce and not reduce:
            from .dist import _as_tensor
            return {r: _as_tensor(self._partial_ptr(r, par), vp.ranks[r].n_rows * ld,
                                  torch.float32).view(vp.ranks[r].n_rows, ld)
                    for r in self.local}
        if self.reduce:
            self.world.barrier()                        # every replica's partial is ready
            spread = [r for r in self.local if self._group_spans_processes(r)]
            for r in self.local:
                if r in spread:
                    continue
                i, _ = self.grid.coords(r)
                grp = self.grid.row_group(i)
                n = vp.ranks[r].n_rows * ld
                L.check(lib.dg_group_reduce(len(grp), L.ptr_array(
                    [self._partial_ptr(m, par) for m in grp]), 1, L.ptr_array([out[r]]), 0,
                    n, 0, st))
            if spread:
                self._reduce_scatter_all_gather(spread, par, ld, out, st)
        return out

    def _group_spans_processes(self, r):
        grp = self.grid.row_group(self.grid.coords(r)[0])
        return len({self.world.proc_of(m, self.grid.p) for m in grp}) > 1

    def _reduce_scatter_all_gather(self, ranks, par, ld, out, st):
        """Row-group sum across processes, bandwidth-optimal (reference
        spmm.py:227, runtime.py:437-466): member k of a c-member group sums
        chunk k of the n x ld partials -- reading (c-1)/c of the data from
        its peers -- and stores the sum into chunk k of EVERY member's
        partial buffer (peer stores); after one device barrier each member
        copies the whole sum out of its own buffer.  2 (c-1)/c n bytes cross
        NVLink per member instead of (c-1) n for read-all-partials; every
        element is reduced once, in ascending member order, so the replicas
        stay bitwise identical."""
        lib = L.lib()
        vp = self.vplan
        for r in ranks:
            i, _ = self.grid.coords(r)
            grp = self.grid.row_group(i)
            c = len(grp)
            k = grp.index(r)
            n = vp.ranks[r].n_rows * ld
            lo, hi = (n * k // c) // 4 * 4, (n * (k + 1) // c) // 4 * 4 if k + 1 < c else n
            ptrs = L.ptr_array([self._partial_ptr(m, par) for m in grp])
            L.check(lib.dg_group_reduce(c, ptrs, c, ptrs, lo, hi, 1, st))
        self.world.barrier()                            # every chunk landed everywhere
        for r in ranks:
            n = vp.ranks[r].n_rows * ld
            L.check(lib.dg_group_reduce(1, L.ptr_array([self._partial_ptr(r, par)]), 1,
                                        L.ptr_array([out[r]]), 0, n, 0, st))

    def can_fuse(self, f, n_out):
        """Whether `run_fused` applies: a single-pass phase (one process, or
        a narrow multi-process phase on the single-pass plan), no 1.5D
        partials, 13..16-float rows, n_out <= 64."""
        single = (not self.multi) or (self._fplan is not None and int(f) < OVERLAP_MIN_F)
        return single and (not self.reduce) and 13 <= int(f) <= 16 and int(n_out) <= 64

    def run_fused(self, hs: dict, f: int, ld: int, w, n_out: int, ld_out: int, z: dict,
                  h: dict = None):
        """One multiply phase with the forward transform fused into the SpMM
        epilogue (gcn.py:273-276): z[r] = (A_r [H_r; halo]) W, h[r] = relu(z[r])
        -- T never reaches HBM.  `w` (f x n_out, padded pitch) is the layer's
        weight, identical on every rank (replicated, gcn.py:263)."""
        if not self.can_fuse(f, n_out):
            raise ValueError("run_fused: needs a single-pass 1D plan and 13 <= f <= 16, "
                             "n_out <= 64")
        lib = L.lib()
        st = _stream()
        vp = self.vplan
        if self.multi:                                  # IPC halos, as in run()
            if ld > self.max_ld:
                raise ValueError(f"row pitch {ld} exceeds the registered maximum {self.max_ld}")
            par = self.parity
            self.parity ^= 1
            dst = [self._halo_ptr(d, par) for d in range(self.grid.p)]
            halo_ptrs = [self._halo_ptr(r, par) for r in self.local]
            if self.parities == 1:
                self.world.barrier()
            self._xchg(hs, dst, f, ld, st, self._narrow_ctas(ld))
            self.world.barrier()                        # every peer's rows have landed
            plan = self._fplan
        else:
            halos = {r: self._buffer(self.halo, r, vp.ranks[r].halo_rows, ld)
                     for r in self.local}
            dst = [0] * self.grid.p
            for r in self.local:
                dst[r] = halos[r].data_ptr()
            halo_ptrs = [halos[r].data_ptr() for r in self.local]
            self._xchg(hs, dst, f, ld, st)
            plan = self._splan
        L.check(lib.dg_spmm_run_fused(
            plan, L.ptr_array([hs[r] for r in self.local]),
            L.ptr_array(halo_ptrs), L.ptr_array([z[r] for r in self.local]),
            L.ptr_array([h[r] for r in self.local]) if h is not None else None, f, ld, ld_out,
            C.c_void_p(w.data_ptr()), w.stride(0), n_out, st))
        return z

    # ---- pieces of a phase, for per-kernel timing in bench.py ------------
    def exchange_only(self, hs: dict, f: int, ld: int):
        """The halo exchange of one phase (+ the device barrier that makes
        the rows visible), without the SpMM."""
        p = self.grid.p
        if self.multi:
            par = self.parity
            dst = [self._halo_ptr(d, par) for d in range(p)]
        else:
            dst = [0] * p
            for r in self.local:
                dst[r] = self._buffer(self.halo, r, self.vplan.ranks[r].halo_rows,
                                      ld).data_ptr()
        self._xchg(hs, dst, f, ld, _stream())
        if self.multi:
            self.world.barrier()

    def spmm_only(self, hs: dict, f: int, ld: int, out: dict):
        """The local SpMM of one phase (own block + halo) over the current
        halo contents, no exchange."""
        if self.multi:
            halo_ptrs = [self._halo_ptr(r, self.parity) for r in self.local]
        else:
            halo_ptrs = [self._buffer(self.halo, r, self.vplan.ranks[r].halo_rows,
                                      ld).data_ptr() for r in self.local]
        zp = [out[r].data_ptr() for r in self.local]
        if self.multi and self._fplan is not None and f < OVERLAP_MIN_F:
            self._spmm(self._fplan, hs, halo_ptrs, zp, f, ld, 0, _stream())   # as run()
            return
        self._spmm(self._splan, hs, halo_ptrs, zp, f, ld, 0, _stream())
        if self._bplan is not None:
            self._spmm(self._bplan, hs, halo_ptrs, zp, f, ld, 1, _stream())

    def traffic_rows(self):
        """(rows sent, rows received) per rank in one phase."""
        p = self.grid.p
        snd, rcv = [0] * p, [0] * p
        for sg in self.vplan.segments:
            snd[sg.src] += sg.count
            rcv[sg.dst] += sg.count
        return snd, rcv


class GroupReducer:
    """Cross-process `all_reduce_sum` for small tensors (the GCN weight
    gradients): every hosted rank copies its buffer into a symmetric slot,
    one device barrier, then each rank sums its group's slots (ascending
    member order, peer-mapped reads) -- bit-identical on every member."""

    def __init__(self, p, numel):
        from .dist import SymBuffer, world
        self.w = world()
        self.p = p
        self.numel = int(numel)
        self.slot = (self.numel * 4 + 255) // 256 * 256
        counts = [0] * self.w.size
        self.idx = {}
        for r in range(p):
            q = self.w.proc_of(r, p)
            self.idx[r] = counts[q]
            counts[q] += 1
        self.sym = SymBuffer(self.w, max(2 * counts[self.w.proc] * self.slot, 16))
        self.parity = 0

    def close(self):
        """Collective release of the symmetric slots."""
        if self.sym is not None:
            self.sym.close(self.w)
            self.sym = None

    def _ptr(self, r, par):
        q = self.w.proc_of(r, self.p)
        per_par = sum(1 for x in range(self.p) if self.w.proc_of(x, self.p) == q) * self.slot
        return self.sym.ptrs[q] + par * per_par + self.idx[r] * self.slot

    def __call__(self, bufs: dict, groups: dict) -> dict:
        from .dist import _as_tensor
        lib = L.lib()
        par = self.parity
        self.parity ^= 1
        for r, b in bufs.items():
            _as_tensor(self._ptr(r, par), self.numel, torch.float32).copy_(b.reshape(-1))
        self.w.barrier()
        out = {}
        for r, b in bufs.items():
            grp = groups[r]
            o = torch.empty_like(b)
            L.check(lib.dg_group_reduce(len(grp), L.ptr_array([self._ptr(m, par) for m in grp]),
                                        1, L.ptr_array([o]), 0, self.numel, 0, _stream()))
            out[r] = o
        return out


class RowGroupReducer:
    """Row-group sum of per-replica (n_i x ld) tensors, bit-identical on
    every replica (ascending member order).  Multi-process: symmetric slots
    sized for the largest block row, two parities, one device barrier."""

    def __init__(self, grid, vplan, ld):
        from .dist import SymBuffer, world
        self.grid, self.w, self.ld = grid, world(), int(ld)
        self.rows = {r: vplan.ranks[r].n_rows for r in range(grid.p)}
        self.sym = None
        if self.w.multi:
            p = grid.p
            self.slot = max(self.rows.values()) * self.ld * 4
            self.idx, counts = {}, [0] * self.w.size
            for r in range(p):
                q = self.w.proc_of(r, p)
                self.idx[r] = counts[q]
                counts[q] += 1
            self.per_par = {q: counts[q] * self.slot for q in range(self.w.size)}
            self.sym = SymBuffer(self.w, max(2 * counts[self.w.proc] * self.slot, 16))
        self.parity = 0

    def close(self):
        if self.sym is not None:
            self.sym.close(self.w)
            self.sym = None

    def _ptr(self, r, par):
        q = self.w.proc_of(r, self.grid.p)
        return self.sym.ptrs[q] + par * self.per_par[q] + self.idx[r] * self.slot

    def __call__(self, parts: dict) -> dict:
        lib = L.lib()
        out = {r: torch.empty_like(t) for r, t in parts.items()}
        if not self.w.multi:
            for i in range(self.grid.n_rows):
                grp = self.grid.row_group(i)
                if not all(r in parts for r in grp):
                    continue
                n = parts[grp[0]].numel()
                L.check(lib.dg_group_reduce(len(grp), L.ptr_array([parts[r] for r in grp]),
                                            len(grp), L.ptr_array([out[r] for r in grp]), 0, n,
                                            0, _stream()))
            return out
        from .dist import _as_tensor
        par = self.parity
        self.parity ^= 1
        for r, t in parts.items():
            _as_tensor(self._ptr(r, par), t.numel(), torch.float32).copy_(t.reshape(-1))
        self.w.barrier()
        for r, t in parts.items():
            grp = self.grid.row_group(self.grid.coords(r)[0])
            L.check(lib.dg_group_reduce(len(grp), L.ptr_array([self._ptr(m, par) for m in grp]),
                                        1, L.ptr_array([out[r]]), 0, t.numel(), 0, _stream()))
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
    L.check(lib.dg_group_reduce(len(src), L.ptr_array(src), len(outs), L.ptr_array(outs), 0, n,
                                0, _stream()))
    res = []
    for t, o in zip(tensors, outs):
        res.append(o if isinstance(t, torch.Tensor) else o.double().cpu().numpy())
    return res


class _LocalPlan:
    """A one-rank VariantPlan whose columns are all local (local_spmm)."""

    def __init__(self, ro):
        from .runtime import ProcessGrid
        self.grid = ProcessGrid(1, 1)
        self.ranks = [ro]
        self.segments = []
        self.widths = [ro.n_local]
        self.variant = "1d-sparse"


def single_spmm(a, h):
    """`local_spmm` on one GPU: one rank whose columns are all local; a
    process-local plan (no collective, also under torchrun)."""
    from .plan import RankOperand
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
    plan = DevicePlan(_LocalPlan(ro), standalone=True)
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
