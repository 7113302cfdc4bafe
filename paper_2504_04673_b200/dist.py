"""Multi-process (one process per GPU) plumbing: who hosts which rank,
symmetric device buffers shared through CUDA IPC, and the device barrier.

Launched with torchrun (RANK / WORLD_SIZE / LOCAL_RANK in the env), every
process runs the same program (SPMD, like the reference's rank programs,
runtime.py:498-538) and builds the same deterministic host plan.  Process
q hosts the virtual ranks with `proc_of(rank) == q` (a block map, so the c
replicas of a row group share a GPU whenever p/N >= c).

Data moves only through device memory: each process allocates its halo /
partial / reduction buffers with cudaMalloc, exports CUDA-IPC handles, and
every process maps every peer's buffers.  A pack kernel then stores rows
straight into the peer's halo over NVLink; `barrier()` is a device kernel
over IPC-mapped flag words (bounded spin, no host round trip).  The host
side only exchanges the 64-byte IPC handles (gloo) once per buffer.

Co-located processes (more processes than GPUs, e.g. the driver's 1-GPU
test box running 2 or 4 processes on cuda:0) never run the device barrier:
two kernels that spin on each other's flags from different contexts on one
GPU have no co-scheduling guarantee (time-sliced contexts; on B200 such
pairs raised Xid 109).  There `barrier()` is host-side instead -- finish
this process's work on the current stream, then a gloo barrier -- and every
other piece of the multi-process data path (IPC-mapped halos, peer stores,
parity double-buffering, split own/halo SpMM, the cross-process reducers)
runs unchanged.  `DG_BARRIER=device|host` overrides the choice.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib as L

__all__ = ["World", "world", "SymBuffer"]

BARRIER_TIMEOUT_NS = 60 * 10**9


class World:
    """Process group facts (single process: size 1, proc 0)."""

    def __init__(self):
        self.size = int(os.environ.get("WORLD_SIZE", "1"))
        self.proc = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", str(self.proc)))
        self._pg = None
        self._flags = None
        self._epoch = 0
        self._err = None
        self.device = None
        self.barrier_mode = "device"

    @property
    def multi(self) -> bool:
        return self.size > 1

    def init(self):
        """Bring up torch.distributed (gloo: host handle exchange only) and
        the device barrier flags.  Idempotent."""
        if self.device is not None:
            return self
        if not torch.cuda.is_available():
            # host-only use (the generic Comm primitives over gloo, CPU tests):
            # no device buffers, host barriers
            self.device = torch.device("cpu")
            self.barrier_mode = "host"
            if self.multi:
                self._init_pg()
            return self
        if self.multi:
            torch.cuda.set_device(self.local % max(torch.cuda.device_count(), 1))
        self.device = torch.device("cuda", torch.cuda.current_device())
        if not self.multi:
            return self
        self._init_pg()
        lib = L.lib()
        for d in range(torch.cuda.device_count()):
            if d != torch.cuda.current_device():
                try:
                    L.check(lib.dg_enable_peer(d))
                except L.DgError:
                    pass
        self._flags = SymBuffer(self, 8 * self.size)
        self._err = torch.zeros(1, dtype=torch.int32, device=self.device)
        uuid = str(torch.cuda.get_device_properties(self.device).uuid)
        colocated = len(set(self.all_gather_object(uuid))) < self.size
        mode = os.environ.get("DG_BARRIER", "host" if colocated else "device")
        if mode not in ("device", "host"):
            raise ValueError(f"DG_BARRIER must be 'device' or 'host', got {mode!r}")
        if mode == "device" and colocated:
            raise ValueError("DG_BARRIER=device with several processes on one GPU: spinning "
                             "kernels in different contexts are not co-scheduled")
        self.barrier_mode = mode
        return self

    def _init_pg(self):
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.proc, world_size=self.size)
        self._pg = dist.group.WORLD

    def all_gather_object(self, obj):
        if not self.multi:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.size
        dist.all_gather_object(out, obj, group=self._pg)
        return out

    def host_barrier(self):
        if self.multi:
            import torch.distributed as dist
            dist.barrier(group=self._pg)

    def barrier(self):
        """Barrier of all processes, ordered on the current stream: a device
        kernel over the IPC flag words, or (co-located processes) a stream
        synchronize followed by a host barrier."""
        if not self.multi:
            return
        if self.barrier_mode == "host":
            if self.device.type == "cuda":
                torch.cuda.current_stream().synchronize()
            self.host_barrier()
            return
        self._epoch += 1
        ptrs = (C.c_void_p * self.size)(*self._flags.ptrs)
        L.check(L.lib().dg_barrier(ptrs, self.size, self.proc, self._epoch, BARRIER_TIMEOUT_NS,
                                   self._err.data_ptr(), L.stream_ptr()))

    def check(self):
        """Raise if a device barrier timed out (call at sync points)."""
        if self.multi and self._err is not None and int(self._err.item()) != 0:
            raise RuntimeError("device barrier timed out: a peer process stalled")

    @property
    def rank_map(self):
        """How virtual ranks map onto processes (DG_RANK_MAP): "block"
        (default; rank r on process floor(r N / p), so the c replicas of a
        row group share a GPU when p/N >= c and the row-group reduction runs
        in HBM) or "cyclic" (rank r on process r mod N: replicas on
        different GPUs, the reduction crosses NVLink as a reduce-scatter +
        all-gather; column-group peers share GPUs instead)."""
        m = os.environ.get("DG_RANK_MAP", "block")
        if m not in ("block", "cyclic"):
            raise ValueError(f"DG_RANK_MAP must be 'block' or 'cyclic', got {m!r}")
        return m

    def proc_of(self, rank, p):
        """The process hosting virtual rank `rank` of p (see rank_map)."""
        if self.rank_map == "cyclic":
            return rank % self.size
        return (rank * self.size) // p

    def local_ranks(self, p):
        return [r for r in range(p) if self.proc_of(r, p) == self.proc]


class SymBuffer:
    """A zero-filled device buffer of `nbytes` on every process; `ptrs[q]`
    is process q's buffer as mapped into this process (own: local pointer;
    peers: CUDA-IPC mapped).  Collective: every process must construct it."""

    def __init__(self, world: "World", nbytes: int):
        lib = L.lib()
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        L.check(lib.dg_malloc(C.byref(p), self.nbytes))
        self.local = p.value
        self.ptrs = [self.local]
        if world.multi:
            h = (C.c_uint8 * 64)()
            L.check(lib.dg_ipc_get_handle(C.c_void_p(self.local), h))
            handles = world.all_gather_object(bytes(h))
            self.ptrs = []
            for q, hb in enumerate(handles):
                if q == world.proc:
                    self.ptrs.append(self.local)
                else:
                    out = C.c_void_p()
                    L.check(lib.dg_ipc_open_handle((C.c_uint8 * 64)(*hb), C.byref(out)))
                    self.ptrs.append(out.value)

    def close(self, world: "World"):
        """Collective release: unmap the peers' buffers, wait until every
        process has done the same, then free the local buffer (a peer must
        never touch freed memory)."""
        if self.local is None:
            return
        lib = L.lib()
        if world.multi:
            torch.cuda.synchronize()
            for q, ptr in enumerate(self.ptrs):
                if q != world.proc:
                    L.check(lib.dg_ipc_close(C.c_void_p(ptr)))
            world.host_barrier()
        L.check(lib.dg_free(C.c_void_p(self.local)))
        self.local, self.ptrs = None, []

    def tensor(self, numel, dtype=torch.float32, offset_bytes=0):
        """The local buffer as a torch tensor view (no copy)."""
        return _as_tensor(self.local + offset_bytes, numel, dtype)


def _as_tensor(ptr, numel, dtype):
    """Wrap raw device memory as a torch tensor via __cuda_array_interface__."""
    typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4",
               torch.int64: "<i8"}[dtype]

    class _Arr:
        __cuda_array_interface__ = {"shape": (int(numel),), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3, "strides": None}
    return torch.as_tensor(_Arr(), device="cuda")


_WORLD = None


def world() -> World:
    global _WORLD
    if _WORLD is None:
        _WORLD = World()
    return _WORLD
