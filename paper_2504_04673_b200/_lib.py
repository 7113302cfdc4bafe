"""ctypes binding of the in-tree C-ABI library `libdgb200.so`.

The library is the product: every compute call of the hot path goes
through it.  There is no CPU fallback -- if the library is missing or no
CUDA device is visible, `lib()` raises instead of silently degrading.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# DG_LIB_PATH: alternative build (tuning experiments only)
LIB_PATH = os.environ.get("DG_LIB_PATH", os.path.join(_HERE, "libdgb200.so"))

DG_MAX_LOCAL = 64
DG_MAX_GROUP = 64
DG_PLAN_SKIP_EMPTY_ROWS = 1
DG_PLAN_DEVICE_SRC = 2

_lock = threading.Lock()
_lib = None

c_i32p = C.POINTER(C.c_int32)
c_i64p = C.POINTER(C.c_int64)
c_f32p = C.POINTER(C.c_float)
c_vp = C.c_void_p
c_vpp = C.POINTER(C.c_void_p)

_SIGS = {
    "dg_last_error": (C.c_char_p, []),
    "dg_version": (C.c_int, []),
    "dg_launch_count": (C.c_int64, []),
    "dg_device_sync": (C.c_int, []),
    "dg_malloc": (C.c_int, [c_vpp, C.c_int64]),
    "dg_free": (C.c_int, [c_vp]),
    "dg_memset0": (C.c_int, [c_vp, C.c_int64, c_vp]),
    "dg_enable_peer": (C.c_int, [C.c_int]),
    "dg_ipc_get_handle": (C.c_int, [c_vp, C.POINTER(C.c_uint8)]),
    "dg_ipc_open_handle": (C.c_int, [C.POINTER(C.c_uint8), c_vpp]),
    "dg_ipc_close": (C.c_int, [c_vp]),
    "dg_spmm_plan_create": (C.c_int, [c_vpp, C.c_int, c_i64p, c_i64p, c_i64p, c_vpp, c_vpp,
                                      c_vpp, C.c_int32, C.c_int32]),
    "dg_spmm_plan_create_ordered": (C.c_int, [c_vpp, C.c_int, c_i64p, c_i64p, c_i64p, c_vpp,
                                              c_vpp, c_vpp, C.c_int32, C.c_int32, c_vpp,
                                              C.c_int64]),
    "dg_spmm_plan_destroy": (C.c_int, [c_vp]),
    "dg_spmm_plan_reserve": (C.c_int, [c_vp, C.c_int64]),
    "dg_spmm_plan_info": (C.c_int, [c_vp, c_i64p]),
    "dg_spmm_run": (C.c_int, [c_vp, c_vpp, c_vpp, c_vpp, C.c_int32, C.c_int64, C.c_int64,
                              C.c_int32, C.c_int32, C.c_int32, c_vp]),
    "dg_spmm_run_fused": (C.c_int, [c_vp, c_vpp, c_vpp, c_vpp, c_vpp, C.c_int32, C.c_int64,
                                    C.c_int64, c_vp, C.c_int64, C.c_int32, c_vp]),
    "dg_xchg_plan_create": (C.c_int, [c_vpp, C.c_int, c_i32p, c_i64p, c_vpp, c_i64p, c_i32p,
                                      c_i64p]),
    "dg_xchg_plan_destroy": (C.c_int, [c_vp]),
    "dg_xchg_run": (C.c_int, [c_vp, c_vpp, C.c_int, c_vpp, C.c_int, C.c_int32, C.c_int64,
                              C.c_int32, c_vp]),
    "dg_xchg_run_ctas": (C.c_int, [c_vp, c_vpp, C.c_int, c_vpp, C.c_int, C.c_int32, C.c_int64,
                                   C.c_int32, C.c_int32, c_vp]),
    "dg_group_reduce": (C.c_int, [C.c_int, c_vpp, C.c_int, c_vpp, C.c_int64, C.c_int64,
                                  C.c_int32, c_vp]),
    "dg_barrier": (C.c_int, [c_vpp, C.c_int, C.c_int, C.c_uint64, C.c_int64, c_vp, c_vp]),
    "dg_xent": (C.c_int, [c_vp, C.c_int64, C.c_int32, C.c_int64, c_vp, c_vp, C.c_double, c_vp,
                          C.c_int64, c_vp, c_vp, c_vp, c_vp]),
    "dg_relu": (C.c_int, [c_vp, c_vp, C.c_int64, C.c_int32, C.c_int64, c_vp]),
    "dg_relu_grad_mul": (C.c_int, [c_vp, C.c_int64, c_vp, C.c_int64, C.c_int64, C.c_int32,
                                   c_vp]),
    "dg_sgd": (C.c_int, [c_vp, c_vp, C.c_int64, C.c_float, c_vp]),
    "dg_dense_rows": (C.c_int, [c_vp, C.c_int64, C.c_int64, C.c_int32, c_vp, C.c_int64, C.c_int32,
                                C.c_int32, c_vp, C.c_int64, c_vp, c_vp, C.c_int64, c_vp]),
    "dg_dense_tn_work": (C.c_int64, [C.c_int64, C.c_int32, C.c_int32]),
    "dg_dense_tn": (C.c_int, [c_vp, C.c_int64, C.c_int64, C.c_int32, c_vp, C.c_int64, C.c_int32,
                              c_vp, C.c_int64, c_vp, C.c_int64, c_vp]),
    "dg_diag_gather_tma": (C.c_int, [c_vp, C.c_int64, C.c_int64, C.c_int32, C.c_int32, c_vp,
                                     C.c_int64, C.c_int32, C.c_int32, c_vp, c_vp]),
    "dg_diag_gather": (C.c_int, [c_vp, C.c_int64, c_vp, C.c_int64, C.c_int32, C.c_int64,
                                 C.c_int32, c_vp, c_vp]),
    "dg_host_permute": (C.c_int, [C.c_int64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dg_host_greedy_tv": (C.c_int, [C.c_int64, c_vp, c_vp, C.c_int32, C.c_double, C.c_int32,
                                    c_vp, c_vp]),
    "dg_host_gvb": (C.c_int, [C.c_int64, c_vp, c_vp, c_vp, c_vp, c_vp, C.c_int32, C.c_double,
                              C.c_double, C.c_int32, c_vp]),
    "dg_host_transpose": (C.c_int, [C.c_int64, C.c_int64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
}

# symbols include/dgb200.h declares (checked by tests/test_cabi.py)
EXPORTED = tuple(_SIGS)


class DgError(RuntimeError):
    pass


def load_library(path=LIB_PATH):
    """Load the shared library and attach signatures (no device needed)."""
    if not os.path.exists(path):
        raise DgError(f"CUDA extension not built: {path} is missing "
                      "(run __graft_entry__.build() or make -C paper_2504_04673_b200/csrc)")
    h = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


_host = None


def host_lib():
    """The library for host-only entry points (no CUDA device required)."""
    global _host
    if _host is None:
        with _lock:
            if _host is None:
                _host = load_library()
    return _host


def lib():
    """The library, loaded once; refuses to run without a CUDA device."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch
                if not torch.cuda.is_available():
                    raise DgError("paper_2504_04673_b200 needs a CUDA device (B200, sm_100a); "
                                  "there is no CPU fallback")
                torch.cuda.init()
                _lib = load_library()
    return _lib


def check(rc):
    if rc != 0:
        msg = lib().dg_last_error().decode(errors="replace")
        raise DgError(f"libdgb200 error {rc}: {msg}")


def ptr_array(ptrs):
    """C array of void* from ints / tensors."""
    vals = [p if isinstance(p, int) else (0 if p is None else p.data_ptr()) for p in ptrs]
    return (C.c_void_p * max(len(vals), 1))(*vals)


def i64_array(vals):
    return (C.c_int64 * max(len(vals), 1))(*[int(v) for v in vals])


def i32_array(vals):
    return (C.c_int32 * max(len(vals), 1))(*[int(v) for v in vals])


def stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def launch_count() -> int:
    return int(lib().dg_launch_count())
