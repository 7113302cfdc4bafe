"""Reference-side binding of the C ABI: what a
maintainer would add to `distgcn/sparse.py` to keep the reference's own
Python -- its simulated ranks, collectives, ledger and training loop -- and
swap only its hot kernel, `local_spmm` (reference sparse.py:208-223), for
the sm_100a SpMM in libdgb200.so.  Device buffers come from any CUDA
allocator (here torch).  tests/test_gpu_integration.py installs it into the
unmodified reference (baseline/_ref) and runs `distgcn.train` on config 1.

    import distgcn, distgcn_binding
    distgcn_binding.install(distgcn)      # sparse / spmm / gcn now call the GPU
"""
import ctypes as C
import os

import numpy as np
import torch

_LIB = os.environ.get("DGB200_LIB", os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2504_04673_b200",
    "libdgb200.so"))
_dg = C.CDLL(_LIB)
_vpp = C.POINTER(C.c_void_p)
_i64p = C.POINTER(C.c_int64)
_dg.dg_spmm_plan_create.argtypes = [_vpp, C.c_int, _i64p, _i64p, _i64p, _vpp, _vpp, _vpp,
                                    C.c_int32, C.c_int32]
_dg.dg_spmm_run.argtypes = [C.c_void_p, _vpp, _vpp, _vpp, C.c_int32, C.c_int64, C.c_int64,
                            C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
_dg.dg_spmm_plan_destroy.argtypes = [C.c_void_p]
_dg.dg_last_error.restype = C.c_char_p


def _ck(rc):
    if rc != 0:
        raise RuntimeError(_dg.dg_last_error().decode())


def local_spmm(a, h):
    """Drop-in for distgcn.sparse.local_spmm (sparse.py:208): same
    arguments and checks, float64 NumPy in and out; the product runs on the
    GPU in fp32 (two-level fp32 / fp64-folded sums, within the 1e-5
    contract)."""
    h = np.asarray(h, dtype=np.float64)
    if h.ndim != 2:
        raise ValueError("dense operand must be 2-D")
    if a.n_cols != h.shape[0]:
        raise ValueError(f"dimension mismatch: {a.shape} @ {h.shape}")
    f = h.shape[1]
    if f == 0 or a.n_rows == 0 or a.nnz == 0:
        return np.zeros((a.n_rows, f))
    ld = (f + 3) // 4 * 4
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(a.col_idx, dtype=np.int32)     # all columns "local"
    val = np.ascontiguousarray(a.values, dtype=np.float32)
    plan = C.c_void_p()

    def arr(v):
        return (C.c_int64 * 1)(v)

    def ptr(x):
        return (C.c_void_p * 1)(x.ctypes.data if isinstance(x, np.ndarray) else x)

    _ck(_dg.dg_spmm_plan_create(C.byref(plan), 1, arr(a.n_rows), arr(a.n_cols), arr(a.nnz),
                                ptr(rp), ptr(col), ptr(val), 1024, 0))
    try:
        hd = torch.zeros((a.n_cols, ld), device="cuda")
        hd[:, :f] = torch.from_numpy(h)
        zd = torch.empty((a.n_rows, ld), device="cuda")
        _ck(_dg.dg_spmm_run(plan, ptr(hd.data_ptr()), ptr(hd.data_ptr()), ptr(zd.data_ptr()),
                            f, ld, ld, 1, 0, 0,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        out = zd[:, :f].double().cpu().numpy()
    finally:
        _dg.dg_spmm_plan_destroy(plan)
    return out


def install(distgcn):
    """Point every module of the reference package that calls local_spmm
    (sparse.py, spmm.py:178/190/226, gcn.py:154/168) at the GPU kernel."""
    for mod in (distgcn, distgcn.sparse, distgcn.spmm, distgcn.gcn):
        if hasattr(mod, "local_spmm"):
            mod.local_spmm = local_spmm
