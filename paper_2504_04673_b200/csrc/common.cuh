// dgb200.cu -- B200 (sm_100a) kernels and C ABI for the sparsity-aware
// distributed SpMM that drives full-graph GCN training.
//
// Reference path (pure NumPy, /root/reference/pkg/src/distgcn):
//   sparse.local_spmm            sparse.py:208-223   -> spmm_rows_kernel (+ chunk fixup)
//   pack h_block[NnzCols(d, me)] spmm.py:185, 212    -> xchg_kernel (gather + peer store)
//   Comm.all_to_allv/isend/bcast runtime.py:311-435  -> xchg_kernel stores into peer halos
//   _scatter                     spmm.py:166-169     -> eliminated (column remap)
//   Comm.all_reduce_sum          runtime.py:437-466  -> group_reduce_kernel
//   gcn._xent_parts              gcn.py:98-120       -> xent_kernel
//   relu / relu_grad / SGD       gcn.py:76-82,276,282-283 -> small elementwise kernels
//
// Design notes (DESIGN.md has the full story):
//  * SpMM is HBM/L2-gather bound (<= f/4 flop/B), not tensor-core work.
//    Each work item (a row, or a fixed chunk of a long row) is handled by a
//    group of G lanes; lane l owns float4 chunks l, l+G, ... of the current
//    feature slab.  (col, val) pairs are loaded coalesced by the group and
//    broadcast with shuffles, so every H-row gather is a G x 16 B request.
//  * Items are bucketed by length on the host (stable, so row order -- and
//    partition locality -- survives inside a bucket): warps see similar
//    trip counts on power-law graphs.
//  * Wide layers are processed in feature slabs sized so one slab of every
//    gathered row fits in L2 (126 MB); grid.y = slab, slab-major launch.
//  * Accumulation in fp64 (default) or fp32, always in CSR storage order;
//    long rows are split at fixed boundaries and their fp64 partials summed
//    in chunk order -> results are deterministic and independent of the
//    variant (aware == oblivious, 1.5D c=1 == 1D, bitwise).

#ifndef DG_COMMON_CUH
#define DG_COMMON_CUH

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <cmath>
#include <vector>

#include "../../include/dgb200.h"

namespace dg {

// thread-local last error and the launch counter live in common.cu
int set_err(int code, const std::string& msg);
void count_launch();

}  // namespace dg

using dg::set_err;

#define DG_CK(call)                                                                   \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess)                                                            \
      return set_err(DG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define DG_LAUNCHED()                                                                  \
  do {                                                                                 \
    dg::count_launch();                                                                \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess)                                                             \
      return set_err(DG_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e));   \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#endif  // DG_COMMON_CUH

