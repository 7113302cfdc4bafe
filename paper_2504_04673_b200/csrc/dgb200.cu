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

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dgb200.h"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DG_CK(call)                                                                   \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess)                                                            \
      return set_err(DG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define DG_LAUNCHED()                                                                  \
  do {                                                                                 \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess)                                                             \
      return set_err(DG_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e));   \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// SpMM
// ---------------------------------------------------------------------------

struct Item {          // 24 B: one row, or one fixed chunk of a long row
  int64_t lo;          // first nonzero (rank-local CSR offset)
  int32_t row;         // output row
  int32_t len;         // nonzeros in this item
  int32_t rank;        // local rank index
  int32_t slot;        // -1: write z directly; else fp64 partial slot
};

struct Fixup {         // a split row: partial slots [slot0, slot0 + n)
  int32_t row;
  int32_t rank;
  int32_t slot0;
  int32_t n;
};

struct RankArgs {
  const int32_t* col;
  const float* val;
  const float* hl;     // own H block (ext < n_local)
  const float* hh;     // halo rows (ext >= n_local)
  float* z;
  int64_t n_local;
};

struct SpmmArgs {
  RankArgs r[DG_MAX_LOCAL];
  const Item* items;
  double* part;
  int64_t n_items;
  int64_t ld_h;
  int64_t ld_z;
  int64_t ld_part;
  int32_t chunks;      // ceil(f / 4): float4 chunks that carry features
  int32_t slab;        // chunks per slab (= G * CPL)
};

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31;
    return ((1u << G) - 1u) << (lane & ~(G - 1));
  }
}

template <typename Acc>
__device__ __forceinline__ void fma4(Acc* a, float v, const float4 x) {
  a[0] += (Acc)v * (Acc)x.x;
  a[1] += (Acc)v * (Acc)x.y;
  a[2] += (Acc)v * (Acc)x.z;
  a[3] += (Acc)v * (Acc)x.w;
}

template <int G, int CPL, typename Acc>
__global__ void __launch_bounds__(256) spmm_rows_kernel(const __grid_constant__ SpmmArgs a) {
  const int lig = threadIdx.x & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if (gid >= a.n_items) return;                     // whole group leaves together
  const unsigned gm = group_mask<G>();
  const Item it = a.items[gid];
  const RankArgs& R = a.r[it.rank];
  const int slab0 = blockIdx.y * a.slab;
  const int64_t ld = a.ld_h;
  const int32_t* __restrict__ cp = R.col + it.lo;
  const float* __restrict__ vp = R.val + it.lo;
  const float* __restrict__ hl = R.hl;
  const float* __restrict__ hh = R.hh;
  const int64_t nl = R.n_local;

  int chk[CPL];
  bool on[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    chk[q] = slab0 + lig + q * G;
    on[q] = chk[q] < a.chunks && (lig + q * G) < a.slab;
  }
  Acc acc[CPL][4];
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[q][k] = (Acc)0;

  const int len = it.len;
  int e = 0;
  // full batches: G nonzeros, no bounds checks inside
  for (; e + G <= len; e += G) {
    const int c = __ldg(cp + e + lig);
    const float v = __ldg(vp + e + lig);
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int ct = __shfl_sync(gm, c, t, G);
      const float vt = __shfl_sync(gm, v, t, G);
      const float* hp = ct < nl ? hl + (int64_t)ct * ld : hh + (int64_t)(ct - nl) * ld;
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (on[q]) fma4(acc[q], vt, __ldg(reinterpret_cast<const float4*>(hp) + chk[q]));
    }
  }
  if (e < len) {                                    // tail batch (group-uniform)
    const int nb = len - e;
    int c = 0;
    float v = 0.f;
    if (lig < nb) {
      c = __ldg(cp + e + lig);
      v = __ldg(vp + e + lig);
    }
#pragma unroll
    for (int t = 0; t < G; ++t) {
      if (t < nb) {
        const int ct = __shfl_sync(gm, c, t, G);
        const float vt = __shfl_sync(gm, v, t, G);
        const float* hp = ct < nl ? hl + (int64_t)ct * ld : hh + (int64_t)(ct - nl) * ld;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (on[q]) fma4(acc[q], vt, __ldg(reinterpret_cast<const float4*>(hp) + chk[q]));
      }
    }
  }

  if (it.slot < 0) {
    float* zp = R.z + (int64_t)it.row * a.ld_z;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (on[q])
        reinterpret_cast<float4*>(zp)[chk[q]] =
            make_float4((float)acc[q][0], (float)acc[q][1], (float)acc[q][2], (float)acc[q][3]);
  } else {
    double* pp = a.part + (int64_t)it.slot * a.ld_part;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (on[q]) {
        double4 d;
        d.x = (double)acc[q][0];
        d.y = (double)acc[q][1];
        d.z = (double)acc[q][2];
        d.w = (double)acc[q][3];
        reinterpret_cast<double4*>(pp)[chk[q]] = d;
      }
  }
}

struct FixArgs {
  float* z[DG_MAX_LOCAL];
  const Fixup* fix;
  const double* part;
  int64_t ld_z;
  int64_t ld_part;
  int32_t nfloat;      // chunks * 4
};

__global__ void __launch_bounds__(128) spmm_fixup_kernel(const __grid_constant__ FixArgs a) {
  const Fixup fx = a.fix[blockIdx.x];
  float* zp = a.z[fx.rank] + (int64_t)fx.row * a.ld_z;
  for (int c = threadIdx.x; c < a.nfloat; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < fx.n; ++k) s += a.part[(int64_t)(fx.slot0 + k) * a.ld_part + c];
    zp[c] = (float)s;
  }
}

}  // namespace

struct dg_spmm_plan {
  int n_ranks = 0;
  std::vector<int64_t> n_rows, n_local, nnz, ext_rows;
  std::vector<int32_t*> col;
  std::vector<float*> val;
  Item* items = nullptr;
  int64_t n_items = 0;
  Fixup* fix = nullptr;
  int64_t n_fix = 0;
  int64_t n_slots = 0;
  double* part = nullptr;
  int64_t part_cap = 0;  // doubles
  int64_t dev_bytes = 0;
};

namespace {

int32_t bucket_of(int32_t len) {
  int32_t b = 0;
  while ((1 << b) <= len && b < 30) ++b;
  return b;
}

template <int G, int CPL, typename Acc>
void launch_spmm(const SpmmArgs& a, int nslabs, cudaStream_t s) {
  const int64_t threads = a.n_items * G;
  const unsigned gx = (unsigned)((threads + 255) / 256);
  spmm_rows_kernel<G, CPL, Acc><<<dim3(gx, nslabs), 256, 0, s>>>(a);
}

using LaunchFn = void (*)(const SpmmArgs&, int, cudaStream_t);

template <typename Acc>
LaunchFn pick_launch(int G, int CPL) {
#define DG_CASE(g, c) \
  if (G == g && CPL == c) return &launch_spmm<g, c, Acc>;
  DG_CASE(1, 1) DG_CASE(1, 2) DG_CASE(1, 3) DG_CASE(1, 4)
  DG_CASE(2, 1) DG_CASE(2, 2) DG_CASE(2, 3) DG_CASE(2, 4)
  DG_CASE(4, 1) DG_CASE(4, 2) DG_CASE(4, 3) DG_CASE(4, 4)
  DG_CASE(8, 1) DG_CASE(8, 2) DG_CASE(8, 3) DG_CASE(8, 4)
  DG_CASE(16, 1) DG_CASE(16, 2) DG_CASE(16, 3) DG_CASE(16, 4)
  DG_CASE(32, 1) DG_CASE(32, 2) DG_CASE(32, 3) DG_CASE(32, 4)
#undef DG_CASE
  return nullptr;
}

// Choose the lane-group size G and chunks-per-lane CPL for `chunks` float4
// chunks of features when one slab may hold at most `wmax` chunks.
void choose_config(int chunks, int wmax, int* G_out, int* CPL_out, int* nslabs_out) {
  static const int Gs[6] = {32, 16, 8, 4, 2, 1};
  int bestG = 1, bestC = 1, bestS = 1 << 30, bestWaste = 1 << 30;
  int wmin = 1 << 30;
  for (int gi = 0; gi < 6; ++gi)
    for (int c = 1; c <= 4; ++c) wmin = std::min(wmin, Gs[gi] * c);
  wmax = std::max(wmax, wmin);
  for (int gi = 0; gi < 6; ++gi) {
    for (int c = 1; c <= 4; ++c) {
      const int G = Gs[gi], W = G * c;
      if (W > wmax) continue;
      const int ns = (chunks + W - 1) / W;
      const int waste = ns * W - chunks;
      // fewer slabs first, then less waste; ties keep the larger G
      if (ns < bestS || (ns == bestS && waste < bestWaste)) {
        bestS = ns;
        bestWaste = waste;
        bestG = G;
        bestC = c;
      }
    }
  }
  *G_out = bestG;
  *CPL_out = bestC;
  *nslabs_out = bestS;
}

}  // namespace

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }
int dg_version(void) { return 1; }
int64_t dg_launch_count(void) { return g_launches.load(); }
int dg_device_sync(void) {
  DG_CK(cudaDeviceSynchronize());
  return DG_OK;
}

int dg_malloc(void** ptr, int64_t bytes) {
  if (!ptr || bytes < 0) return set_err(DG_ERR_ARG, "dg_malloc: bad args");
  *ptr = nullptr;
  if (bytes == 0) bytes = 16;
  DG_CK(cudaMalloc(ptr, (size_t)bytes));
  DG_CK(cudaMemset(*ptr, 0, (size_t)bytes));
  return DG_OK;
}

int dg_free(void* ptr) {
  if (ptr) DG_CK(cudaFree(ptr));
  return DG_OK;
}

int dg_memset0(void* ptr, int64_t bytes, void* stream) {
  if (bytes > 0) DG_CK(cudaMemsetAsync(ptr, 0, (size_t)bytes, S(stream)));
  return DG_OK;
}

int dg_enable_peer(int peer) {
  int dev = 0, can = 0;
  DG_CK(cudaGetDevice(&dev));
  if (peer == dev) return DG_OK;
  DG_CK(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (!can) return set_err(DG_ERR_ARG, "dg_enable_peer: no P2P path between devices");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return DG_OK;
  }
  DG_CK(e);
  return DG_OK;
}

int dg_ipc_get_handle(void* dev_ptr, uint8_t handle_out[64]) {
  cudaIpcMemHandle_t h;
  DG_CK(cudaIpcGetMemHandle(&h, dev_ptr));
  static_assert(sizeof(h) == 64, "ipc handle size");
  std::memcpy(handle_out, &h, 64);
  return DG_OK;
}

int dg_ipc_open_handle(const uint8_t handle[64], void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  DG_CK(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return DG_OK;
}

int dg_ipc_close(void* dev_ptr) {
  DG_CK(cudaIpcCloseMemHandle(dev_ptr));
  return DG_OK;
}

// ---------------------------------------------------------------------------
// SpMM plan (native host-side work-list builder)
// ---------------------------------------------------------------------------

int dg_spmm_plan_create(dg_spmm_plan** out, int n_ranks, const int64_t* n_rows,
                        const int64_t* n_local, const int64_t* nnz,
                        const int64_t* const* row_ptr, const int32_t* const* col_ext,
                        const float* const* val, int32_t max_chunk) {
  if (!out || n_ranks < 1 || n_ranks > DG_MAX_LOCAL || max_chunk < 1)
    return set_err(DG_ERR_ARG, "dg_spmm_plan_create: bad args");
  auto* p = new dg_spmm_plan();
  p->n_ranks = n_ranks;
  std::vector<Item> items;
  std::vector<Fixup> fix;
  int64_t slots = 0;
  for (int r = 0; r < n_ranks; ++r) {
    p->n_rows.push_back(n_rows[r]);
    p->n_local.push_back(n_local[r]);
    p->nnz.push_back(nnz[r]);
    if (n_rows[r] > INT32_MAX || nnz[r] > ((int64_t)1 << 40)) {
      delete p;
      return set_err(DG_ERR_ARG, "dg_spmm_plan_create: rank too large for int32 rows");
    }
    int32_t mx = -1;
    for (int64_t k = 0; k < nnz[r]; ++k) mx = std::max(mx, col_ext[r][k]);
    p->ext_rows.push_back((int64_t)mx + 1);
    for (int64_t i = 0; i < n_rows[r]; ++i) {
      const int64_t lo = row_ptr[r][i], hi = row_ptr[r][i + 1];
      const int64_t len = hi - lo;
      if (len <= max_chunk) {
        items.push_back(Item{lo, (int32_t)i, (int32_t)len, r, -1});
      } else {
        const int32_t n = (int32_t)((len + max_chunk - 1) / max_chunk);
        fix.push_back(Fixup{(int32_t)i, r, (int32_t)slots, n});
        for (int32_t k = 0; k < n; ++k) {
          const int64_t a0 = lo + (int64_t)k * max_chunk;
          const int64_t a1 = std::min(hi, a0 + max_chunk);
          items.push_back(Item{a0, (int32_t)i, (int32_t)(a1 - a0), r, (int32_t)(slots + k)});
        }
        slots += n;
      }
    }
  }
  // bucket by length (descending, stable): similar trip counts per warp,
  // heavy items first, row order kept inside a bucket for locality
  std::stable_sort(items.begin(), items.end(), [](const Item& x, const Item& y) {
    return bucket_of(x.len) > bucket_of(y.len);
  });
  p->n_items = (int64_t)items.size();
  p->n_fix = (int64_t)fix.size();
  p->n_slots = slots;
  auto fail = [&](cudaError_t e, const char* what) {
    dg_spmm_plan_destroy(p);
    return set_err(DG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  for (int r = 0; r < n_ranks; ++r) {
    int32_t* dc = nullptr;
    float* dv = nullptr;
    const size_t nb = (size_t)std::max<int64_t>(nnz[r], 1);
    cudaError_t e = cudaMalloc(&dc, nb * sizeof(int32_t));
    if (e != cudaSuccess) return fail(e, "cudaMalloc(col)");
    p->col.push_back(dc);
    e = cudaMalloc(&dv, nb * sizeof(float));
    if (e != cudaSuccess) return fail(e, "cudaMalloc(val)");
    p->val.push_back(dv);
    if (nnz[r]) {
      e = cudaMemcpy(dc, col_ext[r], nnz[r] * sizeof(int32_t), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(e, "cudaMemcpy(col)");
      e = cudaMemcpy(dv, val[r], nnz[r] * sizeof(float), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(e, "cudaMemcpy(val)");
    }
    p->dev_bytes += (int64_t)nb * 8;
  }
  cudaError_t e = cudaMalloc(&p->items, std::max<size_t>(items.size(), 1) * sizeof(Item));
  if (e != cudaSuccess) return fail(e, "cudaMalloc(items)");
  if (!items.empty()) {
    e = cudaMemcpy(p->items, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(e, "cudaMemcpy(items)");
  }
  e = cudaMalloc(&p->fix, std::max<size_t>(fix.size(), 1) * sizeof(Fixup));
  if (e != cudaSuccess) return fail(e, "cudaMalloc(fix)");
  if (!fix.empty()) {
    e = cudaMemcpy(p->fix, fix.data(), fix.size() * sizeof(Fixup), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(e, "cudaMemcpy(fix)");
  }
  p->dev_bytes += (int64_t)(items.size() * sizeof(Item) + fix.size() * sizeof(Fixup));
  *out = p;
  return DG_OK;
}

int dg_spmm_plan_destroy(dg_spmm_plan* p) {
  if (!p) return DG_OK;
  for (auto* c : p->col) cudaFree(c);
  for (auto* v : p->val) cudaFree(v);
  if (p->items) cudaFree(p->items);
  if (p->fix) cudaFree(p->fix);
  if (p->part) cudaFree(p->part);
  delete p;
  return DG_OK;
}

int dg_spmm_plan_info(const dg_spmm_plan* p, int64_t info[8]) {
  if (!p) return set_err(DG_ERR_ARG, "null plan");
  int64_t nnz = 0;
  for (auto x : p->nnz) nnz += x;
  int64_t ext = 0;
  for (auto x : p->ext_rows) ext += x;
  info[0] = p->n_items;
  info[1] = p->n_fix;
  info[2] = p->n_slots;
  info[3] = nnz;
  info[4] = p->dev_bytes + p->part_cap * 8;
  info[5] = ext;
  info[6] = 0;
  info[7] = 0;
  return DG_OK;
}

int dg_spmm_run(dg_spmm_plan* p, const float* const* h_local, const float* const* h_halo,
                float* const* z, int32_t f, int64_t ld_h, int64_t ld_z, int32_t acc,
                int32_t slab_floats, void* stream) {
  if (!p) return set_err(DG_ERR_ARG, "dg_spmm_run: null plan");
  if (f < 1 || ld_h % 4 || ld_z % 4 || f > ld_h || f > ld_z)
    return set_err(DG_ERR_ARG, "dg_spmm_run: need 1 <= f <= ld, ld % 4 == 0");
  const int chunks = (f + 3) / 4;
  SpmmArgs a;
  std::memset(&a, 0, sizeof(a));
  int64_t ext_total = 0;
  for (int r = 0; r < p->n_ranks; ++r) {
    const uintptr_t al = (uintptr_t)h_local[r] | (uintptr_t)z[r] |
                         (uintptr_t)(h_halo ? h_halo[r] : nullptr);
    if (al & 15) return set_err(DG_ERR_ARG, "dg_spmm_run: H/Z must be 16-byte aligned");
    a.r[r] = RankArgs{p->col[r], p->val[r], h_local[r], h_halo ? h_halo[r] : nullptr, z[r],
                      p->n_local[r]};
    ext_total += p->ext_rows[r];
  }
  if (p->n_slots) {
    const int64_t need = p->n_slots * ld_h;
    if (need > p->part_cap) {
      if (p->part) cudaFree(p->part);
      p->part = nullptr;
      p->part_cap = 0;
      DG_CK(cudaMalloc(&p->part, need * sizeof(double)));
      p->part_cap = need;
    }
  }
  int wmax;
  if (slab_floats > 0) {
    wmax = std::max(1, slab_floats / 4);
  } else {
    // keep one slab of every gathered row within ~64 MB of the 126 MB L2
    const double budget = 64.0 * 1024 * 1024;
    const double per_chunk = (double)std::max<int64_t>(ext_total, 1) * 16.0;
    wmax = (int)std::max(1.0, budget / per_chunk);
  }
  int G, CPL, ns;
  choose_config(chunks, wmax, &G, &CPL, &ns);
  a.items = p->items;
  a.part = p->part;
  a.n_items = p->n_items;
  a.ld_h = ld_h;
  a.ld_z = ld_z;
  a.ld_part = ld_h;
  a.chunks = chunks;
  a.slab = G * CPL;
  if (p->n_items == 0) return DG_OK;
  LaunchFn fn = acc ? pick_launch<double>(G, CPL) : pick_launch<float>(G, CPL);
  if (!fn) return set_err(DG_ERR_ARG, "dg_spmm_run: no kernel for config");
  fn(a, ns, S(stream));
  DG_LAUNCHED();
  if (p->n_fix) {
    FixArgs fa;
    std::memset(&fa, 0, sizeof(fa));
    for (int r = 0; r < p->n_ranks; ++r) fa.z[r] = z[r];
    fa.fix = p->fix;
    fa.part = p->part;
    fa.ld_z = ld_z;
    fa.ld_part = ld_h;
    fa.nfloat = chunks * 4;
    spmm_fixup_kernel<<<(unsigned)p->n_fix, 128, 0, S(stream)>>>(fa);
    DG_LAUNCHED();
  }
  return DG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// halo exchange: fused gather + (peer) store
// ---------------------------------------------------------------------------

namespace {

struct XSeg {
  const int32_t* idx;  // rows of the source H block (nullptr: contiguous)
  int64_t src_row0;
  int64_t count;
  int64_t dst_row0;
  int32_t src_local;
  int32_t dst_buf;
};

struct XArgs {
  const float* src[DG_MAX_LOCAL];
  float* dst[2 * DG_MAX_LOCAL * 2];
  const XSeg* segs;
  int64_t ld;
  int32_t chunks;
  int32_t fence_sys;
};

template <int G>
__global__ void __launch_bounds__(256) xchg_kernel(const __grid_constant__ XArgs a) {
  const XSeg sg = a.segs[blockIdx.y];
  const int lig = threadIdx.x & (G - 1);
  const int64_t per_block = blockDim.x / G;
  const float4* __restrict__ src = reinterpret_cast<const float4*>(a.src[sg.src_local]);
  float4* dst = reinterpret_cast<float4*>(a.dst[sg.dst_buf]);
  const int64_t ld4 = a.ld / 4;
  for (int64_t k = blockIdx.x * per_block + threadIdx.x / G; k < sg.count;
       k += (int64_t)gridDim.x * per_block) {
    const int64_t srow = sg.idx ? (int64_t)__ldg(sg.idx + k) : sg.src_row0 + k;
    const float4* s = src + srow * ld4;
    float4* d = dst + (sg.dst_row0 + k) * ld4;
    for (int c = lig; c < a.chunks; c += G) d[c] = __ldg(s + c);
  }
  if (a.fence_sys) __threadfence_system();
}

}  // namespace

struct dg_xchg_plan {
  int n_segs = 0;
  XSeg* segs = nullptr;
  int32_t* idx = nullptr;
  int64_t max_count = 0;
  int max_src = 0, max_dst = 0;
};

extern "C" {

int dg_xchg_plan_create(dg_xchg_plan** out, int n_segs, const int32_t* src_local,
                        const int64_t* count, const int32_t* const* idx,
                        const int64_t* src_row0, const int32_t* dst_buf,
                        const int64_t* dst_row0) {
  if (!out || n_segs < 0 || n_segs > 65535) return set_err(DG_ERR_ARG, "xchg: bad args");
  auto* p = new dg_xchg_plan();
  p->n_segs = n_segs;
  int64_t tot = 0;
  for (int s = 0; s < n_segs; ++s)
    if (idx && idx[s]) tot += count[s];
  std::vector<XSeg> segs(n_segs);
  if (tot) {
    cudaError_t e = cudaMalloc(&p->idx, tot * sizeof(int32_t));
    if (e != cudaSuccess) {
      delete p;
      return set_err(DG_ERR_CUDA, std::string("xchg idx: ") + cudaGetErrorString(e));
    }
  }
  int64_t off = 0;
  for (int s = 0; s < n_segs; ++s) {
    const int32_t* di = nullptr;
    if (idx && idx[s] && count[s]) {
      cudaError_t e = cudaMemcpy(p->idx + off, idx[s], count[s] * sizeof(int32_t),
                                 cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        dg_xchg_plan_destroy(p);
        return set_err(DG_ERR_CUDA, std::string("xchg idx copy: ") + cudaGetErrorString(e));
      }
      di = p->idx + off;
      off += count[s];
    }
    if (src_local[s] < 0 || src_local[s] >= DG_MAX_LOCAL || dst_buf[s] < 0 ||
        dst_buf[s] >= 2 * DG_MAX_LOCAL * 2) {
      dg_xchg_plan_destroy(p);
      return set_err(DG_ERR_ARG, "xchg: segment index out of range");
    }
    segs[s] = XSeg{di, src_row0[s], count[s], dst_row0[s], src_local[s], dst_buf[s]};
    p->max_count = std::max(p->max_count, count[s]);
    p->max_src = std::max(p->max_src, src_local[s] + 1);
    p->max_dst = std::max(p->max_dst, dst_buf[s] + 1);
  }
  if (n_segs) {
    cudaError_t e = cudaMalloc(&p->segs, n_segs * sizeof(XSeg));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->segs, segs.data(), n_segs * sizeof(XSeg), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      dg_xchg_plan_destroy(p);
      return set_err(DG_ERR_CUDA, std::string("xchg segs: ") + cudaGetErrorString(e));
    }
  }
  *out = p;
  return DG_OK;
}

int dg_xchg_plan_destroy(dg_xchg_plan* p) {
  if (!p) return DG_OK;
  if (p->segs) cudaFree(p->segs);
  if (p->idx) cudaFree(p->idx);
  delete p;
  return DG_OK;
}

int dg_xchg_run(dg_xchg_plan* p, const float* const* h_src, int n_src, float* const* dst_bufs,
                int n_dst, int32_t f, int64_t ld, int32_t fence_sys, void* stream) {
  if (!p) return set_err(DG_ERR_ARG, "xchg_run: null plan");
  if (p->n_segs == 0 || p->max_count == 0) return DG_OK;
  if (n_src < p->max_src || n_dst < p->max_dst || n_src > DG_MAX_LOCAL ||
      n_dst > 2 * DG_MAX_LOCAL * 2 || ld % 4 || f > ld || f < 1)
    return set_err(DG_ERR_ARG, "xchg_run: bad buffer tables / ld");
  XArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int i = 0; i < n_src; ++i) a.src[i] = h_src[i];
  for (int i = 0; i < n_dst; ++i) a.dst[i] = dst_bufs[i];
  a.segs = p->segs;
  a.ld = ld;
  a.chunks = (f + 3) / 4;
  a.fence_sys = fence_sys;
  int G = 1;
  while (G < a.chunks && G < 32) G <<= 1;
  const int64_t per_block = 256 / G;
  int64_t gx = (p->max_count + per_block - 1) / per_block;
  gx = std::min<int64_t>(std::max<int64_t>(gx, 1), 4 * 148);
  dim3 grid((unsigned)gx, (unsigned)p->n_segs);
  switch (G) {
    case 1: xchg_kernel<1><<<grid, 256, 0, S(stream)>>>(a); break;
    case 2: xchg_kernel<2><<<grid, 256, 0, S(stream)>>>(a); break;
    case 4: xchg_kernel<4><<<grid, 256, 0, S(stream)>>>(a); break;
    case 8: xchg_kernel<8><<<grid, 256, 0, S(stream)>>>(a); break;
    case 16: xchg_kernel<16><<<grid, 256, 0, S(stream)>>>(a); break;
    default: xchg_kernel<32><<<grid, 256, 0, S(stream)>>>(a); break;
  }
  DG_LAUNCHED();
  return DG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// group all-reduce (ascending member order, one reduction per element)
// ---------------------------------------------------------------------------

namespace {

struct RArgs {
  const float* src[DG_MAX_GROUP];
  float* dst[DG_MAX_GROUP];
  int64_t lo, hi;
  int32_t g;
  int32_t vec;         // all pointers 16 B aligned and lo % 4 == 0
  int32_t fence_sys;
};

__global__ void __launch_bounds__(256) group_reduce_kernel(const __grid_constant__ RArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t tail = a.lo;
  if (a.vec) {
    const int64_t n4 = (a.hi - a.lo) / 4;
    for (int64_t i = t0; i < n4; i += stride) {
      const int64_t e = a.lo + 4 * i;
      float4 s = *reinterpret_cast<const float4*>(a.src[0] + e);
      for (int m = 1; m < a.g; ++m) {
        const float4 x = *reinterpret_cast<const float4*>(a.src[m] + e);
        s.x += x.x;
        s.y += x.y;
        s.z += x.z;
        s.w += x.w;
      }
      for (int m = 0; m < a.g; ++m) *reinterpret_cast<float4*>(a.dst[m] + e) = s;
    }
    tail = a.lo + 4 * n4;
  }
  for (int64_t e = tail + t0; e < a.hi; e += stride) {
    float s = a.src[0][e];
    for (int m = 1; m < a.g; ++m) s += a.src[m][e];
    for (int m = 0; m < a.g; ++m) a.dst[m][e] = s;
  }
  if (a.fence_sys) __threadfence_system();
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct BArgs {
  uint64_t* flags[DG_MAX_LOCAL];
  int32_t* err;
  uint64_t epoch;
  int64_t timeout_ns;
  int32_t n;
  int32_t me;
};

__global__ void barrier_kernel(const __grid_constant__ BArgs a) {
  const int q = threadIdx.x;
  __threadfence_system();
  __syncthreads();
  if (q < a.n) {
    uint64_t* remote = a.flags[q] + a.me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote), "l"(a.epoch) : "memory");
  }
  if (q < a.n) {
    uint64_t* mine = a.flags[a.me] + q;
    const uint64_t t0 = gtimer();
    while (true) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= a.epoch) break;
      if (gtimer() - t0 > (uint64_t)a.timeout_ns) {
        atomicExch(a.err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

}  // namespace

extern "C" {

int dg_group_reduce(int g, const float* const* src, float* const* dst, int64_t lo, int64_t hi,
                    int32_t fence_sys, void* stream) {
  if (g < 1 || g > DG_MAX_GROUP || hi < lo) return set_err(DG_ERR_ARG, "group_reduce: bad args");
  if (hi == lo) return DG_OK;
  RArgs a;
  std::memset(&a, 0, sizeof(a));
  bool aligned = (lo & 3) == 0;
  for (int m = 0; m < g; ++m) {
    a.src[m] = src[m];
    a.dst[m] = dst[m];
    aligned = aligned && (((uintptr_t)src[m] | (uintptr_t)dst[m]) & 15) == 0;
  }
  a.lo = lo;
  a.hi = hi;
  a.g = g;
  a.vec = aligned ? 1 : 0;
  a.fence_sys = fence_sys;
  const int64_t n = hi - lo;
  int64_t blocks = ((aligned ? n / 4 : n) + 255) / 256;
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 8 * 148);
  group_reduce_kernel<<<(unsigned)blocks, 256, 0, S(stream)>>>(a);
  DG_LAUNCHED();
  return DG_OK;
}

int dg_barrier(uint64_t* const* flags, int n_procs, int me, uint64_t epoch, int64_t timeout_ns,
               int32_t* err_dev, void* stream) {
  if (n_procs < 1 || n_procs > DG_MAX_LOCAL || me < 0 || me >= n_procs)
    return set_err(DG_ERR_ARG, "barrier: bad args");
  if (n_procs == 1) return DG_OK;
  BArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int q = 0; q < n_procs; ++q) a.flags[q] = flags[q];
  a.err = err_dev;
  a.epoch = epoch;
  a.timeout_ns = timeout_ns;
  a.n = n_procs;
  a.me = me;
  barrier_kernel<<<1, 64, 0, S(stream)>>>(a);
  DG_LAUNCHED();
  return DG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// host preprocessing (native): stable O(nnz + n) CSR transpose
// (sparse.transpose_csr, sparse.py:237-247 -- a stable argsort of the column
// indices; a counting sort gives the identical permutation)
// ---------------------------------------------------------------------------

extern "C" int dg_host_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                                 const int64_t* col, const double* val, int64_t* out_row_ptr,
                                 int64_t* out_col, double* out_val) {
  if (n_rows < 0 || n_cols < 0) return set_err(DG_ERR_ARG, "transpose: bad dims");
  const int64_t nnz = row_ptr[n_rows];
  std::vector<int64_t> fill(n_cols + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) {
    const int64_t c = col[e];
    if (c < 0 || c >= n_cols) return set_err(DG_ERR_ARG, "transpose: column out of range");
    ++fill[c + 1];
  }
  for (int64_t c = 0; c < n_cols; ++c) fill[c + 1] += fill[c];
  std::memcpy(out_row_ptr, fill.data(), (n_cols + 1) * sizeof(int64_t));
  for (int64_t r = 0; r < n_rows; ++r) {
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      const int64_t d = fill[col[e]]++;
      out_col[d] = r;
      out_val[d] = val[e];
    }
  }
  return DG_OK;
}

// ---------------------------------------------------------------------------
// GCN pieces
// ---------------------------------------------------------------------------

namespace {

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_min(int v) {
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// one warp per row; 8 rows per block; deterministic two-level reduction
__global__ void __launch_bounds__(256) xent_kernel(const float* __restrict__ x, int64_t n, int C,
                                                   int64_t ld, const int64_t* __restrict__ labels,
                                                   const uint8_t* __restrict__ mask, double denom,
                                                   float* __restrict__ grad, int64_t ldg,
                                                   double* scratch, unsigned* counter,
                                                   double* out) {
  __shared__ double s_loss[8];
  __shared__ double s_corr[8];
  __shared__ bool s_last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + w;
  double loss = 0.0, corr = 0.0;
  if (row < n) {
    const float* xr = x + row * ld;
    float m = -INFINITY;
    for (int j = lane; j < C; j += 32) m = fmaxf(m, xr[j]);
    m = warp_max(m);
    double s = 0.0;
    for (int j = lane; j < C; j += 32) s += exp((double)xr[j] - (double)m);
    s = warp_sum(s);
    int am = C;
    for (int j = lane; j < C; j += 32)
      if (xr[j] == m) {
        am = j;
        break;
      }
    am = warp_min(am);
    const bool on = mask[row] != 0;
    const int64_t lbl = labels[row];
    float* gr = grad + row * ldg;
    for (int j = lane; j < C; j += 32) {
      float gv = 0.f;
      if (on) {
        double sm = exp((double)xr[j] - (double)m) / s;
        if (j == lbl) sm -= 1.0;
        gv = (float)(sm / denom);
      }
      gr[j] = gv;
    }
    for (int j = C + lane; j < ldg; j += 32) gr[j] = 0.f;
    if (on) {
      loss = log(s) - ((double)xr[lbl] - (double)m);
      corr = (am == lbl) ? 1.0 : 0.0;
    }
  }
  if (lane == 0) {
    s_loss[w] = loss;
    s_corr[w] = corr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0, c = 0.0;
    for (int i = 0; i < 8; ++i) {
      l += s_loss[i];
      c += s_corr[i];
    }
    scratch[2 * blockIdx.x] = l;
    scratch[2 * blockIdx.x + 1] = c;
    __threadfence();
    const unsigned done = atomicAdd(counter, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    __shared__ double r_l[256];
    __shared__ double r_c[256];
    double l = 0.0, c = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
      l += ((volatile double*)scratch)[2 * b];
      c += ((volatile double*)scratch)[2 * b + 1];
    }
    r_l[threadIdx.x] = l;
    r_c[threadIdx.x] = c;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
      if ((int)threadIdx.x < o) {
        r_l[threadIdx.x] += r_l[threadIdx.x + o];
        r_c[threadIdx.x] += r_c[threadIdx.x + o];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      out[0] += r_l[0];
      out[1] += r_c[0];
      *counter = 0u;
    }
  }
}

__global__ void relu_kernel(const float4* __restrict__ z, float4* __restrict__ h, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = z[i];
    v.x = fmaxf(v.x, 0.f);
    v.y = fmaxf(v.y, 0.f);
    v.z = fmaxf(v.z, 0.f);
    v.w = fmaxf(v.w, 0.f);
    h[i] = v;
  }
}

__global__ void relu_grad_mul_kernel(float* g, int64_t ldg, const float* __restrict__ z,
                                     int64_t ldz, int64_t rows, int f) {
  const int64_t n = rows * (int64_t)f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / f;
    const int c = (int)(i - r * f);
    if (!(z[r * ldz + c] > 0.f)) g[r * ldg + c] = 0.f;
  }
}

__global__ void sgd_kernel(float* w, const float* __restrict__ y, int64_t n, float lr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] -= lr * y[i];
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)std::min<int64_t>(std::max<int64_t>(b, 1), 16 * 148);
}

}  // namespace

extern "C" {

int dg_xent(const float* logits, int64_t n, int32_t C, int64_t ld, const int64_t* labels,
            const uint8_t* mask, double denom, float* grad, int64_t ld_grad, double* scratch,
            uint32_t* counter, double* stats_out, void* stream) {
  if (n < 1 || C < 1 || C > ld || C > ld_grad) return set_err(DG_ERR_ARG, "xent: bad args");
  const unsigned blocks = (unsigned)((n + 7) / 8);
  xent_kernel<<<blocks, 256, 0, S(stream)>>>(logits, n, C, ld, labels, mask, denom, grad,
                                             ld_grad, scratch, counter, stats_out);
  DG_LAUNCHED();
  return DG_OK;
}

int dg_relu(const float* z, float* h, int64_t rows, int32_t f, int64_t ld, void* stream) {
  if (ld % 4 || f > ld) return set_err(DG_ERR_ARG, "relu: ld % 4 != 0");
  const int64_t n4 = rows * ld / 4;
  if (!n4) return DG_OK;
  relu_kernel<<<grid_for(n4, 256), 256, 0, S(stream)>>>(reinterpret_cast<const float4*>(z),
                                                        reinterpret_cast<float4*>(h), n4);
  DG_LAUNCHED();
  return DG_OK;
}

int dg_relu_grad_mul(float* g, int64_t ld_g, const float* zprev, int64_t ld_z, int64_t rows,
                     int32_t f, void* stream) {
  const int64_t n = rows * (int64_t)f;
  if (!n) return DG_OK;
  relu_grad_mul_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(g, ld_g, zprev, ld_z, rows, f);
  DG_LAUNCHED();
  return DG_OK;
}

int dg_sgd(float* w, const float* y, int64_t n, float lr, void* stream) {
  if (!n) return DG_OK;
  sgd_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(w, y, n, lr);
  DG_LAUNCHED();
  return DG_OK;
}

}  // extern "C"
