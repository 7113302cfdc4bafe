// comm.cu -- halo exchange (fused gather + peer store), group all-reduce
// and the cross-process device barrier.

#include "common.cuh"

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

// One group of G lanes moves one row; lane l owns float4 chunks l, l+G, ...
// (up to CPL per lane).  All of a lane's loads are issued before its
// stores, so a warp keeps CPL x 512 B of (possibly remote, NVLink) stores in
// flight per row instead of one load-store round trip per chunk.
template <int G, int CPL>
__global__ void __launch_bounds__(256) xchg_kernel(const __grid_constant__ XArgs a) {
  const XSeg sg = a.segs[blockIdx.y];
  const int lig = threadIdx.x & (G - 1);
  const int64_t per_block = blockDim.x / G;
  const float4* __restrict__ src = reinterpret_cast<const float4*>(a.src[sg.src_local]);
  float4* dst = reinterpret_cast<float4*>(a.dst[sg.dst_buf]);
  const int64_t ld4 = a.ld / 4;
  // two rows per group per step: both rows' loads are issued before either
  // row's stores, so a capped grid (few CTAs beside an overlapped SpMM)
  // still keeps enough DRAM / L2 reads in flight
  const int64_t stride = (int64_t)gridDim.x * per_block;
  for (int64_t k = blockIdx.x * per_block + threadIdx.x / G; k < sg.count; k += 2 * stride) {
    const int64_t k2 = k + stride;
    const bool two = k2 < sg.count;
    const int64_t srow = sg.idx ? (int64_t)__ldg(sg.idx + k) : sg.src_row0 + k;
    const int64_t srow2 = two ? (sg.idx ? (int64_t)__ldg(sg.idx + k2) : sg.src_row0 + k2) : srow;
    const float4* s = src + srow * ld4;
    const float4* s2 = src + srow2 * ld4;
    float4 v[CPL], v2[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lig + q * G;
      if (c < a.chunks) {
        v[q] = __ldg(s + c);
        if (two) v2[q] = __ldg(s2 + c);
      }
    }
    float4* d = dst + (sg.dst_row0 + k) * ld4;
    float4* d2 = dst + (sg.dst_row0 + k2) * ld4;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lig + q * G;
      if (c < a.chunks) {
        d[c] = v[q];
        if (two) d2[c] = v2[q];
      }
    }
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
                                 cudaMemcpyDefault);   // host or device lists (UVA)
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
  return dg_xchg_run_ctas(p, h_src, n_src, dst_bufs, n_dst, f, ld, fence_sys, 0, stream);
}

int dg_xchg_run_ctas(dg_xchg_plan* p, const float* const* h_src, int n_src,
                     float* const* dst_bufs, int n_dst, int32_t f, int64_t ld,
                     int32_t fence_sys, int32_t max_ctas, void* stream) {
  if (!p) return set_err(DG_ERR_ARG, "xchg_run: null plan");
  if (p->n_segs == 0 || p->max_count == 0) return DG_OK;
  if (n_src < p->max_src || n_dst < p->max_dst || n_src > DG_MAX_LOCAL ||
      n_dst > 2 * DG_MAX_LOCAL * 2 || ld % 4 || f > ld || f < 1 || (f + 3) / 4 > 512)
    return set_err(DG_ERR_ARG, "xchg_run: bad buffer tables / ld");
  XArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int i = 0; i < n_src; ++i) a.src[i] = h_src[i];
  for (int i = 0; i < n_dst; ++i) a.dst[i] = dst_bufs[i];
  a.segs = p->segs;
  a.ld = ld;
  // whole 32-B chunks when the rows allow it: the SpMM's 256-bit path reads
  // rows in 8-float units, so the halo must carry the zero padding too
  a.chunks = (ld % 8 == 0) ? std::min<int>((int)(ld / 4), 2 * ((f + 7) / 8)) : (f + 3) / 4;
  a.fence_sys = fence_sys;
  int G = 1;
  while (G < a.chunks && G < 32) G <<= 1;
  const int cpl = (a.chunks + G - 1) / G;
  const int64_t per_block = 256 / G;
  int64_t gx = (p->max_count + per_block - 1) / per_block;
  gx = std::min<int64_t>(std::max<int64_t>(gx, 1), 16 * 148);
  // max_ctas: CTAs in flight across all segments.  Uncapped (0), the grid
  // keeps thousands of rows in flight -- what an exchange whose source rows
  // come from DRAM needs (papers-shaped: a 296-CTA grid halved its NVLink
  // rate) -- but beside the own-block SpMM of an overlapped phase it takes
  // every SM first; the caller caps it there (profiles/r02/xchg_cap/)
  if (max_ctas > 0)
    gx = std::min<int64_t>(gx, std::max(1, max_ctas / std::max(1, p->n_segs)));
  dim3 grid((unsigned)gx, (unsigned)p->n_segs);
  cudaStream_t st = S(stream);
#define DG_X(g, c) xchg_kernel<g, c><<<grid, 256, 0, st>>>(a)
  if (G < 32) {
    switch (G) {
      case 1: DG_X(1, 1); break;
      case 2: DG_X(2, 1); break;
      case 4: DG_X(4, 1); break;
      case 8: DG_X(8, 1); break;
      default: DG_X(16, 1); break;
    }
  } else if (cpl <= 1) {
    DG_X(32, 1);
  } else if (cpl <= 2) {
    DG_X(32, 2);
  } else if (cpl <= 4) {
    DG_X(32, 4);
  } else if (cpl <= 8) {
    DG_X(32, 8);
  } else {
    DG_X(32, 16);
  }
#undef DG_X
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
  int32_t nd;
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
      for (int m = 0; m < a.nd; ++m) *reinterpret_cast<float4*>(a.dst[m] + e) = s;
    }
    tail = a.lo + 4 * n4;
  }
  for (int64_t e = tail + t0; e < a.hi; e += stride) {
    float s = a.src[0][e];
    for (int m = 1; m < a.g; ++m) s += a.src[m][e];
    for (int m = 0; m < a.nd; ++m) a.dst[m][e] = s;
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
        // Fail closed: a stalled peer means the halos / partial slots the
        // following kernels read are stale.  Record the cause, then trap so
        // the context faults and every later launch (and the host's next
        // sync) reports the error instead of computing on stale data.
        atomicExch(a.err, 1);
        __threadfence_system();
        __trap();
      }
    }
  }
  __syncthreads();
}

}  // namespace

extern "C" {

int dg_group_reduce(int g, const float* const* src, int n_dst, float* const* dst, int64_t lo,
                    int64_t hi, int32_t fence_sys, void* stream) {
  if (g < 1 || g > DG_MAX_GROUP || n_dst < 1 || n_dst > DG_MAX_GROUP || hi < lo)
    return set_err(DG_ERR_ARG, "group_reduce: bad args");
  if (hi == lo) return DG_OK;
  RArgs a;
  std::memset(&a, 0, sizeof(a));
  bool aligned = (lo & 3) == 0;
  for (int m = 0; m < g; ++m) {
    a.src[m] = src[m];
    aligned = aligned && ((uintptr_t)src[m] & 15) == 0;
  }
  for (int m = 0; m < n_dst; ++m) {
    a.dst[m] = dst[m];
    aligned = aligned && ((uintptr_t)dst[m] & 15) == 0;
  }
  a.nd = n_dst;
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
// diagnostic: random-row gather bandwidth (the practical ceiling of the SpMM's
// H-row gathers).  Each group of G lanes sums `per_group` rows of `row_bytes`
// (= 16*G) chosen by idx[]; the table has `rows` rows of pitch `ld` floats.
// ---------------------------------------------------------------------------

namespace {

template <int G>
__global__ void __launch_bounds__(256) gather_probe_kernel(const float* __restrict__ tab,
                                                           int64_t ld, const int32_t* __restrict__ idx,
                                                           int64_t n_idx, int per_group,
                                                           float* __restrict__ out) {
  const int lig = threadIdx.x & (G - 1);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t base = grp * per_group;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < per_group; k += 4) {
    int r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = __ldg(idx + ((base + k + u) % n_idx));
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      x[u] = __ldg(reinterpret_cast<const float4*>(tab + (int64_t)r[u] * ld) + lig);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc.x += x[u].x;
      acc.y += x[u].y;
      acc.z += x[u].z;
      acc.w += x[u].w;
    }
  }
  if (acc.x == 123.456f) out[0] = acc.y + acc.z + acc.w;   // keep the loads alive
}

// 256-bit variant: each lane loads 32 B (two float4) with one
// ld.global.nc.v8 (Blackwell); G lanes cover 32*G bytes of a row.
template <int G>
__global__ void __launch_bounds__(256) gather_probe_v8_kernel(const float* __restrict__ tab,
                                                              int64_t ld,
                                                              const int32_t* __restrict__ idx,
                                                              int64_t n_idx, int per_group,
                                                              float* __restrict__ out) {
  const int lig = threadIdx.x & (G - 1);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t base = grp * per_group;
  float acc = 0.f;
  for (int k = 0; k < per_group; k += 4) {
    int r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = __ldg(idx + ((base + k + u) % n_idx));
    float x[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float* p = tab + (int64_t)r[u] * ld + 8 * lig;
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(x[u][0]), "=f"(x[u][1]), "=f"(x[u][2]), "=f"(x[u][3]), "=f"(x[u][4]),
                     "=f"(x[u][5]), "=f"(x[u][6]), "=f"(x[u][7])
                   : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc += x[u][e];
  }
  if (acc == 123.456f) out[0] = acc;
}

}  // namespace

extern "C" int dg_diag_gather(const float* tab, int64_t ld, const int32_t* idx, int64_t n_idx,
                              int32_t lanes, int64_t groups, int32_t per_group, float* out,
                              void* stream) {
  const unsigned blocks = (unsigned)((groups * lanes + 255) / 256);
  if (lanes < 0) {                       // 256-bit loads: -lanes lanes x 32 B
    switch (-lanes) {
      case 2: gather_probe_v8_kernel<2><<<(unsigned)((groups * 2 + 255) / 256), 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
      case 4: gather_probe_v8_kernel<4><<<(unsigned)((groups * 4 + 255) / 256), 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
      case 8: gather_probe_v8_kernel<8><<<(unsigned)((groups * 8 + 255) / 256), 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
      case 16: gather_probe_v8_kernel<16><<<(unsigned)((groups * 16 + 255) / 256), 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
      default: return set_err(DG_ERR_ARG, "diag_gather: v8 lanes must be 2, 4, 8 or 16");
    }
    DG_LAUNCHED();
    return DG_OK;
  }
  switch (lanes) {
    case 4: gather_probe_kernel<4><<<blocks, 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
    case 8: gather_probe_kernel<8><<<blocks, 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
    case 16: gather_probe_kernel<16><<<blocks, 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
    case 32: gather_probe_kernel<32><<<blocks, 256, 0, S(stream)>>>(tab, ld, idx, n_idx, per_group, out); break;
    default: return set_err(DG_ERR_ARG, "diag_gather: lanes must be 4, 8, 16 or 32");
  }
  DG_LAUNCHED();
  return DG_OK;
}
