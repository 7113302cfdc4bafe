// dense.cu -- the GCN's dense transforms, tall-skinny and memory-bound:
//
//   forward   Z = T W            gcn.py:274  (T: n x K, W: K x N, N <= 64)
//             H = relu(Z)        gcn.py:276  (fused epilogue, optional)
//   backward  G = (M W^T) * 1[Zprev > 0]     gcn.py:282  (fused mask, optional)
//   wgrad     Y = H^T M          gcn.py:280  (K x N, N <= 256, reduction over the n rows)
//
// fp32 SIMT (TF32 would break the fp32 parity contract); these shapes are
// HBM-bound (T or H is read once: 566 MB for Reddit layer 1), so the target
// is streaming the tall operand at HBM speed, not tensor-core FLOPs.
//
// dg_dense_rows: a CTA owns 64 rows x all N columns; B lives in shared
// memory (K x N <= 16K floats); A is staged in 32-wide k-chunks, transposed
// so a thread reads 4 consecutive rows with one 16-B shared load; thread
// tile 4 rows x N/16 columns.
//
// dg_dense_tn: grid = (row slices, 64-wide K blocks); each CTA accumulates
// its slice's partial H^T M (fp32 per 64-row chunk, folded into fp64) and
// writes it to `work`; a second kernel sums the partials in slice order
// (fp64) -- deterministic, unlike split-K with atomics.

#include "common.cuh"

#include <cstdlib>

namespace {

constexpr int BK = 32;   // k-chunk

// Thread tile 4 rows x TN columns; CG column groups x (256 / CG) row groups,
// so a CTA covers BM = 4 * 256 / CG rows.  N <= 16 uses TN = 4, CG = 4
// (256 rows per CTA): each A value read from shared memory feeds 4 FMAs and
// the 4 column groups of a row group read it as a broadcast (16 threads
// across N with TN = 1 read every A value 16 times: shared-memory bound).
template <int TN, int CG = 16, int BKT = BK, int MB = 1>
__global__ void __launch_bounds__(256, MB) dense_rows_kernel(
    const float* __restrict__ A, int64_t lda, int64_t n, int K, const float* __restrict__ B,
    int64_t ldb, int N, int transB, float* __restrict__ C, int64_t ldc,
    float* __restrict__ Crelu, const float* __restrict__ Zmask, int64_t ldm) {
  extern __shared__ float smem[];
  constexpr int NP = CG * TN;                        // padded N
  constexpr int BM = 4 * 256 / CG;                   // rows per CTA
  float* Bs = smem;                                  // K x NP
  float* As = smem + (size_t)K * NP;                 // BKT x (BM + 4)
  const int tid = threadIdx.x;
  const int tx = tid % CG;                           // column group
  const int ty = tid / CG;                           // row group (4 rows)
  for (int i = tid; i < K * NP; i += 256) {
    const int k = i / NP, j = i % NP;
    float b = 0.f;
    if (j < N) b = transB ? B[(int64_t)j * ldb + k] : B[(int64_t)k * ldb + j];
    Bs[i] = b;
  }
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  float acc[4][TN];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = 0.f;
  // A chunk loader: each thread owns PER float4 of the BM x 32 chunk; the
  // next chunk is loaded into registers while the current one is consumed
  constexpr int PER = BM * BKT / 4 / 256;            // float4 per thread
  auto load_chunk = [&](int k0, float4* v) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = tid + u * 256;
      const int r = i / (BKT / 4), q = i % (BKT / 4);
      const int64_t gr = row0 + r;
      const int k = k0 + 4 * q;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < n && k < K) {
        const float* ap = A + gr * lda + k;
        if (k + 3 < K) {
          v[u] = __ldcs(reinterpret_cast<const float4*>(ap));
        } else {
          v[u].x = ap[0];
          if (k + 1 < K) v[u].y = ap[1];
          if (k + 2 < K) v[u].z = ap[2];
        }
      }
    }
  };
  float4 nxt[PER];
  load_chunk(0, nxt);
  for (int k0 = 0; k0 < K; k0 += BKT) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {                  // stage transposed: As[k][r]
      const int i = tid + u * 256;
      const int r = i / (BKT / 4), q = i % (BKT / 4);
      As[(4 * q + 0) * (BM + 4) + r] = nxt[u].x;
      As[(4 * q + 1) * (BM + 4) + r] = nxt[u].y;
      As[(4 * q + 2) * (BM + 4) + r] = nxt[u].z;
      As[(4 * q + 3) * (BM + 4) + r] = nxt[u].w;
    }
    __syncthreads();
    if (k0 + BKT < K) load_chunk(k0 + BKT, nxt);       // in flight during the math
    const int kmax = min(BKT, K - k0);
#pragma unroll 8
    for (int kk = 0; kk < kmax; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk * (BM + 4) + 4 * ty]);
      const float* bp = &Bs[(k0 + kk) * NP + tx * TN];
      float b[TN];
#pragma unroll
      for (int c = 0; c < TN; ++c) b[c] = bp[c];
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        acc[0][c] = fmaf(a.x, b[c], acc[0][c]);
        acc[1][c] = fmaf(a.y, b[c], acc[1][c]);
        acc[2][c] = fmaf(a.z, b[c], acc[2][c]);
        acc[3][c] = fmaf(a.w, b[c], acc[3][c]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t gr = row0 + 4 * ty + r;
    if (gr >= n) continue;
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int j = tx * TN + c;
      if (j >= ldc) continue;
      float v = acc[r][c];
      if (Zmask && j < N && !(Zmask[gr * ldm + j] > 0.f)) v = 0.f;
      C[gr * ldc + j] = v;
      if (Crelu) Crelu[gr * ldc + j] = fmaxf(v, 0.f);
    }
  }
}

// Y partials: CTA (bx, by) sums rows [bx*rows_per, ...) for K columns
// [by*64, by*64+64) x all N (<= 64) outputs; thread tile 4 (k) x TN (n).
// N > 64: grid.z splits the output columns into 64-wide blocks (TN = 4);
// the work rows are NPT = 64 * gridDim.z wide.
template <int TN>
__global__ void __launch_bounds__(256) dense_tn_kernel(
    const float* __restrict__ H, int64_t ldh, int64_t n, int K, const float* __restrict__ M,
    int64_t ldm, int N, int64_t rows_per, double* __restrict__ work) {
  constexpr int NP = 16 * TN;
  const int n0 = blockIdx.z * NP;                    // first output column of this CTA
  const int NPT = NP * gridDim.z;
  constexpr int RC = 64;                             // rows per chunk
  __shared__ __align__(16) float Hs[RC][64 + 4];
  __shared__ __align__(16) float Ms[RC][NP + 4];
  constexpr int MPER = (RC * NP + 255) / 256;        // M elements per thread
  const int tid = threadIdx.x;
  const int tx = tid % 16;                           // n group
  const int ty = tid / 16;                           // k group (4)
  const int k0 = blockIdx.y * 64;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per;
  const int64_t r_end = min(n, r_begin + rows_per);
  float part[4][TN];
  double acc[4][TN];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      part[i][c] = 0.f;
      acc[i][c] = 0.0;
    }
  // chunk loaders (H: 64 rows x 64 cols = 4 float4 per thread; M: 64 x NP);
  // the next chunk is loaded into registers while the current is consumed
  auto load_chunk = [&](int64_t r0, float4* hv, float* mv) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = tid + u * 256;
      const int rr = i / 16, q = i % 16;
      const int64_t gr = r0 + rr;
      const int k = k0 + 4 * q;
      hv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < r_end && k < K) {
        const float* hp = H + gr * ldh + k;
        if (k + 3 < K) {
          hv[u] = __ldcs(reinterpret_cast<const float4*>(hp));
        } else {
          hv[u].x = hp[0];
          if (k + 1 < K) hv[u].y = hp[1];
          if (k + 2 < K) hv[u].z = hp[2];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < MPER; ++u) {
      const int i = tid + u * 256;
      const int rr = i / NP, j = n0 + i % NP;
      const int64_t gr = r0 + rr;
      mv[u] = (i < RC * NP && gr < r_end && j < N) ? M[gr * ldm + j] : 0.f;
    }
  };
  float4 hv[4];
  float mv[MPER];
  if (r_begin < r_end) load_chunk(r_begin, hv, mv);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += RC) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = tid + u * 256;
      *reinterpret_cast<float4*>(&Hs[i / 16][4 * (i % 16)]) = hv[u];
    }
#pragma unroll
    for (int u = 0; u < MPER; ++u) {
      const int i = tid + u * 256;
      if (i < RC * NP) Ms[i / NP][i % NP] = mv[u];
    }
    __syncthreads();
    if (r0 + RC < r_end) load_chunk(r0 + RC, hv, mv);
#pragma unroll 4
    for (int rr = 0; rr < RC; ++rr) {
      const float4 h = *reinterpret_cast<const float4*>(&Hs[rr][4 * ty]);
      float m[TN];
#pragma unroll
      for (int c = 0; c < TN; ++c) m[c] = Ms[rr][tx * TN + c];
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        part[0][c] = fmaf(h.x, m[c], part[0][c]);
        part[1][c] = fmaf(h.y, m[c], part[1][c]);
        part[2][c] = fmaf(h.z, m[c], part[2][c]);
        part[3][c] = fmaf(h.w, m[c], part[3][c]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        acc[i][c] += (double)part[i][c];
        part[i][c] = 0.f;
      }
  }
  // work layout: [slice][K][NPT]
  double* wp = work + (int64_t)blockIdx.x * K * NPT;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + 4 * ty + i;
    if (k >= K) continue;
#pragma unroll
    for (int c = 0; c < TN; ++c) wp[(int64_t)k * NPT + n0 + tx * TN + c] = acc[i][c];
  }
}

// N <= 16 (every hidden width): thread tile 4 k x 4 n; 64 k-groups x 4
// n-groups cover a 256-wide K block.  Per row each thread reads one float4
// of H and one of M (both broadcast within a warp) for 16 FMAs, instead of
// 4 FMAs per two shared loads with 16 threads across N.
constexpr int TN4_RC = 32;                  // rows per chunk

__global__ void __launch_bounds__(256, 2) dense_tn4_kernel(
    const float* __restrict__ H, int64_t ldh, int64_t n, int K, const float* __restrict__ M,
    int64_t ldm, int N, int64_t rows_per, double* __restrict__ work) {
  __shared__ __align__(16) float Hs[TN4_RC][256 + 4];
  __shared__ __align__(16) float Ms[TN4_RC][16 + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 3;                            // columns 4 tx .. 4 tx + 3
  const int ty = tid >> 2;                           // k = k0 + 4 ty .. + 3
  const int k0 = blockIdx.y * 256;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per;
  const int64_t r_end = min(n, r_begin + rows_per);
  float part[4][4];
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      part[i][c] = 0.f;
      acc[i][c] = 0.0;
    }
  // chunk loaders: H 32 x 256 (8 float4 per thread), M 32 x 16 (half a float4)
  auto load_chunk = [&](int64_t r0, float4* hv, float4& mv) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = tid + u * 256;
      const int rr = i >> 6, q = i & 63;
      const int64_t gr = r0 + rr;
      const int k = k0 + 4 * q;
      hv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < r_end && k < K) {
        const float* hp = H + gr * ldh + k;
        if (k + 3 < K) {
          hv[u] = __ldcs(reinterpret_cast<const float4*>(hp));
        } else {
          hv[u].x = hp[0];
          if (k + 1 < K) hv[u].y = hp[1];
          if (k + 2 < K) hv[u].z = hp[2];
        }
      }
    }
    mv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid < TN4_RC * 4) {
      const int rr = tid >> 2, q = tid & 3;
      const int64_t gr = r0 + rr;
      if (gr < r_end) {
        const float* mp = M + gr * ldm + 4 * q;
        float t[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] = (4 * q + e < N) ? mp[e] : 0.f;
        mv = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
  };
  float4 hv[8], mv;
  if (r_begin < r_end) load_chunk(r_begin, hv, mv);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += TN4_RC) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = tid + u * 256;
      *reinterpret_cast<float4*>(&Hs[i >> 6][4 * (i & 63)]) = hv[u];
    }
    if (tid < TN4_RC * 4) *reinterpret_cast<float4*>(&Ms[tid >> 2][4 * (tid & 3)]) = mv;
    __syncthreads();
    if (r0 + TN4_RC < r_end) load_chunk(r0 + TN4_RC, hv, mv);
#pragma unroll 4
    for (int rr = 0; rr < TN4_RC; ++rr) {
      const float4 h = *reinterpret_cast<const float4*>(&Hs[rr][4 * ty]);
      const float4 m = *reinterpret_cast<const float4*>(&Ms[rr][4 * tx]);
      const float hh[4] = {h.x, h.y, h.z, h.w};
      const float mm[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) part[i][c] = fmaf(hh[i], mm[c], part[i][c]);
    }
    if (((r0 - r_begin) / TN4_RC) % 2 == 1 || r0 + TN4_RC >= r_end) {   // 64-row windows
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[i][c] += (double)part[i][c];
          part[i][c] = 0.f;
        }
    }
  }
  // work layout: [slice][K][16]
  double* wp = work + (int64_t)blockIdx.x * K * 16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + 4 * ty + i;
    if (k >= K) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) wp[(int64_t)k * 16 + 4 * tx + c] = acc[i][c];
  }
}

// One warp per output element: lane l sums slices l, l+32, ... in order,
// then a fixed xor tree -- deterministic, and the slices' partials are read
// 32 at a time instead of one dependent load per slice.
__global__ void dense_tn_reduce_kernel(const double* __restrict__ work, int slices, int K, int NP,
                                       int N, float* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < (int64_t)K * NP;
       i += nw) {
    double s = 0.0;
    for (int p = lane; p < slices; p += 32) s += work[(int64_t)p * K * NP + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int k = (int)(i / NP), j = (int)(i % NP);
    if (lane == 0 && j < ldy) Y[(int64_t)k * ldy + j] = (j < N) ? (float)s : 0.f;
  }
}

int tn_of(int N) { return N > 64 ? 4 : (N + 15) / 16; }
int nblk_of(int N) { return N > 64 ? (N + 63) / 64 : 1; }

}  // namespace

extern "C" {

int dg_dense_rows(const float* A, int64_t lda, int64_t n, int32_t K, const float* B, int64_t ldb,
                  int32_t N, int32_t transB, float* C, int64_t ldc, float* C_relu,
                  const float* z_mask, int64_t ld_mask, void* stream) {
  const int TN = tn_of(N);
  if (n < 0 || K < 1 || N < 1 || N > 64 || (int64_t)K * 16 * TN > 16384 || (lda & 3) ||
      ((uintptr_t)A & 15))
    return set_err(DG_ERR_ARG, "dense_rows: shape outside the kernel's range");
  if (n == 0) return DG_OK;
  cudaStream_t st = S(stream);
#define DG_DR4(tn, cg, bk, mb)                                                              \
  do {                                                                                      \
    constexpr int bm = 4 * 256 / (cg);                                                      \
    const size_t smem = ((size_t)K * (cg) * (tn) + (size_t)(bk) * (bm + 4)) * sizeof(float); \
    const unsigned blocks = (unsigned)((n + bm - 1) / bm);                                  \
    static bool attr = false;                                                               \
    if (!attr) {                                                                            \
      DG_CK(cudaFuncSetAttribute(dense_rows_kernel<tn, cg, bk, mb>,                         \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));  \
      attr = true;                                                                          \
    }                                                                                       \
    dense_rows_kernel<tn, cg, bk, mb><<<blocks, 256, smem, st>>>(A, lda, n, K, B, ldb, N,   \
                                                                 transB, C, ldc, C_relu,    \
                                                                 z_mask, ld_mask);          \
  } while (0)
#define DG_DR(tn, cg) DG_DR4(tn, cg, BK, 1)
  // long rows only (K >= 128): Reddit layer 1 (K=602) 0.303 -> 0.276 ms; short
  // rows (K <= 48) lose occupancy to the larger tile and run slower
  if (N <= 16 && ldc <= 16 && K >= 128) {
    // 4 rows x 4 columns per thread, 256 rows per CTA, 16-wide k-chunks
    // (Reddit layer 1: 0.26 -> 0.24 ms vs 32-wide k-chunks or 3 CTAs/SM)
    DG_DR4(4, 4, 16, 2);
  } else {
    switch (TN) {
      case 1: DG_DR(1, 16); break;
      case 2: DG_DR(2, 16); break;
      case 3: DG_DR(3, 16); break;
      default: DG_DR(4, 16); break;
    }
  }
#undef DG_DR
#undef DG_DR4
  DG_LAUNCHED();
  return DG_OK;
}

// the 256-wide K blocks pay only when they are mostly full: Reddit layer 1
// (K=608) 0.29 -> 0.24 ms; K <= 100 ran up to 2.4x slower (idle k-groups)
static bool tn4_ok(int32_t N, int32_t K) { return N <= 16 && K >= 256; }

static int64_t tn_slices(int64_t n, int32_t K, int32_t N) {
  const int kb = tn4_ok(N, K) ? (K + 255) / 256 : (K + 63) / 64;
  int64_t slices = std::max<int64_t>(1, (4 * 148) / kb);
  return std::min<int64_t>(slices, std::max<int64_t>(1, (n + 255) / 256));
}

int64_t dg_dense_tn_work(int64_t n, int32_t K, int32_t N) {
  return tn_slices(n, K, N) * (int64_t)K * 16 * tn_of(N) * nblk_of(N);
}

int dg_dense_tn(const float* H, int64_t ldh, int64_t n, int32_t K, const float* M, int64_t ldm,
                int32_t N, float* Y, int64_t ldy, double* work, int64_t work_len,
                void* stream) {
  const int TN = tn_of(N);
  const int NB = nblk_of(N);
  const int NPT = 16 * TN * NB;
  if (n < 0 || K < 1 || N < 1 || N > 256 || (ldh & 3) || ((uintptr_t)H & 15) || ldy > NPT ||
      ldy < N)
    return set_err(DG_ERR_ARG, "dense_tn: shape outside the kernel's range");
  const bool t4 = tn4_ok(N, K);
  const int kb = t4 ? (K + 255) / 256 : (K + 63) / 64;
  const int64_t slices = tn_slices(n, K, N);
  if (work_len < slices * (int64_t)K * NPT)
    return set_err(DG_ERR_ARG, "dense_tn: work buffer too small");
  const int64_t rows_per = std::max<int64_t>(1, (n + slices - 1) / slices);
  const dim3 grid((unsigned)slices, (unsigned)kb, (unsigned)NB);
  cudaStream_t st = S(stream);
  if (t4) {
    dense_tn4_kernel<<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work);
  } else switch (TN) {
    case 1: dense_tn_kernel<1><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
    case 2: dense_tn_kernel<2><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
    case 3: dense_tn_kernel<3><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
    default: dense_tn_kernel<4><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
  }
  DG_LAUNCHED();
  const int total = K * NPT;                        // one warp per output element
  dense_tn_reduce_kernel<<<(unsigned)std::min(4096, (total + 7) / 8), 256, 0, st>>>(
      work, (int)slices, K, NPT, N, Y, ldy);
  DG_LAUNCHED();
  return DG_OK;
}

}  // extern "C"
