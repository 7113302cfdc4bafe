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
#include "tma.cuh"

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

// TMA-fed form of dense_rows (the default for N <= 64).  Persistent CTAs,
// one producer warp + 8 consumer warps.  The producer streams 128-row x
// 32-column tiles of A (16 KB, 128-byte swizzle) into a 4-deep shared-memory
// ring with cp.async.bulk.tensor (mbarrier completion): 64 KB of A in
// flight per CTA without a register held, which the register-staged kernel
// above could not reach (ncu: 24% warps active, ~36% of HBM).  B (K x NP)
// sits in shared memory for the whole kernel.  Consumer thread tile: rows
// rg and rg + 64 of the 128-row tile x NP/4 columns; per k-quad two
// swizzled 16-B A loads (8 consecutive rows hit 8 distinct bank groups)
// and NP/16 16-B B loads (broadcast) feed 2 * NP FMAs.
constexpr int TR_BM = 128;          // rows per tile
constexpr int TR_BK = 32;           // columns per stage (one 128-byte swizzle span)
constexpr int TR_STAGES = 4;
constexpr int TR_STAGE_BYTES = TR_BM * TR_BK * 4;
// rows per consumer thread for N <= 16: 4 rows x 4 columns (4 consumer
// warps) read 8 shared-memory vectors per 64 FMAs instead of 6 per 32 -- the
// kernel was bound by shared-memory wavefronts (ncu: MIO throttle); K=602
// 0.191 -> 0.145 ms, K=100 0.382 -> 0.289 ms
#ifndef DG_TR_RPT16
#define DG_TR_RPT16 4
#endif

template <int NP, int RPT>
__global__ void __launch_bounds__(32 * (TR_BM * 4 / RPT / 32 + 1), 2) dense_rows_tma_kernel(
    const __grid_constant__ CUtensorMap amap, int64_t n, int K, const float* __restrict__ B,
    int64_t ldb, int N, int transB, float* __restrict__ C, int64_t ldc,
    float* __restrict__ Crelu, const float* __restrict__ Zmask, int64_t ldm) {
  constexpr int TN = NP / 4;                         // columns per thread
  constexpr int RSPAN = TR_BM / RPT;                 // row stride between a thread's rows
  constexpr int CW = RSPAN * 4 / 32;                 // consumer warps
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B alignment of the ring (128-byte swizzle atoms), computed in the
  // shared window and applied as an offset to the shared array -- an integer
  // round trip of the pointer would turn every ring / B read into a generic
  // load (ncu: LG-throttle and L1TEX stalls, 0.22 ms at K=602)
  const uint32_t s0 = smem_u32(smem_raw);
  unsigned char* base = smem_raw + (((s0 + 1023u) & ~1023u) - s0);
  unsigned char* ring = base;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + TR_STAGES * TR_STAGE_BYTES);
  uint64_t* empty = full + TR_STAGES;
  float* Bs = reinterpret_cast<float*>(empty + TR_STAGES);   // K_pad x NP
  const int nk = (K + TR_BK - 1) / TR_BK;
  const int tid = threadIdx.x;
  for (int i = tid; i < nk * TR_BK * NP; i += blockDim.x) {
    const int k = i / NP, j = i % NP;
    float b = 0.f;
    if (k < K && j < N) b = transB ? B[(int64_t)j * ldb + k] : B[(int64_t)k * ldb + j];
    Bs[i] = b;
  }
  if (tid == 0) {
    for (int s = 0; s < TR_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t ntiles = (n + TR_BM - 1) / TR_BM;
  const int warp = tid >> 5, lane = tid & 31;
  if (warp == CW) {                                  // producer
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int slot = (int)(it % TR_STAGES);
          if (it >= TR_STAGES) mbar_wait(&empty[slot], (uint32_t)(((it / TR_STAGES) - 1) & 1));
          mbar_arrive_expect_tx(&full[slot], TR_STAGE_BYTES);
          tma_load_2d(ring + (size_t)slot * TR_STAGE_BYTES, &amap, &full[slot], kc * TR_BK,
                      (int32_t)(t * TR_BM));
        }
    }
    return;
  }
  const int cg = tid & 3;                            // columns cg*TN .. cg*TN+TN-1
  const int rg = tid >> 2;                           // rows rg + RSPAN r of the tile
  int64_t it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    float acc[RPT][TN];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[r][c] = 0.f;
    for (int kc = 0; kc < nk; ++kc, ++it) {
      const int slot = (int)(it % TR_STAGES);
      mbar_wait(&full[slot], (uint32_t)((it / TR_STAGES) & 1));
      const unsigned char* st = ring + (size_t)slot * TR_STAGE_BYTES;
      const float* bk = Bs + (size_t)kc * TR_BK * NP + cg * TN;
#pragma unroll
      for (int q = 0; q < TR_BK / 4; ++q) {
        float4 a[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int row = rg + RSPAN * r;
          a[r] = *reinterpret_cast<const float4*>(st + row * 128 + ((q ^ (row & 7)) << 4));
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          float b[TN];
#pragma unroll
          for (int c4 = 0; c4 < TN / 4; ++c4) {
            const float4 v = *reinterpret_cast<const float4*>(bk + (4 * q + kk) * NP + 4 * c4);
            b[4 * c4] = v.x;
            b[4 * c4 + 1] = v.y;
            b[4 * c4 + 2] = v.z;
            b[4 * c4 + 3] = v.w;
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const float ar = kk == 0 ? a[r].x : kk == 1 ? a[r].y : kk == 2 ? a[r].z : a[r].w;
#pragma unroll
            for (int c = 0; c < TN; ++c) acc[r][c] = fmaf(ar, b[c], acc[r][c]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int64_t gr = t * TR_BM + rg + RSPAN * r;
      if (gr >= n) continue;
#pragma unroll
      for (int c4 = 0; c4 < TN / 4; ++c4) {
        const int j = cg * TN + 4 * c4;
        if (j >= ldc) continue;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = acc[r][4 * c4 + e];
          if (Zmask && j + e < N && !(Zmask[gr * ldm + j + e] > 0.f)) v[e] = 0.f;
        }
        *reinterpret_cast<float4*>(C + gr * ldc + j) = make_float4(v[0], v[1], v[2], v[3]);
        if (Crelu)
          *reinterpret_cast<float4*>(Crelu + gr * ldc + j) =
              make_float4(fmaxf(v[0], 0.f), fmaxf(v[1], 0.f), fmaxf(v[2], 0.f), fmaxf(v[3], 0.f));
      }
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

// TMA-fed form of dense_tn (the default for N <= 64).  CTA (slice, K block):
// a producer lane streams RC-row tiles of H (KB columns from k0) and of M
// (NP columns) into a 3-deep shared-memory ring; consumer thread (kq, nq, rs)
// owns the 4 x 4 outputs k0+4kq.., 4nq.. over rows rs, rs+RS, ... of every
// tile (fp32 per tile, folded into fp64), then the RS row subsets are summed
// in fixed order through shared memory -- deterministic, like the slice sum
// that follows.
constexpr int TT_STAGES = 3;

struct TnGeom {
  int KB, NP, RC, RS;
};

__global__ void __launch_bounds__(288, 2) dense_tn_tma_kernel(
    const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap mmap,
    int K, const TnGeom g, int64_t rows_per, int64_t n, double* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int KB = g.KB, NP = g.NP, RC = g.RC, RS = g.RS;
  const int hfl = RC * KB, mfl = RC * NP;              // floats per stage
  float* ring = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)TT_STAGES * (hfl + mfl));
  uint64_t* empty = full + TT_STAGES;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < TT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int k0 = blockIdx.y * KB;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per;
  const int64_t r_end = min(n, r_begin + rows_per);
  const int64_t nst = r_end > r_begin ? (r_end - r_begin + RC - 1) / RC : 0;
  const int warp = tid >> 5, lane = tid & 31;
  if (warp == 8) {
    if (lane == 0) {
      for (int64_t s = 0; s < nst; ++s) {
        const int slot = (int)(s % TT_STAGES);
        if (s >= TT_STAGES) mbar_wait(&empty[slot], (uint32_t)(((s / TT_STAGES) - 1) & 1));
        mbar_arrive_expect_tx(&full[slot], (uint32_t)(hfl + mfl) * 4);
        float* st = ring + (size_t)slot * (hfl + mfl);
        const int32_t r0 = (int32_t)(r_begin + s * RC);
        tma_load_2d(st, &hmap, &full[slot], k0, r0);
        tma_load_2d(st + hfl, &mmap, &full[slot], 0, r0);
      }
    }
    return;
  }
  const int nkq = KB / 4, nnq = NP / 4;
  const int kq = tid % nkq, nq = (tid / nkq) % nnq, rs = tid / (nkq * nnq);
  const bool active = rs < RS;
  float part[4][4];
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      part[i][c] = 0.f;
      acc[i][c] = 0.0;
    }
  for (int64_t s = 0; s < nst; ++s) {
    const int slot = (int)(s % TT_STAGES);
    mbar_wait(&full[slot], (uint32_t)((s / TT_STAGES) & 1));
    const float* hs = ring + (size_t)slot * (hfl + mfl);
    const float* ms = hs + hfl;
    if (active) {
      // pointer walk with fixed strides (ncu: the indexed form spent 2.3
      // issued instructions per FMA on address arithmetic at K=602)
      const float4* hp = reinterpret_cast<const float4*>(hs + rs * KB + 4 * kq);
      const float4* mp = reinterpret_cast<const float4*>(ms + rs * NP + 4 * nq);
      const int hstep = RS * KB / 4, mstep = RS * NP / 4;
      const int cnt = (RC - rs + RS - 1) / RS;
#pragma unroll 4
      for (int i = 0; i < cnt; ++i) {
        const float4 h = *hp;
        const float4 m = *mp;
        hp += hstep;
        mp += mstep;
        const float hh[4] = {h.x, h.y, h.z, h.w};
        const float mm[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) part[a][c] = fmaf(hh[a], mm[c], part[a][c]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[i][c] += (double)part[i][c];
          part[i][c] = 0.f;
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  // sum the RS row subsets in order (ring reused once every stage is consumed)
  asm volatile("bar.sync 1, 256;" ::: "memory");
  double* red = reinterpret_cast<double*>(ring);       // [RS][KB][NP]
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        red[((size_t)rs * KB + 4 * kq + i) * NP + 4 * nq + c] = acc[i][c];
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  double* wp = work + (size_t)blockIdx.x * K * NP;
  for (int e = tid; e < KB * NP; e += 256) {
    const int k = k0 + e / NP;
    if (k >= K) continue;
    double v = 0.0;
    for (int r = 0; r < RS; ++r) v += red[(size_t)r * KB * NP + e];
    wp[(size_t)k * NP + e % NP] = v;
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

// 1: the register-staged kernels only (A/B comparison in scripts/dense_probe.py)
int dg_dense_legacy = 0;

int dg_dense_rows(const float* A, int64_t lda, int64_t n, int32_t K, const float* B, int64_t ldb,
                  int32_t N, int32_t transB, float* C, int64_t ldc, float* C_relu,
                  const float* z_mask, int64_t ld_mask, void* stream) {
  const int TN = tn_of(N);
  if (n < 0 || K < 1 || N < 1 || N > 64 || (int64_t)K * 16 * TN > 16384 || (lda & 3) ||
      ((uintptr_t)A & 15))
    return set_err(DG_ERR_ARG, "dense_rows: shape outside the kernel's range");
  if (n == 0) return DG_OK;
  cudaStream_t st = S(stream);
  // TMA-fed kernel: N <= 64, 16-B aligned row pitches (ldc: vector stores)
  if (!dg_dense_legacy && (ldc & 3) == 0 && ((uintptr_t)C & 15) == 0 &&
      (!C_relu || ((uintptr_t)C_relu & 15) == 0)) {
    const int NP = (N + 15) / 16 * 16;
    const int nk = (K + TR_BK - 1) / TR_BK;
    if (ldc <= NP && (size_t)nk * TR_BK * NP * 4 <= 64 * 1024) {
      CUtensorMap amap;
      int rc = dg::make_tensor_map_2d_swz128(&amap, A, n, lda, K, TR_BK, TR_BM);
      if (rc) return rc;
      const size_t smem = 1024 + (size_t)TR_STAGES * TR_STAGE_BYTES + 2 * TR_STAGES * 8 +
                          (size_t)nk * TR_BK * NP * 4;
      const int64_t ntiles = (n + TR_BM - 1) / TR_BM;
      const unsigned grid = (unsigned)std::min<int64_t>(ntiles, 2 * 148);
#define DG_TR(np, rpt)                                                                      \
  do {                                                                                      \
    static bool attr = false;                                                               \
    if (!attr) {                                                                            \
      DG_CK(cudaFuncSetAttribute(dense_rows_tma_kernel<np, rpt>,                            \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024)); \
      attr = true;                                                                          \
    }                                                                                       \
    dense_rows_tma_kernel<np, rpt><<<grid, 32 * (TR_BM * 4 / rpt / 32 + 1), smem, st>>>(    \
        amap, n, K, B, ldb, N, transB, C, ldc, C_relu, z_mask, ld_mask);                    \
  } while (0)
      // 4 rows per thread pay when the k loop dominates (K >= 64); short
      // loops are bound by the epilogue (ReLU mask loads, stores) and want
      // more threads: products M W^T with K=47 0.24 -> 0.30 ms at 4 rows
      switch (NP) {
        case 16:
          if (K >= 64) DG_TR(16, DG_TR_RPT16);
          else DG_TR(16, 2);
          break;
        case 32: DG_TR(32, 2); break;
        case 48: DG_TR(48, 2); break;
        default: DG_TR(64, 2); break;
      }
#undef DG_TR
      DG_LAUNCHED();
      return DG_OK;
    }
  }
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

// geometry of the TMA-fed dense_tn: K blocks of <= 256 columns, rows per
// stage sized for ~32 KB of H + M, RS row subsets filling 256 threads
static bool tn_tma_geom(int32_t K, int32_t N, TnGeom* g, int* kblocks) {
  if (N > 64 || K % 4) return false;
  g->NP = (N + 15) / 16 * 16;
  g->KB = K <= 256 ? K : 256;
  *kblocks = (K + g->KB - 1) / g->KB;
  const int per_row = g->KB + g->NP;
  int rc = 32768 / (per_row * 4);
  rc = std::max(8, std::min(256, rc / 8 * 8));
  g->RC = rc;
  const int th = (g->KB / 4) * (g->NP / 4);
  if (th > 256) return false;
  g->RS = std::max(1, std::min(256 / th, rc));
  return true;
}

// one wave at 2 CTAs per SM (K=602: 0.226 -> 0.215 ms against two waves)
static int64_t tn_tma_slices(int64_t n, int kblocks, int RC) {
  const int64_t want = std::max<int64_t>(1, (2 * 148) / kblocks);
  return std::max<int64_t>(1, std::min<int64_t>(want, (n + RC - 1) / RC));
}

static int64_t tn_slices(int64_t n, int32_t K, int32_t N) {
  const int kb = tn4_ok(N, K) ? (K + 255) / 256 : (K + 63) / 64;
  int64_t slices = std::max<int64_t>(1, (4 * 148) / kb);
  return std::min<int64_t>(slices, std::max<int64_t>(1, (n + 255) / 256));
}

int64_t dg_dense_tn_work(int64_t n, int32_t K, int32_t N) {
  TnGeom g;
  int kb;
  const int64_t legacy = tn_slices(n, K, N) * (int64_t)K * 16 * tn_of(N) * nblk_of(N);
  if (!tn_tma_geom(K, N, &g, &kb)) return legacy;
  return std::max(legacy, tn_tma_slices(n, kb, g.RC) * (int64_t)K * g.NP);
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
  cudaStream_t st0 = S(stream);
  TnGeom g;
  int kbt;
  if (!dg_dense_legacy && tn_tma_geom(K, N, &g, &kbt) && (ldm & 3) == 0 &&
      ((uintptr_t)M & 15) == 0 && ldy <= g.NP) {
    const int64_t slices = tn_tma_slices(n, kbt, g.RC);
    if (work_len < slices * (int64_t)K * g.NP)
      return set_err(DG_ERR_ARG, "dense_tn: work buffer too small");
    int64_t rows_per = (n + slices - 1) / slices;
    rows_per = (rows_per + g.RC - 1) / g.RC * g.RC;          // whole stages per slice
    CUtensorMap hmap, mmap;
    int rc = dg::make_tensor_map_2d(&hmap, H, n, ldh, K, g.KB, g.RC, true);
    if (rc) return rc;
    rc = dg::make_tensor_map_2d(&mmap, M, n, ldm, N, g.NP, g.RC, true);
    if (rc) return rc;
    const size_t ring = (size_t)TT_STAGES * g.RC * (g.KB + g.NP) * 4;
    const size_t red = (size_t)g.RS * g.KB * g.NP * 8;
    const size_t smem = std::max(ring, red) + 2 * TT_STAGES * 8 + 16;
    static bool attr = false;
    if (!attr) {
      DG_CK(cudaFuncSetAttribute(dense_tn_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024));
      attr = true;
    }
    if (smem > 200 * 1024) return set_err(DG_ERR_ARG, "dense_tn: shared memory");
    dense_tn_tma_kernel<<<dim3((unsigned)slices, (unsigned)kbt), 288, smem, st0>>>(
        hmap, mmap, K, g, rows_per, n, work);
    DG_LAUNCHED();
    const int total = K * g.NP;
    dense_tn_reduce_kernel<<<(unsigned)std::min(4096, (total + 7) / 8), 256, 0, st0>>>(
        work, (int)slices, K, g.NP, N, Y, ldy);
    DG_LAUNCHED();
    return DG_OK;
  }
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
