// dense.cu -- the GCN's dense transforms, tall-skinny and memory-bound:
//
//   forward   Z = T W            gcn.py:274  (T: n x K, W: K x N, N <= 256)
//             H = relu(Z)        gcn.py:276  (fused epilogue, optional)
//   backward  G = (M W^T) * 1[Zprev > 0]     gcn.py:282  (fused mask, optional)
//   wgrad     Y = H^T M          gcn.py:280  (K x N, reduction over the n rows)
//
// fp32 SIMT (TF32 would break the fp32 parity contract); these shapes are
// HBM-bound (T or H is read once: 566 MB for Reddit layer 1), so the target
// is streaming the tall operand at HBM speed, not tensor-core FLOPs.
//
// dg_dense_rows: thread = one row x 16 output columns, A staged through
// shared memory once per chunk (see dense_rw_kernel); any N up to 256.
//
// dg_dense_tn: grid = (row slices, 64-wide K blocks); each CTA accumulates
// its slice's partial H^T M (fp32 per 64-row chunk, folded into fp64) and
// writes it to `work`; a second kernel sums the partials in slice order
// (fp64) -- deterministic, unlike split-K with atomics.

#include "common.cuh"

namespace {

// Row-wise form (dg_dense_rows): thread = (one row, NT consecutive output
// columns); a CTA covers RB = 256 / NC rows x all NC column chunks.  A is
// staged through shared memory in KC-wide chunks with coalesced float4 loads
// (the next chunk in flight in registers) and each thread reads its own
// row's values once per chunk (one LDS.128 per 4 k); B (K x NP, zero padded)
// sits in shared memory and is read as broadcast float4s.  Every A element
// crosses shared memory twice (store + one read per column chunk), so the
// kernel streams A at HBM speed instead of being shared-memory bound.
constexpr int KC = 32;   // k-chunk of the row-wise kernel

template <int NT>
__global__ void __launch_bounds__(256) dense_rw_kernel(
    const float* __restrict__ A, int64_t lda, int64_t n, int K, const float* __restrict__ B,
    int64_t ldb, int N, int transB, float* __restrict__ C, int64_t ldc,
    float* __restrict__ Crelu, const float* __restrict__ Zmask, int64_t ldm, int NC) {
  extern __shared__ __align__(16) float smem[];
  const int RB = 256 / NC;                           // rows per CTA
  const int NP = NC * NT;                            // padded output width
  const int Kp = (K + 3) & ~3;
  float* Bs = smem;                                  // Kp x NP
  float* As = smem + (size_t)Kp * NP;                // RB x (KC + 4)
  const int tid = threadIdx.x;
  for (int i = tid; i < Kp * NP; i += 256) {
    const int k = i / NP, j = i % NP;
    float b = 0.f;
    if (k < K && j < N) b = transB ? B[(int64_t)j * ldb + k] : B[(int64_t)k * ldb + j];
    Bs[i] = b;
  }
  const int r = tid / NC, c = tid % NC;
  const int64_t row0 = (int64_t)blockIdx.x * RB;
  const int per = (RB * (KC / 4) + 255) / 256;       // float4 per thread per chunk (<= 8)
  float acc[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j] = 0.f;
  auto load_chunk = [&](int k0, float4* v) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u >= per) continue;
      const int i = tid + u * 256;
      const int rr = i / (KC / 4), q = i % (KC / 4);
      const int64_t gr = row0 + rr;
      const int k = k0 + 4 * q;
      if (rr < RB && gr < n && k < K) {
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
  float4 nxt[8];
  load_chunk(0, nxt);
  const float* arow = As + (size_t)r * (KC + 4);
  for (int k0 = 0; k0 < K; k0 += KC) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u >= per) continue;
      const int i = tid + u * 256;
      const int rr = i / (KC / 4), q = i % (KC / 4);
      if (rr < RB) *reinterpret_cast<float4*>(&As[(size_t)rr * (KC + 4) + 4 * q]) = nxt[u];
    }
    __syncthreads();
    if (k0 + KC < K) load_chunk(k0 + KC, nxt);       // in flight during the math
    const int kmax = min(KC, Kp - k0);
    if (r < RB) {
      for (int kk = 0; kk < kmax; kk += 4) {
        const float4 a = *reinterpret_cast<const float4*>(arow + kk);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4* bp = reinterpret_cast<const float4*>(Bs + (size_t)(k0 + kk + e) * NP +
                                                             c * NT);
#pragma unroll
          for (int j4 = 0; j4 < NT / 4; ++j4) {
            const float4 b = bp[j4];
            acc[4 * j4 + 0] = fmaf(av[e], b.x, acc[4 * j4 + 0]);
            acc[4 * j4 + 1] = fmaf(av[e], b.y, acc[4 * j4 + 1]);
            acc[4 * j4 + 2] = fmaf(av[e], b.z, acc[4 * j4 + 2]);
            acc[4 * j4 + 3] = fmaf(av[e], b.w, acc[4 * j4 + 3]);
          }
        }
      }
    }
  }
  const int64_t gr = row0 + r;
  if (r >= RB || gr >= n) return;
#pragma unroll
  for (int j4 = 0; j4 < NT / 4; ++j4) {
    const int j = c * NT + 4 * j4;
    if (j >= ldc) break;
    float o[4] = {acc[4 * j4], acc[4 * j4 + 1], acc[4 * j4 + 2], acc[4 * j4 + 3]};
    if (Zmask) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j + e < N && !(Zmask[gr * ldm + j + e] > 0.f)) o[e] = 0.f;
    }
    *reinterpret_cast<float4*>(C + gr * ldc + j) = make_float4(o[0], o[1], o[2], o[3]);
    if (Crelu)
      *reinterpret_cast<float4*>(Crelu + gr * ldc + j) =
          make_float4(fmaxf(o[0], 0.f), fmaxf(o[1], 0.f), fmaxf(o[2], 0.f), fmaxf(o[3], 0.f));
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

__global__ void dense_tn_reduce_kernel(const double* __restrict__ work, int slices, int K, int NP,
                                       int N, float* __restrict__ Y, int64_t ldy) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K * NP; i += gridDim.x * blockDim.x) {
    const int k = i / NP, j = i % NP;
    double s = 0.0;
    for (int p = 0; p < slices; ++p) s += work[(int64_t)p * K * NP + i];
    if (j < ldy) Y[(int64_t)k * ldy + j] = (j < N) ? (float)s : 0.f;
  }
}

int tn_of(int N) { return N > 64 ? 4 : (N + 15) / 16; }
int nblk_of(int N) { return N > 64 ? (N + 63) / 64 : 1; }

}  // namespace

extern "C" {

int dg_dense_rows(const float* A, int64_t lda, int64_t n, int32_t K, const float* B, int64_t ldb,
                  int32_t N, int32_t transB, float* C, int64_t ldc, float* C_relu,
                  const float* z_mask, int64_t ld_mask, void* stream) {
  // NT output columns per thread: 16 (4 float4) unless the row is narrower
  const int NT = ldc <= 4 ? 4 : (ldc <= 8 ? 8 : 16);
  const int NC = (int)((ldc + NT - 1) / NT);
  const int Kp = (K + 3) & ~3;
  if (n < 0 || K < 1 || N < 1 || N > ldc || (ldc & 3) || NC > 16 || (lda & 3) ||
      ((uintptr_t)A & 15) || ((uintptr_t)C & 15) || (C_relu && ((uintptr_t)C_relu & 15)))
    return set_err(DG_ERR_ARG, "dense_rows: shape outside the kernel's range");
  const int RB = 256 / NC;
  const size_t smem = ((size_t)Kp * NC * NT + (size_t)RB * (KC + 4)) * sizeof(float);
  if (smem > 200 * 1024) return set_err(DG_ERR_ARG, "dense_rows: B too large for shared memory");
  if (n == 0) return DG_OK;
  const unsigned blocks = (unsigned)((n + RB - 1) / RB);
  cudaStream_t st = S(stream);
#define DG_DR(nt)                                                                           \
  do {                                                                                      \
    static bool attr = false;                                                               \
    if (!attr) {                                                                            \
      DG_CK(cudaFuncSetAttribute(dense_rw_kernel<nt>,                                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
      attr = true;                                                                          \
    }                                                                                       \
    dense_rw_kernel<nt><<<blocks, 256, smem, st>>>(A, lda, n, K, B, ldb, N, transB, C, ldc, \
                                                   C_relu, z_mask, ld_mask, NC);            \
  } while (0)
  switch (NT) {
    case 4: DG_DR(4); break;
    case 8: DG_DR(8); break;
    default: DG_DR(16); break;
  }
#undef DG_DR
  DG_LAUNCHED();
  return DG_OK;
}

int64_t dg_dense_tn_work(int64_t n, int32_t K, int32_t N) {
  const int kb = (K + 63) / 64;
  int64_t slices = std::max<int64_t>(1, (4 * 148) / kb);
  slices = std::min<int64_t>(slices, std::max<int64_t>(1, (n + 255) / 256));
  return slices * (int64_t)K * 16 * tn_of(N) * nblk_of(N);
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
  const int kb = (K + 63) / 64;
  int64_t slices = std::max<int64_t>(1, (4 * 148) / kb);
  slices = std::min<int64_t>(slices, std::max<int64_t>(1, (n + 255) / 256));
  if (work_len < slices * (int64_t)K * NPT)
    return set_err(DG_ERR_ARG, "dense_tn: work buffer too small");
  const int64_t rows_per = std::max<int64_t>(1, (n + slices - 1) / slices);
  const dim3 grid((unsigned)slices, (unsigned)kb, (unsigned)NB);
  cudaStream_t st = S(stream);
  switch (TN) {
    case 1: dense_tn_kernel<1><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
    case 2: dense_tn_kernel<2><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
    case 3: dense_tn_kernel<3><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
    default: dense_tn_kernel<4><<<grid, 256, 0, st>>>(H, ldh, n, K, M, ldm, N, rows_per, work); break;
  }
  DG_LAUNCHED();
  const int total = K * NPT;
  dense_tn_reduce_kernel<<<(unsigned)std::min(1024, (total + 255) / 256), 256, 0, st>>>(
      work, (int)slices, K, NPT, N, Y, ldy);
  DG_LAUNCHED();
  return DG_OK;
}

}  // extern "C"
