// gcn.cu -- GCN step pieces: masked softmax cross-entropy, ReLU, ReLU
// gradient mask, SGD.

#include <cmath>

#include "common.cuh"

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

// Masked softmax cross-entropy (gcn.py:98-120).  One warp per row in a
// grid-stride loop over a fixed grid (<= 4 CTAs per SM), so the cross-CTA
// reduction touches one counter a few hundred times, not once per 8 rows.
// Loss / correct sums are deterministic: each warp sums its rows in order,
// each CTA its warps in order, the last CTA the CTA partials in order.
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
  double loss = 0.0, corr = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + w; row < n; row += (int64_t)gridDim.x * 8) {
    const float* xr = x + row * ld;
    float m = -INFINITY;
    for (int j = lane; j < C; j += 32) m = fmaxf(m, xr[j]);
    m = warp_max(m);
    double s = 0.0;
    for (int j = lane; j < C; j += 32) s += (double)expf(xr[j] - m);
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
    const double inv_s = 1.0 / s;
    for (int j = lane; j < C; j += 32) {
      float gv = 0.f;
      if (on) {
        double sm = (double)expf(xr[j] - m) * inv_s;
        if (j == lbl) sm -= 1.0;
        gv = (float)(sm / denom);
      }
      gr[j] = gv;
    }
    for (int j = C + lane; j < ldg; j += 32) gr[j] = 0.f;
    if (on) {
      loss += log(s) - ((double)xr[lbl] - (double)m);
      corr += (am == lbl) ? 1.0 : 0.0;
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
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    double l = 0.0, c = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      l += ((volatile double*)scratch)[2 * b];
      c += ((volatile double*)scratch)[2 * b + 1];
    }
    out[0] += l;
    out[1] += c;
    *counter = 0u;
  }
}

template <int G>
__device__ __forceinline__ float grp_max(float v) {
#pragma unroll
  for (int o = G / 2; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, G));
  return v;
}
template <int G>
__device__ __forceinline__ double grp_sum(double v) {
#pragma unroll
  for (int o = G / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}
template <int G>
__device__ __forceinline__ float grp_sumf(float v) {
#pragma unroll
  for (int o = G / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}
template <int G>
__device__ __forceinline__ int grp_min(int v) {
#pragma unroll
  for (int o = G / 2; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o, G));
  return v;
}

// Vectorised variant for C <= 4*G*K: a group of G lanes owns a row, lane l
// holds float4 chunks l, l+G, ... in registers (one pass over the row, one
// expf per element).  Same numerics and deterministic reduction order as
// xent_kernel (rows in order per group, groups in order per CTA, CTAs in
// order in the last CTA).
// 3 CTAs/SM for rows <= 256 classes (C=172: 20.9 -> 17.5 ms at 27.8M rows).
template <int G, int K>
__global__ void __launch_bounds__(256, (K <= 2 ? 3 : 2)) xent_vec_kernel(
    const float* __restrict__ x, int64_t n, int C, int64_t ld, const int64_t* __restrict__ labels,
    const uint8_t* __restrict__ mask, double denom, float* __restrict__ grad, int64_t ldg,
    double* scratch, unsigned* counter, double* out) {
  constexpr int GPW = 32 / G;                        // groups per warp
  constexpr int RPB = 256 / G;                       // groups per CTA
  constexpr int RU = 4;                              // rows per group per step (loads batched)
  __shared__ double s_loss[RPB];
  __shared__ double s_corr[RPB];
  __shared__ bool s_last;
  const int lig = threadIdx.x & (G - 1);
  const int grp = threadIdx.x / G;
  double loss = 0.0, corr = 0.0;
  const int nchunk = (C + 3) / 4;
  const int gchunk = (int)(ldg / 4);
  // warp-uniform trip count: the groups of a warp share the loop (their
  // shuffles use the full-warp mask); rows past the end run predicated.
  // A warp covers RU consecutive blocks of GPW rows per step.
  const int warp = threadIdx.x >> 5;
  const int64_t step = (int64_t)gridDim.x * (256 / 32) * GPW * RU;
  for (int64_t base = ((int64_t)blockIdx.x * (256 / 32) + warp) * GPW * RU; base < n;
       base += step) {
    float v[RU][K][4];
    int64_t rowu[RU];
    bool valid[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {                   // all loads first
      const int64_t rr = base + u * GPW + (grp % GPW);
      valid[u] = rr < n;
      rowu[u] = valid[u] ? rr : n - 1;
      const float4* xr = reinterpret_cast<const float4*>(x + rowu[u] * ld);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lig + k * G;
        float4 t = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (c < nchunk) t = xr[c];
        v[u][k][0] = t.x;
        v[u][k][1] = (4 * c + 1 < C) ? t.y : -INFINITY;
        v[u][k][2] = (4 * c + 2 < C) ? t.z : -INFINITY;
        v[u][k][3] = (4 * c + 3 < C) ? t.w : -INFINITY;
      }
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int64_t row = rowu[u];
      float m = -INFINITY;
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) m = fmaxf(m, v[u][k][e]);
      m = grp_max<G>(m);
      const int64_t lbl = labels[row];
      const bool lin = lbl >= 0 && lbl < C;
      // the label's logit straight from memory (an L1 hit: the row was just
      // loaded) instead of a compare-and-select per element
      const float xv = lin ? x[row * ld + lbl] : 0.f;
      // the exponentials (each in (0, 1]) summed in fp32: a lane's <= 4K
      // terms, then a fixed xor tree over the G lanes (<= (4K + log2 G) ulp).
      // Columns past C hold -inf (see the loads), so they add exp(-inf) = 0
      // and never equal the maximum of a row with a finite entry: no
      // per-element class test.  argmax: the lane's first maximal element,
      // tracked as an offset (4kG + e) so the select takes an immediate
      float sl = 0.f;
      int a = 4 * K * G;
#pragma unroll
      for (int k = K - 1; k >= 0; --k)
#pragma unroll
        for (int e = 3; e >= 0; --e)
          if (v[u][k][e] == m) a = 4 * k * G + e;
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[u][k][e] = expf(v[u][k][e] - m);
          sl += v[u][k][e];
        }
      const double s = (double)grp_sumf<G>(sl);
      const double xl = (double)xv - (double)m;
      int am = (a == 4 * K * G) ? C : min(4 * lig + a, C);
      am = grp_min<G>(am);
      const bool on = valid[u] && mask[row] != 0;
      // (softmax - onehot) / denom with one division per row: p_j/denom =
      // e_j * (1 / (s * denom)); the label term subtracts 1/denom.  The
      // fp64 division (and the loss's fp64 log below) run on the group's
      // first lane only and the scale is broadcast: 16-lane groups (C=47)
      // otherwise spend most of the kernel in redundant fp64 math
      double scale_l = 0.0;
      if (lig == 0) scale_l = 1.0 / (s * denom);
      const double scale =
          __shfl_sync(0xffffffffu, scale_l, (threadIdx.x & 31) & ~(G - 1));
      const float scale_f = (float)scale;
      float4* gr = reinterpret_cast<float4*>(grad + row * ldg);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lig + k * G;
        if (valid[u] && c < gchunk) {
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)   // fp32 product (<= 1.5 ulp)
            o[e] = (on && 4 * c + e < C) ? v[u][k][e] * scale_f : 0.f;
          gr[c] = make_float4(o[0], o[1], o[2], o[3]);
        }
      }
      if (valid[u])
        for (int c = lig + K * G; c < gchunk; c += G) gr[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      // the label entry, where p - 1 may cancel, in fp64; rewritten by the
      // lane that stored its float4 (same-thread order: the later store wins)
      if (on && lin && (int)(lbl >> 2) % G == lig) {
        const float el = expf(xv - m);
        grad[row * ldg + lbl] = (float)((double)el * scale - 1.0 / denom);
      }
      if (on && lig == 0) {
        loss += log(s) - xl;
        corr += (am == lbl) ? 1.0 : 0.0;
      }
    }
  }
  if (lig == 0) {
    s_loss[grp] = loss;
    s_corr[grp] = corr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0, c = 0.0;
    for (int i = 0; i < RPB; ++i) {
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
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    double l = 0.0, c = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      l += ((volatile double*)scratch)[2 * b];
      c += ((volatile double*)scratch)[2 * b + 1];
    }
    out[0] += l;
    out[1] += c;
    *counter = 0u;
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
  const bool vec = ld % 4 == 0 && ld_grad % 4 == 0 && (((uintptr_t)logits | (uintptr_t)grad) & 15) == 0;
  const int nchunk = (C + 3) / 4;
  // lanes per row: the narrowest power of two that keeps <= 4 float4 chunks
  // per lane -- fewer lanes per row means fewer shuffle steps and fewer
  // redundant per-row instructions (C=47: 16 lanes x 1 chunk was issue-bound
  // at 447M warp instructions, ncu profiles/r02; 4 lanes x 3 chunks)
  int G = 1;
  while (G * 4 < nchunk && G < 32) G <<= 1;
  const int K = (nchunk + G - 1) / G;
  if (vec && K <= 4) {
    const int rpb = (256 / G) * 4;                   // rows per CTA step (RU = 4)
    const unsigned blocks = (unsigned)std::min<int64_t>((n + rpb - 1) / rpb, 12 * 148);
    cudaStream_t st = S(stream);
#define DG_XV(g, k) xent_vec_kernel<g, k><<<blocks, 256, 0, st>>>(logits, n, C, ld, labels, mask, \
                                                                  denom, grad, ld_grad, scratch, \
                                                                  counter, stats_out)
#define DG_XVK(g)                 \
  switch (K) {                    \
    case 1: DG_XV(g, 1); break;   \
    case 2: DG_XV(g, 2); break;   \
    case 3: DG_XV(g, 3); break;   \
    default: DG_XV(g, 4); break;  \
  }
    switch (G) {
      case 1: DG_XVK(1); break;
      case 2: DG_XVK(2); break;
      case 4: DG_XVK(4); break;
      case 8: DG_XVK(8); break;
      case 16: DG_XVK(16); break;
      default: DG_XVK(32); break;
    }
#undef DG_XVK
#undef DG_XV
  } else {
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 7) / 8, 4 * 148);
    xent_kernel<<<blocks, 256, 0, S(stream)>>>(logits, n, C, ld, labels, mask, denom, grad,
                                               ld_grad, scratch, counter, stats_out);
  }
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
