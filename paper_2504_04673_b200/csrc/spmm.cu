// spmm.cu -- the local SpMM of every hosted rank (sm_100a).
//
// Replaces sparse.local_spmm (sparse.py:208-223) and the per-source-block
// loops of spmm._kernel_1d_* / _kernel_15d (spmm.py:172-227): one launch
// computes Z_r = A_r [H_r ; halo_r] for all ranks hosted by the process.
//
// Why this shape (DESIGN.md has the measurements):
//  * SpMM is gather-bound (<= f/4 flop per byte), not tensor-core work.
//    The limiter on B200 is memory-level parallelism: every nonzero needs
//    its (col, val) before its H row can be gathered, and the gathered rows
//    wait in registers, so rows in flight per SM = warps x entries per step.
//  * Entries are stored interleaved, 8 B per nonzero ({col, val}), each
//    work item starting 16-B aligned.
//  * A group of G lanes owns one item; lane l owns lane-chunks l, l+G, ...
//    of the current feature slab, so one H-row gather is a G x 16 B (128-bit
//    lanes) or G x 32 B (Blackwell 256-bit ld.global.nc.v8) contiguous
//    request.  Wide layers are split into slabs (grid.y) sized so one slab of
//    all gathered rows stays L2-resident; the CSR stream is evict-first.
//  * Two forms.  128-bit lanes (rows <= 48 floats): entries loaded with
//    uniform 16-B vector loads one step ahead, 8-entry fp32 windows folded
//    into fp64 accumulators.  acc = 2 with 256-bit lanes (rows > 48 floats,
//    and 9..16-float rows of tables far larger than L2): one chunk per lane, the item's
//    entries staged in shared memory by cp.async one window ahead (no
//    registers held by the prefetch), two-level fp32 sums (32-entry windows;
//    <= 64 ulp of the row's sum of |terms| per 1024-entry item), 2 entries per
//    step at 4 CTAs/SM with 64 registers.
//  * Summation follows CSR storage order; long rows are split at fixed
//    boundaries and the fp64 partials summed in chunk order.  Deterministic,
//    and identical for every variant (aware == oblivious, 1.5D c=1 == 1D).

#include "common.cuh"

#include <cstdlib>

#ifndef DG_SPMM_HUB_ROWS
// rows per rank kept in L1 by the wide (256-bit, staged) gathers, all other
// wide gathers bypass L1: f=602 17.41 -> 17.19 ms, products f=100 4.76 ->
// 4.62 ms (profiles/r02/r2_hub_*); 0 disables the flags
#define DG_SPMM_HUB_ROWS 512
#endif

namespace {

struct Item {          // 24 B: one row, or one fixed chunk of a long row
  int64_t lo;          // first entry (even: 16-B aligned)
  int32_t row;         // output row
  int32_t len;         // entries in this item
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
  const int4* ent;     // interleaved {col, val bits} pairs, two per int4
  const float* hl;     // own H block (ext < n_local)
  const float* hh;     // halo rows (ext >= n_local)
  float* z;
  float* hr;           // fused epilogue: relu(z) (nullable)
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
  int32_t beta;        // 1: z += result (boundary pass of an overlapped phase)
  // fused forward epilogue (FN > 0): z = (A H) W, hr = relu(z); W is f x n_out
  const float* w;
  int32_t ld_w;
  int32_t n_out;
};

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// CSR stream: read once per slab pass; keep it out of L1 and first in line
// for L2 eviction so the gathered H rows stay resident.
__device__ __forceinline__ int4 ld_stream(const int4* p, uint64_t pol) {
  int4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "l"(pol));
  return v;
}

// Occupancy vs in-flight loads (measured on B200, Reddit-shaped graph):
// one float4 chunk per lane -> 4 entries per step and >= 4 CTAs/SM (<= 64
// registers); wider lanes keep more registers and fewer CTAs (no spills).
template <int CPL, int V>
struct Tune {
  static constexpr int E = 4;                       // entries per pipeline step
  static constexpr int W = CPL * V / 4;             // float4s per lane
  // one 256-bit chunk per lane: 3 CTAs/SM (80 registers) -- more warps in
  // flight beat a 12-byte spill (sweep, profiles/r01/spmm_sweep_minb.txt:
  // f=602 24.4 -> 19.8 ms, f=100 4.8 -> 4.0 ms; 4 CTAs/SM spill 80 B: slower)
  static constexpr int MINB = W == 1 ? 4 : (CPL == 1 && V == 8 ? 3 : (W == 2 ? 2 : 1));
};

// V floats per lane-chunk: 4 -> 128-bit loads (LDG.128); 8 -> Blackwell's
// 256-bit loads (LDG.E.ENL2.256).  Measured with the gather probe (profiles/
// r01/gather_roofline.txt): random 256-B row gathers reach 18.4 TB/s with
// 256-bit loads vs 10.6 TB/s with 128-bit -- the 128-bit ceiling is the
// load-instruction rate, not L2 bandwidth.  V=8 needs 32-B aligned rows.
template <int V>
struct Vec;
template <>
struct Vec<4> {
  float v[4];
  __device__ __forceinline__ void load(const float* p) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  }
  // hub rows (flagged by the plan) stay in L1 (evict_last); every other
  // gathered row bypasses it (no_allocate) so the hubs are not evicted
  __device__ __forceinline__ void load_hint(const float* p, bool hub) {
    asm("{\n .reg .pred h;\n setp.ne.b32 h, %5, 0;\n"
        " @h ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];\n"
        " @!h ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n}"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
        : "l"(p), "r"((int)hub));
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = 0.f;
  }
};
template <>
struct Vec<8> {
  float v[8];
  __device__ __forceinline__ void load(const float* p) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7])
        : "l"(p));
  }
  __device__ __forceinline__ void load_hint(const float* p, bool hub) {
    asm("{\n .reg .pred h;\n setp.ne.b32 h, %9, 0;\n"
        " @h ld.global.nc.L1::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
        " @!h ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n}"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7])
        : "l"(p), "r"((int)hub));
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.f;
  }
};

// TWO (fp32 accumulation, !F64): two-level fp32 sums -- a window of 32
// entries, folded into a second fp32 accumulator.  Error <= (32 + len/32)
// ulp of the row's sum of |terms| (<= 64 ulp = 3.8e-6 for a 1024-entry
// item), inside the 1e-5 contract, with 8 fewer registers than fp64 folds.
// STG (experiment): the item's entries are staged into shared memory by
// cp.async one 2G-entry window ahead (no registers held by the CSR
// prefetch); every lane reads the window's (col, val) pairs as broadcasts.
// FN > 0: fused forward epilogue for 13..16-float rows (G = 4
// lanes x one float4, fp64 folds): the row of T = A H never leaves the
// registers -- the four lanes swap their quarters, each computes FN/4
// columns of z = t W from W in shared memory and stores z and relu(z).
template <int G, int CPL, bool F64, int V, int MB = Tune<CPL, V>::MINB,
          int EE = Tune<CPL, V>::E, bool TWO = false, bool STG = false, int FN = 0>
__global__ void __launch_bounds__(256, MB)
    spmm_kernel(const __grid_constant__ SpmmArgs a) {
  constexpr int E = EE;                     // entries per pipeline step
  static_assert(!(TWO && F64), "TWO is an fp32 mode");
  static_assert(FN == 0 || (G == 4 && CPL == 1 && V == 4 && F64 && !STG),
                "fused epilogue: 16-float rows only");
  constexpr int WIN = 2 * G;                // STG: entries per staged window (16 B per lane)
  static_assert(!STG || (WIN % E == 0), "STG: window must hold whole steps");
  __shared__ __align__(16) int2 stg[STG ? 256 / G : 1][2][STG ? WIN : 1];
  __shared__ __align__(16) float Ws[FN > 0 ? 16 * FN : 1];
  if constexpr (FN > 0) {                   // W (16 x FN, zero padded), before any exit
    for (int i = threadIdx.x; i < 16 * FN; i += blockDim.x) {
      const int k = i / FN, j = i % FN;
      Ws[i] = (k < 16 && j < a.n_out) ? a.w[(int64_t)k * a.ld_w + j] : 0.f;
    }
    __syncthreads();
  }
  constexpr int E4 = E / 2;                 // int4 loads per step
  const int lig = threadIdx.x & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if (gid >= a.n_items) return;             // whole group leaves together
  const Item it = a.items[gid];
  const RankArgs& R = a.r[it.rank];
  const int slab0 = blockIdx.y * a.slab;
  const int64_t ld = a.ld_h;
  const int4* __restrict__ ep = R.ent + (it.lo >> 1);
  const float* __restrict__ hl = R.hl;
  const float* __restrict__ hh = R.hh;
  const int64_t nl = R.n_local;
  // one base-pointer select per gather (own block, or the halo buffer
  // pre-offset by -n_local rows) and a 32 x 32 -> 64-bit row offset: f=602
  // 18.3 -> 17.6 ms, f=41 1.70 -> 1.54 ms, products f=100 5.15 -> 4.84 ms
  // (profiles/r02/r2_v2_*)
  const int nl32 = (int)nl;
  const int ld32 = (int)ld;
  // halo row c lives at hh_off + c * ld (integer arithmetic: hh may be null
  // when the rank has no halo, and then no c >= n_local occurs)
  const float* hh_off =
      reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(hh) - (uintptr_t)(nl * ld * 4));
  const uint64_t pol = evict_first_policy();

  int chk[CPL];                             // chunk index (units of V floats)
  bool on[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    chk[q] = slab0 + lig + q * G;
    on[q] = chk[q] < a.chunks && (lig + q * G) < a.slab;
  }
  float part[CPL][V];
  double acc[F64 ? CPL : 1][V];
  float acc2[TWO ? CPL : 1][V];
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int k = 0; k < V; ++k) part[q][k] = 0.f;
  if constexpr (TWO) {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int k = 0; k < V; ++k) acc2[q][k] = 0.f;
  }
  if constexpr (F64) {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int k = 0; k < V; ++k) acc[q][k] = 0.0;
  }

  const int len = it.len;
  if constexpr (!STG) {
    const int n4 = (len + 1) >> 1;            // int4 words of this item
    const int steps = (len + E - 1) / E;
    int4 nx[E4];
  #pragma unroll
    for (int u = 0; u < E4; ++u) nx[u] = (u < n4) ? ld_stream(ep + u, pol) : make_int4(0, 0, 0, 0);

    for (int s = 0; s < steps; ++s) {
      int4 cur[E4];
  #pragma unroll
      for (int u = 0; u < E4; ++u) cur[u] = nx[u];
      if (s + 1 < steps) {                    // prefetch the next step's entries
  #pragma unroll
        for (int u = 0; u < E4; ++u) {
          const int w = (s + 1) * E4 + u;
          nx[u] = (w < n4) ? ld_stream(ep + w, pol) : make_int4(0, 0, 0, 0);
        }
      }
      const int nv = min(E, len - s * E);
      Vec<V> x[E][CPL];
      float v[E];
  #pragma unroll
      for (int j = 0; j < E; ++j) {
        const int c = ((j & 1) ? cur[j >> 1].z : cur[j >> 1].x) & 0x7fffffff;  // bit 31: hub
        v[j] = __int_as_float((j & 1) ? cur[j >> 1].w : cur[j >> 1].y);
        if (j < nv) {
          const float* hp = (c < nl32 ? hl : hh_off) + (int64_t)c * ld32;
  #pragma unroll
          for (int q = 0; q < CPL; ++q) {
            // narrow rows keep plain (L1-allocating) loads: their L1 hit rate
            // is 13-14% and no_allocate cost f=41 1.54 -> 2.07 ms
            if (on[q]) x[j][q].load(hp + (int64_t)chk[q] * V);
            else x[j][q].zero();
          }
        } else {
          v[j] = 0.f;
  #pragma unroll
          for (int q = 0; q < CPL; ++q) x[j][q].zero();
        }
      }
  #pragma unroll
      for (int j = 0; j < E; ++j)
  #pragma unroll
        for (int q = 0; q < CPL; ++q)
  #pragma unroll
          for (int k = 0; k < V; ++k) part[q][k] = fmaf(v[j], x[j][q].v[k], part[q][k]);
      if constexpr (F64) {
        if ((s & 1) || s + 1 == steps) {      // 8-entry fp32 windows into fp64
  #pragma unroll
          for (int q = 0; q < CPL; ++q)
  #pragma unroll
            for (int k = 0; k < V; ++k) {
              acc[q][k] += (double)part[q][k];
              part[q][k] = 0.f;
            }
        }
      } else if constexpr (TWO) {
        constexpr int WS = 32 / E;            // steps per 32-entry window
        if (s % WS == WS - 1) {
  #pragma unroll
          for (int q = 0; q < CPL; ++q)
  #pragma unroll
            for (int k = 0; k < V; ++k) {
              acc2[q][k] += part[q][k];
              part[q][k] = 0.f;
            }
        }
      }
    }
  } else {
    // ---- staged entries: window w of the item lives in stg[grp][w & 1]
    const int grp = (threadIdx.x & 255) / G;
    const unsigned gmask = G == 32 ? 0xffffffffu
                                   : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    const int2* __restrict__ src = reinterpret_cast<const int2*>(R.ent) + it.lo;
    const int nwin = (len + WIN - 1) / WIN;
    const int len2 = (len + 1) & ~1;        // storage is padded to even entries
    auto issue = [&](int w) {
      const int e0 = w * WIN + 2 * lig;
      int2* dst = &stg[grp][w & 1][2 * lig];
      if (w < nwin && e0 < len2) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + e0)
                     : "memory");
      } else {
        *reinterpret_cast<int4*>(dst) = make_int4(0, 0, 0, 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    issue(1);
    for (int w = 0; w < nwin; ++w) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp(gmask);
      const int2* win = stg[grp][w & 1];
#pragma unroll
      for (int st = 0; st < WIN / E; ++st) {
        const int base = w * WIN + st * E;
        if (base >= len) break;
        const int nv = min(E, len - base);
        Vec<V> x[E][CPL];
        float v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int2 en = win[st * E + j];
          v[j] = __int_as_float(en.y);
          if (j < nv) {
            const int c = en.x & 0x7fffffff;        // bit 31: a hub row (plan)
            const float* hp = (c < nl32 ? hl : hh_off) + (int64_t)c * ld32;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
              if (on[q]) x[j][q].load_hint(hp + (int64_t)chk[q] * V, en.x < 0);
              else x[j][q].zero();
            }
          } else {
            v[j] = 0.f;
#pragma unroll
            for (int q = 0; q < CPL; ++q) x[j][q].zero();
          }
        }
        const int s = base / E;
    #pragma unroll
        for (int j = 0; j < E; ++j)
    #pragma unroll
          for (int q = 0; q < CPL; ++q)
    #pragma unroll
            for (int k = 0; k < V; ++k) part[q][k] = fmaf(v[j], x[j][q].v[k], part[q][k]);
        if constexpr (F64) {
    #pragma unroll
          for (int q = 0; q < CPL; ++q)
    #pragma unroll
            for (int k = 0; k < V; ++k) {
              acc[q][k] += (double)part[q][k];
              part[q][k] = 0.f;
            }
        } else if constexpr (TWO) {
          constexpr int WS = 32 / E;            // steps per 32-entry window
          if (s % WS == WS - 1) {
    #pragma unroll
            for (int q = 0; q < CPL; ++q)
    #pragma unroll
              for (int k = 0; k < V; ++k) {
                acc2[q][k] += part[q][k];
                part[q][k] = 0.f;
              }
          }
        }
      }
      __syncwarp(gmask);
      issue(w + 2);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  if constexpr (TWO) {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int k = 0; k < V; ++k) part[q][k] += acc2[q][k];
  }

  if constexpr (FN > 0) {
    // the group's four lanes hold t[4 lig .. 4 lig + 3]; swap the quarters
    const int gbase = (threadIdx.x & 31) & ~3;
    const unsigned gm = 0xFu << gbase;
    float mine[4], t[16];
#pragma unroll
    for (int e = 0; e < 4; ++e) mine[e] = (float)acc[0][e];
#pragma unroll
    for (int src = 0; src < 4; ++src)
#pragma unroll
      for (int e = 0; e < 4; ++e) t[4 * src + e] = __shfl_sync(gm, mine[e], gbase + src);
    if (it.slot < 0) {
      constexpr int NPL = FN / 4;             // output columns per lane
      float zz[NPL];
#pragma unroll
      for (int j = 0; j < NPL; ++j) zz[j] = 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float4* wr = reinterpret_cast<const float4*>(Ws + k * FN + lig * NPL);
#pragma unroll
        for (int j4 = 0; j4 < NPL / 4; ++j4) {
          const float4 wv = wr[j4];
          zz[4 * j4 + 0] = fmaf(t[k], wv.x, zz[4 * j4 + 0]);
          zz[4 * j4 + 1] = fmaf(t[k], wv.y, zz[4 * j4 + 1]);
          zz[4 * j4 + 2] = fmaf(t[k], wv.z, zz[4 * j4 + 2]);
          zz[4 * j4 + 3] = fmaf(t[k], wv.w, zz[4 * j4 + 3]);
        }
      }
      float* zp = R.z + (int64_t)it.row * a.ld_z + lig * NPL;
      float* hp = R.hr ? R.hr + (int64_t)it.row * a.ld_z + lig * NPL : nullptr;
#pragma unroll
      for (int j4 = 0; j4 < NPL / 4; ++j4) {
        if (lig * NPL + 4 * j4 >= a.ld_z) break;
        *reinterpret_cast<float4*>(zp + 4 * j4) =
            make_float4(zz[4 * j4], zz[4 * j4 + 1], zz[4 * j4 + 2], zz[4 * j4 + 3]);
        if (hp)
          *reinterpret_cast<float4*>(hp + 4 * j4) =
              make_float4(fmaxf(zz[4 * j4], 0.f), fmaxf(zz[4 * j4 + 1], 0.f),
                          fmaxf(zz[4 * j4 + 2], 0.f), fmaxf(zz[4 * j4 + 3], 0.f));
      }
      return;
    }
  }
  if (it.slot < 0) {
    float* zp = R.z + (int64_t)it.row * a.ld_z;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (on[q]) {
        float o[V];
        float4* zq = reinterpret_cast<float4*>(zp + (int64_t)chk[q] * V);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          if constexpr (F64) {
            o[k] = (float)acc[q][k];
          } else {
            o[k] = part[q][k];
          }
        }
        if (a.beta) {                       // z += result (halo pass)
#pragma unroll
          for (int h4 = 0; h4 < V / 4; ++h4) {
            const float4 zo = zq[h4];
            if constexpr (F64) {
              o[4 * h4 + 0] = (float)(acc[q][4 * h4 + 0] + (double)zo.x);
              o[4 * h4 + 1] = (float)(acc[q][4 * h4 + 1] + (double)zo.y);
              o[4 * h4 + 2] = (float)(acc[q][4 * h4 + 2] + (double)zo.z);
              o[4 * h4 + 3] = (float)(acc[q][4 * h4 + 3] + (double)zo.w);
            } else {
              o[4 * h4 + 0] += zo.x;
              o[4 * h4 + 1] += zo.y;
              o[4 * h4 + 2] += zo.z;
              o[4 * h4 + 3] += zo.w;
            }
          }
        }
#pragma unroll
        for (int h4 = 0; h4 < V / 4; ++h4)
          zq[h4] = make_float4(o[4 * h4], o[4 * h4 + 1], o[4 * h4 + 2], o[4 * h4 + 3]);
      }
  } else {
    double* pp = a.part + (int64_t)it.slot * a.ld_part;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (on[q]) {
        double4* dq = reinterpret_cast<double4*>(pp + (int64_t)chk[q] * V);
#pragma unroll
        for (int h4 = 0; h4 < V / 4; ++h4) {
          double4 d;
          if constexpr (F64) {
            d = make_double4(acc[q][4 * h4], acc[q][4 * h4 + 1], acc[q][4 * h4 + 2],
                             acc[q][4 * h4 + 3]);
          } else {
            d = make_double4(part[q][4 * h4], part[q][4 * h4 + 1], part[q][4 * h4 + 2],
                             part[q][4 * h4 + 3]);
          }
          dq[h4] = d;
        }
      }
  }
}

struct FixArgs {
  float* z[DG_MAX_LOCAL];
  float* hr[DG_MAX_LOCAL];   // fused epilogue: relu(z) (nullable)
  const Fixup* fix;
  const double* part;
  int64_t ld_z;
  int64_t ld_part;
  int32_t nfloat;      // chunks * 4
  int32_t beta;
};

__global__ void __launch_bounds__(128) spmm_fixup_kernel(const __grid_constant__ FixArgs a) {
  const Fixup fx = a.fix[blockIdx.x];
  float* zp = a.z[fx.rank] + (int64_t)fx.row * a.ld_z;
  for (int c = threadIdx.x; c < a.nfloat; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < fx.n; ++k) s += a.part[(int64_t)(fx.slot0 + k) * a.ld_part + c];
    if (a.beta) s += (double)zp[c];
    zp[c] = (float)s;
  }
}

// fused epilogue for the split rows: one warp per split row (8 per CTA);
// lanes 0..15 form t = the ordered sum of the row's partials (as
// spmm_fixup_kernel), broadcast by shuffles, then z = t W, relu(z)
__global__ void __launch_bounds__(256) spmm_fixup_fused_kernel(
    const __grid_constant__ FixArgs a, int64_t n_fix, const float* __restrict__ w, int ld_w,
    int n_out) {
  const int64_t fi = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (fi >= n_fix) return;
  const int lane = threadIdx.x & 31;
  const Fixup fx = a.fix[fi];
  double s = 0.0;
  if (lane < a.nfloat)
    for (int k = 0; k < fx.n; ++k) s += a.part[(int64_t)(fx.slot0 + k) * a.ld_part + lane];
  const float tl = lane < 16 ? (float)s : 0.f;
  float t[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) t[k] = __shfl_sync(0xffffffffu, tl, k);
  float* zp = a.z[fx.rank] + (int64_t)fx.row * a.ld_z;
  float* hp = a.hr[fx.rank] ? a.hr[fx.rank] + (int64_t)fx.row * a.ld_z : nullptr;
  for (int j = lane; j < a.ld_z; j += 32) {
    float v = 0.f;
    if (j < n_out)
#pragma unroll
      for (int k = 0; k < 16; ++k) v = fmaf(t[k], __ldg(w + (int64_t)k * ld_w + j), v);
    zp[j] = v;
    if (hp) hp[j] = fmaxf(v, 0.f);
  }
}

int bucket_of(int32_t len) {
  // ~4 buckets per octave: warps see trip counts within ~19% of each other
  if (len <= 0) return 0;
  return (int)(4.0 * std::log2((double)len)) + 1;
}

template <int G, int CPL, bool F64, int V, int MB = Tune<CPL, V>::MINB,
          int EE = Tune<CPL, V>::E, bool TWO = false, bool STG = false>
void launch_spmm(const SpmmArgs& a, int nslabs, cudaStream_t s) {
  const int64_t threads = a.n_items * G;
  const unsigned gx = (unsigned)((threads + 255) / 256);
  spmm_kernel<G, CPL, F64, V, MB, EE, TWO, STG><<<dim3(gx, nslabs), 256, 0, s>>>(a);
}

using LaunchFn = void (*)(const SpmmArgs&, int, cudaStream_t);

template <bool F64, int V>
LaunchFn pick_launch(int G, int CPL) {
#define DG_CASE(g, c) \
  if (G == g && CPL == c) return &launch_spmm<g, c, F64, V>;
  DG_CASE(1, 1) DG_CASE(1, 2) DG_CASE(1, 3) DG_CASE(1, 4)
  DG_CASE(2, 1) DG_CASE(2, 2) DG_CASE(2, 3) DG_CASE(2, 4)
  DG_CASE(4, 1) DG_CASE(4, 2) DG_CASE(4, 3) DG_CASE(4, 4)
  DG_CASE(8, 1) DG_CASE(8, 2) DG_CASE(8, 3) DG_CASE(8, 4)
  DG_CASE(16, 1) DG_CASE(16, 2) DG_CASE(16, 3) DG_CASE(16, 4)
  DG_CASE(32, 1) DG_CASE(32, 2) DG_CASE(32, 3) DG_CASE(32, 4)
#undef DG_CASE
  return nullptr;
}

// acc == 2 (the default): one 256-bit chunk per lane, entries staged in
// shared memory, two-level fp32 sums, 4 CTAs/SM at 2 entries per step
// (64 registers, no spill).  Sweep (profiles/r01/spmm_sweep_stg.txt): f=602
// 19.8 -> 18.2 ms, f=41 1.95 -> 1.77 ms, products f=100 6.4 -> 6.1 ms.
LaunchFn pick_two(int G) {
  switch (G) {
    case 2: return &launch_spmm<2, 1, false, 8, 4, 2, true, true>;
    case 4: return &launch_spmm<4, 1, false, 8, 4, 2, true, true>;
    case 8: return &launch_spmm<8, 1, false, 8, 4, 2, true, true>;
    // 16-lane groups (97..128-float rows: products f=100, papers f=128; the
    // gathers miss L2 often): 4 entries per step at 3 CTAs/SM keep more bytes
    // in flight than 2 at 4 CTAs/SM -- products f=100 4.84 -> 4.76 ms
    case 16: return &launch_spmm<16, 1, false, 8, 3, 4, true, true>;
    case 32: return &launch_spmm<32, 1, false, 8, 4, 2, true, true>;
    default: return nullptr;
  }
}

// Lane-group size G and chunks-per-lane CPL for `chunks` float4 chunks when
// one slab may hold at most `wmax` chunks: fewest slabs, then least waste,
// ties to the larger G.
void choose_config(int chunks, int wmax, int* G_out, int* CPL_out, int* nslabs_out) {
  static const int Gs[6] = {32, 16, 8, 4, 2, 1};
  int bestG = 1, bestC = 1, bestS = 1 << 30, bestWaste = 1 << 30;
  wmax = std::max(wmax, 1);
  for (int gi = 0; gi < 6; ++gi) {
    for (int c = 1; c <= 4; ++c) {
      const int G = Gs[gi], W = G * c;
      if (W > wmax && !(G == 1 && c == 1)) continue;
      const int ns = (chunks + W - 1) / W;
      const int waste = ns * W - chunks;
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

// Device-source plans (DG_PLAN_DEVICE_SRC): the CSR already lives in HBM
// (graphs built on the GPU, too large to stage through host memory).  The
// items are still built on the host from row_ptr (O(rows)); the entries are
// laid out by this kernel, one warp per item.
struct RelayoutArgs {
  const int32_t* col[DG_MAX_LOCAL];
  const float* val[DG_MAX_LOCAL];
  int2* ent[DG_MAX_LOCAL];
};

__global__ void relayout_kernel(const Item* __restrict__ items, const int64_t* __restrict__ src_lo,
                                int64_t n_items, RelayoutArgs a) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < n_items; w += nw) {
    const Item it = items[w];
    const int64_t s = src_lo[w];
    const int32_t* __restrict__ c = a.col[it.rank] + s;
    const float* __restrict__ v = a.val[it.rank] + s;
    int2* __restrict__ d = a.ent[it.rank] + it.lo;
    for (int32_t k = lane; k < it.len; k += 32) d[k] = make_int2(c[k], __float_as_int(v[k]));
  }
}

__global__ void max_col_kernel(const int32_t* __restrict__ col, int64_t n, int* __restrict__ out) {
  int m = -1;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    m = max(m, col[k]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

struct dg_spmm_plan {
  int n_ranks = 0;
  std::vector<int64_t> n_rows, n_local, nnz, ext_rows;
  std::vector<int4*> ent;
  Item* items = nullptr;
  int64_t n_items = 0;
  Fixup* fix = nullptr;
  int64_t n_fix = 0;
  int64_t n_slots = 0;
  double* part = nullptr;
  int64_t part_cap = 0;  // doubles
  int64_t dev_bytes = 0;
  int64_t window_nnz = 0;  // length-bucketing window used (INT64_MAX: one global window)
};

extern "C" {

int dg_spmm_plan_destroy(dg_spmm_plan* p) {
  if (!p) return DG_OK;
  for (auto* e : p->ent) cudaFree(e);
  if (p->items) cudaFree(p->items);
  if (p->fix) cudaFree(p->fix);
  if (p->part) cudaFree(p->part);
  delete p;
  return DG_OK;
}

int dg_spmm_plan_create(dg_spmm_plan** out, int n_ranks, const int64_t* n_rows,
                        const int64_t* n_local, const int64_t* nnz,
                        const int64_t* const* row_ptr, const int32_t* const* col_ext,
                        const float* const* val, int32_t max_chunk, int32_t flags) {
  return dg_spmm_plan_create_ordered(out, n_ranks, n_rows, n_local, nnz, row_ptr, col_ext, val,
                                     max_chunk, flags, nullptr, 0);
}

int dg_spmm_plan_create_ordered(dg_spmm_plan** out, int n_ranks, const int64_t* n_rows,
                                const int64_t* n_local, const int64_t* nnz,
                                const int64_t* const* row_ptr, const int32_t* const* col_ext,
                                const float* const* val, int32_t max_chunk, int32_t flags,
                                const int32_t* const* row_order, int64_t window_nnz) {
  const bool skip_empty = (flags & DG_PLAN_SKIP_EMPTY_ROWS) != 0;
  const bool dev_src = (flags & DG_PLAN_DEVICE_SRC) != 0;
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
    if (n_rows[r] > INT32_MAX) {
      delete p;
      return set_err(DG_ERR_ARG, "dg_spmm_plan_create: rank too large for int32 rows");
    }
    int32_t mx = -1;
    if (dev_src) {
      int* d_mx = nullptr;
      cudaError_t e = cudaMalloc(&d_mx, sizeof(int));
      if (e == cudaSuccess) e = cudaMemcpy(d_mx, &mx, sizeof(int), cudaMemcpyHostToDevice);
      if (e == cudaSuccess && nnz[r] > 0) {
        max_col_kernel<<<1184, 256>>>(col_ext[r], nnz[r], d_mx);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaMemcpy(&mx, d_mx, sizeof(int), cudaMemcpyDeviceToHost);
      if (d_mx) cudaFree(d_mx);
      if (e != cudaSuccess) {
        delete p;
        return set_err(DG_ERR_CUDA, std::string("plan max col: ") + cudaGetErrorString(e));
      }
    } else {
      for (int64_t k = 0; k < nnz[r]; ++k) mx = std::max(mx, col_ext[r][k]);
    }
    p->ext_rows.push_back((int64_t)mx + 1);
    const int32_t* ord = row_order ? row_order[r] : nullptr;
    if (ord) {                                  // must be a permutation of the rows
      std::vector<char> seen(n_rows[r], 0);
      for (int64_t k = 0; k < n_rows[r]; ++k) {
        const int32_t i = ord[k];
        if (i < 0 || i >= n_rows[r] || seen[i]) {
          delete p;
          return set_err(DG_ERR_ARG, "dg_spmm_plan_create: row_order is not a permutation");
        }
        seen[i] = 1;
      }
    }
    for (int64_t k = 0; k < n_rows[r]; ++k) {
      const int64_t i = ord ? ord[k] : k;
      const int64_t lo = row_ptr[r][i], hi = row_ptr[r][i + 1];
      const int64_t len = hi - lo;
      if (len == 0 && skip_empty) continue;
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
  // Window: explicit, or (window_nnz <= 0) chosen from the graph.  Windows
  // pay when a row's gathers land near it in the processing order (a
  // community order: products-shaped f=100 6.1 -> 5.2 ms with 2^20-entry
  // windows, 5.5 ms with 2^22, 5.3 ms with 2^17); on a graph
  // without locality (Reddit-shaped) the global heavy-first order wins
  // (f=602 18.1 vs 18.9 ms, f=16 0.71 vs 0.81 ms).  Locality score: the
  // share of own-block entries whose column is processed within one window
  // of its row; >= 25% -> windows.
  if (window_nnz <= 0) {
    window_nnz = INT64_MAX;
    int64_t near = 0, total_nnz = 0;
    for (int r = 0; r < n_ranks && !dev_src; ++r) {
      total_nnz += nnz[r];
      if (n_local[r] != n_rows[r] || n_rows[r] == 0 || nnz[r] == 0) continue;
      const int64_t m = n_rows[r];
      std::vector<int64_t> pos(m);
      for (int64_t k = 0; k < m; ++k) pos[row_order && row_order[r] ? row_order[r][k] : k] = k;
      const int64_t reach = std::max<int64_t>(
          1, (int64_t)((double)m * (double)DG_SPMM_WINDOW_NNZ / (double)nnz[r]));
      for (int64_t i = 0; i < m; ++i)
        for (int64_t e = row_ptr[r][i]; e < row_ptr[r][i + 1]; ++e) {
          const int32_t c = col_ext[r][e];
          if (c < m && std::llabs(pos[c] - pos[i]) <= reach) ++near;
        }
    }
    if (total_nnz > 0 && near * 4 >= total_nnz) window_nnz = DG_SPMM_WINDOW_NNZ;
  }
  p->window_nnz = window_nnz;
  // Items follow the row order (identity, or a locality order such as
  // communities) in windows of ~window_nnz entries; inside a window they are
  // bucketed by length (descending, stable): similar trip counts per warp,
  // heavy items first.  Windows keep the rows that are in flight together
  // -- and so the H rows they gather -- close in the row order: a global
  // sort would spread every bucket over the whole matrix and make the whole
  // H table the working set (products-shaped f=16: 34% L2 hit rate).
  {
    size_t w0 = 0;
    int64_t acc_nnz = 0;
    auto by_bucket = [](const Item& x, const Item& y) {
      return bucket_of(x.len) > bucket_of(y.len);
    };
    for (size_t k = 0; k < items.size(); ++k) {
      acc_nnz += items[k].len;
      if (acc_nnz >= window_nnz || k + 1 == items.size()) {
        std::stable_sort(items.begin() + w0, items.begin() + k + 1, by_bucket);
        w0 = k + 1;
        acc_nnz = 0;
      }
    }
  }
  // lay the entries out in item order (the order warps stream them), each
  // item starting at an even entry (16-B aligned int4 pairs)
  std::vector<int64_t> cursor(n_ranks, 0);
  std::vector<int64_t> total(n_ranks, 0);
  for (const Item& it : items) total[it.rank] += (it.len + 1) & ~1LL;
  auto fail = [&](cudaError_t e, const char* what) {
    dg_spmm_plan_destroy(p);
    return set_err(DG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  if (dev_src) {
    std::vector<int64_t> src_lo(items.size());
    for (size_t k = 0; k < items.size(); ++k) {
      Item& it = items[k];
      src_lo[k] = it.lo;
      it.lo = cursor[it.rank];
      cursor[it.rank] += (it.len + 1) & ~1LL;
    }
    RelayoutArgs ra;
    std::memset(&ra, 0, sizeof(ra));
    for (int r = 0; r < n_ranks; ++r) {
      int4* d = nullptr;
      const size_t bytes = (size_t)std::max<int64_t>(total[r], 2) * 8;
      cudaError_t e = cudaMalloc(&d, bytes);
      if (e != cudaSuccess) return fail(e, "cudaMalloc(entries)");
      p->ent.push_back(d);
      e = cudaMemset(d, 0, bytes);
      if (e != cudaSuccess) return fail(e, "cudaMemset(entries)");
      p->dev_bytes += (int64_t)bytes;
      ra.col[r] = col_ext[r];
      ra.val[r] = val[r];
      ra.ent[r] = reinterpret_cast<int2*>(d);
    }
    if (!items.empty()) {
      Item* d_items = nullptr;
      int64_t* d_lo = nullptr;
      cudaError_t e = cudaMalloc(&d_items, items.size() * sizeof(Item));
      if (e == cudaSuccess) e = cudaMalloc(&d_lo, items.size() * sizeof(int64_t));
      if (e == cudaSuccess)
        e = cudaMemcpy(d_items, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice);
      if (e == cudaSuccess)
        e = cudaMemcpy(d_lo, src_lo.data(), items.size() * sizeof(int64_t),
                       cudaMemcpyHostToDevice);
      if (e == cudaSuccess) {
        relayout_kernel<<<148 * 16, 256>>>(d_items, d_lo, (int64_t)items.size(), ra);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (d_lo) cudaFree(d_lo);
      if (e != cudaSuccess) {
        if (d_items) cudaFree(d_items);
        return fail(e, "relayout");
      }
      p->items = d_items;
    }
  } else {
    // hub rows: the DG_SPMM_HUB_ROWS most gathered columns of each rank get
    // bit 31 of their entries set; the kernel keeps their rows in L1
    // (evict_last) and lets every other gather bypass it
    std::vector<std::vector<char>> hub(n_ranks);
    for (int r = 0; r < n_ranks && DG_SPMM_HUB_ROWS > 0; ++r) {
      const int64_t ext = p->ext_rows[r];
      if (ext <= 0 || nnz[r] == 0) continue;
      std::vector<int32_t> cnt(ext, 0);
      for (int64_t k = 0; k < nnz[r]; ++k) ++cnt[col_ext[r][k]];
      const int64_t K = std::min<int64_t>(DG_SPMM_HUB_ROWS, ext);
      std::vector<int32_t> idx(ext);
      for (int64_t i = 0; i < ext; ++i) idx[i] = (int32_t)i;
      std::nth_element(idx.begin(), idx.begin() + (K - 1), idx.end(),
                       [&](int32_t x, int32_t y) { return cnt[x] > cnt[y]; });
      const int32_t kth = cnt[idx[K - 1]];
      hub[r].assign(ext, 0);
      // a hub must be gathered well above the average (>= 4x), else no flag
      const double avg = (double)nnz[r] / (double)ext;
      for (int64_t i = 0; i < K; ++i)
        if (cnt[idx[i]] >= 4.0 * avg && cnt[idx[i]] >= kth) hub[r][idx[i]] = 1;
    }
    std::vector<std::vector<int32_t>> host(n_ranks);
    for (int r = 0; r < n_ranks; ++r) host[r].assign(2 * std::max<int64_t>(total[r], 2), 0);
    for (Item& it : items) {
      const int r = it.rank;
      const int64_t dst = cursor[r];
      int32_t* h = host[r].data() + 2 * dst;
      for (int32_t k = 0; k < it.len; ++k) {
        const int32_t cc = col_ext[r][it.lo + k];
        h[2 * k] = (!hub[r].empty() && hub[r][cc]) ? (int32_t)(cc | 0x80000000u) : cc;
        float v = val[r][it.lo + k];
        std::memcpy(&h[2 * k + 1], &v, 4);
      }
      it.lo = dst;
      cursor[r] += (it.len + 1) & ~1LL;
    }
    for (int r = 0; r < n_ranks; ++r) {
      int4* d = nullptr;
      const size_t bytes = host[r].size() * sizeof(int32_t);
      cudaError_t e = cudaMalloc(&d, bytes);
      if (e != cudaSuccess) return fail(e, "cudaMalloc(entries)");
      p->ent.push_back(d);
      e = cudaMemcpy(d, host[r].data(), bytes, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(e, "cudaMemcpy(entries)");
      p->dev_bytes += (int64_t)bytes;
      std::vector<int32_t>().swap(host[r]);
    }
  }
  p->n_items = (int64_t)items.size();
  p->n_fix = (int64_t)fix.size();
  p->n_slots = slots;
  cudaError_t e = cudaSuccess;
  if (!p->items) {
    e = cudaMalloc(&p->items, std::max<size_t>(items.size(), 1) * sizeof(Item));
    if (e != cudaSuccess) return fail(e, "cudaMalloc(items)");
    if (!items.empty()) {
      e = cudaMemcpy(p->items, items.data(), items.size() * sizeof(Item),
                     cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(e, "cudaMemcpy(items)");
    }
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

int dg_spmm_plan_reserve(dg_spmm_plan* p, int64_t ld_max) {
  if (!p || ld_max < 0) return set_err(DG_ERR_ARG, "dg_spmm_plan_reserve: bad args");
  const int64_t need = p->n_slots * ld_max;
  if (need <= p->part_cap) return DG_OK;
  if (p->part) DG_CK(cudaFree(p->part));
  p->part = nullptr;
  p->part_cap = 0;
  DG_CK(cudaMalloc(&p->part, need * sizeof(double)));
  p->part_cap = need;
  return DG_OK;
}

int dg_spmm_plan_info(const dg_spmm_plan* p, int64_t info[8]) {
  if (!p) return set_err(DG_ERR_ARG, "null plan");
  int64_t nnz = 0, ext = 0;
  for (auto x : p->nnz) nnz += x;
  for (auto x : p->ext_rows) ext += x;
  info[0] = p->n_items;
  info[1] = p->n_fix;
  info[2] = p->n_slots;
  info[3] = nnz;
  info[4] = p->dev_bytes + p->part_cap * 8;
  info[5] = ext;
  info[6] = p->window_nnz;
  info[7] = 0;
  return DG_OK;
}

int dg_spmm_run(dg_spmm_plan* p, const float* const* h_local, const float* const* h_halo,
                float* const* z, int32_t f, int64_t ld_h, int64_t ld_z, int32_t acc,
                int32_t slab_floats, int32_t beta, void* stream) {
  if (!p) return set_err(DG_ERR_ARG, "dg_spmm_run: null plan");
  if (f < 1 || ld_h % 4 || ld_z % 4 || f > ld_h || f > ld_z || acc < 0 || acc > 2)
    return set_err(DG_ERR_ARG, "dg_spmm_run: need 1 <= f <= ld, ld % 4 == 0, acc in 0..2");
  // 256-bit lane chunks when rows are >= 32 floats and 32-B aligned
  // 256-bit lanes for rows of >= 32 floats, and for 9..16-float rows gathered
  // from a table far larger than L2 (papers-shaped f=16: 55.7 -> 53.0 ms at
  // N=4).  Tables near L2 size keep 128-bit lanes (Reddit f=16 0.71 vs 0.78 ms;
  // products N=4 halo pass 0.62 vs 0.90 ms; profiles/r01/spmm_f16_lanes.txt)
  int64_t ext_rows_all = 0;
  for (int r = 0; r < p->n_ranks; ++r) ext_rows_all += p->ext_rows[r];
  const bool dram_table = (double)ext_rows_all * (double)ld_h * 4.0 > 1024.0 * 1024 * 1024;
  // 128-bit lanes for rows of up to 48 floats: f=41/47 rows take 12 lane-
  // chunks of 16 B (3 per lane) instead of 6 x 32 B with two idle lanes of
  // eight, 1.66 vs 1.77 ms (profiles/r01/spmm_f41_lanes.txt)
  // (round 2, products-shaped with LPA order: 256-bit lanes for 17..48
  // floats 2.99 vs 2.72 ms at f=47; for all 9..48 floats f=16 1.42 vs 1.22 ms;
  // one 128-bit chunk per lane (G=16) at f=47 3.80 ms -- profiles/r02/r2_lanes_*)
  bool v8 = (f > 48 || (f > 8 && f <= 16 && acc == 2 && dram_table)) && ld_h % 8 == 0 &&
            ld_z % 8 == 0;
  for (int r = 0; r < p->n_ranks && v8; ++r) {
    const uintptr_t al = (uintptr_t)h_local[r] | (uintptr_t)z[r] |
                         (uintptr_t)(h_halo ? h_halo[r] : nullptr);
    v8 = (al & 31) == 0;
  }
  const int V = v8 ? 8 : 4;
  // chunks cover the row up to the next 32-B boundary when the pitch allows
  // (f=41 -> 48 floats): the zero padding of H is carried into Z's padding
  const int chunks = (V == 4 && ld_h % 8 == 0 && ld_z % 8 == 0) ? (f + 7) / 8 * 2
                                                                 : (f + V - 1) / V;
  SpmmArgs a;
  std::memset(&a, 0, sizeof(a));
  int64_t ext_total = 0;
  for (int r = 0; r < p->n_ranks; ++r) {
    const uintptr_t al = (uintptr_t)h_local[r] | (uintptr_t)z[r] |
                         (uintptr_t)(h_halo ? h_halo[r] : nullptr);
    if (al & 15) return set_err(DG_ERR_ARG, "dg_spmm_run: H/Z must be 16-byte aligned");
    a.r[r] = RankArgs{p->ent[r], h_local[r], h_halo ? h_halo[r] : nullptr, z[r], nullptr,
                      p->n_local[r]};
    ext_total += p->ext_rows[r];
  }
  if (p->n_slots) {
    const int64_t need = p->n_slots * ld_h;
    if (need > p->part_cap) {
      // growing frees and allocates (a device-wide sync): never inside a
      // stream capture -- plans used by captured epochs are reserved up
      // front (dg_spmm_plan_reserve) for the widest pitch of the run
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      DG_CK(cudaStreamIsCapturing(S(stream), &cs));
      if (cs != cudaStreamCaptureStatusNone)
        return set_err(DG_ERR_ARG, "dg_spmm_run: split-row buffer too small during capture "
                                   "(reserve the plan for the widest pitch first)");
      if (const int rc = dg_spmm_plan_reserve(p, ld_h)) return rc;
    }
  }
  int wmax;
  if (slab_floats > 0) {
    wmax = std::max(1, slab_floats / V);
  } else {
    // Slabs pay off only when a slab of >= 128 B per gathered row stays
    // L2-resident (~64 MB of the 126 MB L2; measured on B200: Reddit-shaped
    // f=602 with 128-B rows -> 64-float slabs).  When even that does not
    // fit, the gathers hit DRAM whatever the slab, and one wide slab
    // (fewest CSR passes, widest G) wins.
    const double budget = 64.0 * 1024 * 1024;
    const double per_chunk = (double)std::max<int64_t>(ext_total, 1) * 4.0 * V;
    const int fit = (int)std::max(0.0, budget / per_chunk);
    const int min_w = 32 / V;                     // >= 128 B of every row per slab
    wmax = fit >= min_w ? fit : 128;
  }
  int G, CPL, ns;
  choose_config(chunks, wmax, &G, &CPL, &ns);

  const bool two = acc == 2 && v8;
  if (two) {
    // one chunk per lane (the two-level kernel's shape): the narrowest
    // power-of-two group covering a slab, same number of slabs
    int g = 2;
    while (g < (chunks + ns - 1) / ns && g < 32) g <<= 1;
    if (g * ns >= chunks) {
      G = g;
      CPL = 1;
    }
  }
  a.items = p->items;
  a.part = p->part;
  a.n_items = p->n_items;
  a.ld_h = ld_h;
  a.ld_z = ld_z;
  a.ld_part = ld_h;
  a.chunks = chunks;
  a.slab = G * CPL;
  a.beta = beta ? 1 : 0;
  if (p->n_items == 0) return DG_OK;
  LaunchFn fn = v8 ? (acc ? pick_launch<true, 8>(G, CPL) : pick_launch<false, 8>(G, CPL))
                   : (acc ? pick_launch<true, 4>(G, CPL) : pick_launch<false, 4>(G, CPL));
  if (two && CPL == 1) fn = pick_two(G);
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
    fa.nfloat = std::min<int>(chunks * V, (int)ld_z);
    fa.beta = beta ? 1 : 0;
    spmm_fixup_kernel<<<(unsigned)p->n_fix, 128, 0, S(stream)>>>(fa);
    DG_LAUNCHED();
  }
  return DG_OK;
}

int dg_spmm_run_fused(dg_spmm_plan* p, const float* const* h_local, const float* const* h_halo,
                      float* const* z, float* const* h_relu, int32_t f, int64_t ld_h,
                      int64_t ld_z, const float* w, int64_t ld_w, int32_t n_out, void* stream) {
  if (!p) return set_err(DG_ERR_ARG, "dg_spmm_run_fused: null plan");
  if (f < 13 || f > 16 || ld_h < 16 || ld_h % 4 || n_out < 1 || n_out > 64 || ld_z < n_out ||
      ld_z % 4 || ld_w < n_out || !w)
    return set_err(DG_ERR_ARG, "dg_spmm_run_fused: needs 13 <= f <= 16, n_out <= 64, "
                               "ld_z >= n_out, ld % 4 == 0");
  const int FN = (n_out + 15) / 16 * 16;
  if (ld_z > FN) return set_err(DG_ERR_ARG, "dg_spmm_run_fused: ld_z beyond the padded width");
  SpmmArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int r = 0; r < p->n_ranks; ++r) {
    const uintptr_t al = (uintptr_t)h_local[r] | (uintptr_t)z[r] |
                         (uintptr_t)(h_halo ? h_halo[r] : nullptr) |
                         (uintptr_t)(h_relu ? h_relu[r] : nullptr);
    if (al & 15) return set_err(DG_ERR_ARG, "dg_spmm_run_fused: pointers must be 16-B aligned");
    a.r[r] = RankArgs{p->ent[r], h_local[r], h_halo ? h_halo[r] : nullptr, z[r],
                      h_relu ? h_relu[r] : nullptr, p->n_local[r]};
  }
  if (p->n_slots) {
    const int64_t need = p->n_slots * ld_h;
    if (need > p->part_cap) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      DG_CK(cudaStreamIsCapturing(S(stream), &cs));
      if (cs != cudaStreamCaptureStatusNone)
        return set_err(DG_ERR_ARG, "dg_spmm_run_fused: split-row buffer too small during capture");
      if (const int rc = dg_spmm_plan_reserve(p, ld_h)) return rc;
    }
  }
  a.items = p->items;
  a.part = p->part;
  a.n_items = p->n_items;
  a.ld_h = ld_h;
  a.ld_z = ld_z;
  a.ld_part = ld_h;
  a.chunks = 4;
  a.slab = 4;
  a.beta = 0;
  a.w = w;
  a.ld_w = (int32_t)ld_w;
  a.n_out = n_out;
  if (p->n_items) {
    const unsigned gx = (unsigned)((p->n_items * 4 + 255) / 256);
    switch (FN) {
      case 16: spmm_kernel<4, 1, true, 4, 4, 4, false, false, 16><<<gx, 256, 0, S(stream)>>>(a); break;
      case 32: spmm_kernel<4, 1, true, 4, 4, 4, false, false, 32><<<gx, 256, 0, S(stream)>>>(a); break;
      case 48: spmm_kernel<4, 1, true, 4, 4, 4, false, false, 48><<<gx, 256, 0, S(stream)>>>(a); break;
      default: spmm_kernel<4, 1, true, 4, 4, 4, false, false, 64><<<gx, 256, 0, S(stream)>>>(a); break;
    }
    DG_LAUNCHED();
  }
  if (p->n_fix) {
    FixArgs fa;
    std::memset(&fa, 0, sizeof(fa));
    for (int r = 0; r < p->n_ranks; ++r) {
      fa.z[r] = z[r];
      fa.hr[r] = h_relu ? h_relu[r] : nullptr;
    }
    fa.fix = p->fix;
    fa.part = p->part;
    fa.ld_z = ld_z;
    fa.ld_part = ld_h;
    fa.nfloat = f;
    fa.beta = 0;
    spmm_fixup_fused_kernel<<<(unsigned)((p->n_fix + 7) / 8), 256, 0, S(stream)>>>(
        fa, p->n_fix, w, (int)ld_w, n_out);
    DG_LAUNCHED();
  }
  return DG_OK;
}

}  // extern "C"
