// probe.cu -- tensor-map construction for the TMA kernels, and a diagnostic
// probe of random-row gathers through TMA tile::gather4 (the Blackwell
// instruction for indexed row gathers): 4 table rows x box_cols floats per
// instruction into a shared-memory ring tracked by mbarriers, one producer
// lane per CTA, consumer warps draining the ring.  Compared against the
// register-path gather probe (dg_diag_gather) it answers whether TMA can
// feed the SpMM's H-row gathers faster than 256-bit LDGs.
#include "common.cuh"
#include "tma.cuh"

namespace dg {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}
}  // namespace

static int encode_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t ld, int64_t cols,
                     int box_cols, int box_rows, bool l2_promote_256, CUtensorMapSwizzle swz);

int make_tensor_map_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t ld,
                       int64_t cols, int box_cols, int box_rows, bool l2_promote_256) {
  return encode_2d(map, base, rows, ld, cols, box_cols, box_rows, l2_promote_256,
                   CU_TENSOR_MAP_SWIZZLE_NONE);
}

int make_tensor_map_2d_swz128(CUtensorMap* map, const void* base, int64_t rows, int64_t ld,
                              int64_t cols, int box_cols, int box_rows) {
  if (box_cols * 4 != 128) return set_err(DG_ERR_ARG, "128-byte swizzle needs 128-byte boxes");
  return encode_2d(map, base, rows, ld, cols, box_cols, box_rows, true,
                   CU_TENSOR_MAP_SWIZZLE_128B);
}

static int encode_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t ld, int64_t cols,
                     int box_cols, int box_rows, bool l2_promote_256, CUtensorMapSwizzle swz) {
  EncodeFn fn = encode_fn();
  if (!fn) return set_err(DG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)base & 15) || (ld * 4) % 16 || box_cols < 1 || box_cols > 256 ||
      box_rows < 1 || box_rows > 256 || (box_cols * 4) % 16)
    return set_err(DG_ERR_ARG, "tensor map: misaligned base / pitch or bad box");
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        l2_promote_256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                       : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(DG_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return DG_OK;
}

}  // namespace dg

namespace {

// ring of STAGES slots, each G4 gather4 loads (4*G4 rows of BOX floats)
template <int BOX, int G4, int STAGES, int CW>
__global__ void __launch_bounds__(32 * (CW + 1)) gather_tma_probe_kernel(
    const __grid_constant__ CUtensorMap map, int32_t c0, const int4* __restrict__ idx4,
    int64_t n_quads, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int ROWS = 4 * G4;
  constexpr int STAGE_FLOATS = ROWS * BOX;
  float* ring = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * STAGE_FLOATS * 4);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // this CTA's quads: a contiguous share of the index list, whole stages
  const int64_t per = (n_quads / G4 + gridDim.x - 1) / gridDim.x;   // stages per CTA
  const int64_t s0 = (int64_t)blockIdx.x * per;
  const int64_t s1 = min((int64_t)(blockIdx.x + 1) * per, n_quads / G4);
  const int64_t nst = max((int64_t)0, s1 - s0);
  if (warp == 0) {
    // lanes 0..G4-1 each issue one gather4 per stage (TMA issue from
    // several lanes); every lane's indices are loaded one stage ahead so no
    // issue waits on an index load
    int4 nxt = make_int4(0, 0, 0, 0);
    if (nst > 0 && lane < G4) nxt = __ldg(idx4 + s0 * G4 + lane);
    for (int64_t s = 0; s < nst; ++s) {
      const int slot = (int)(s % STAGES);
      if (s >= STAGES) mbar_wait(&empty[slot], (uint32_t)(((s / STAGES) - 1) & 1));
      if (lane == 0) mbar_arrive_expect_tx(&full[slot], STAGE_FLOATS * 4);
      __syncwarp();
      const int4 r = nxt;
      if (s + 1 < nst && lane < G4) nxt = __ldg(idx4 + (s0 + s + 1) * G4 + lane);
      if (lane < G4)
        tma_gather4(ring + (size_t)slot * STAGE_FLOATS + lane * 4 * BOX, &map, &full[slot], c0,
                    r.x, r.y, r.z, r.w);
    }
    return;
  }
  float acc = 0.f;
  const int t = threadIdx.x - 32;
  for (int64_t s = 0; s < nst; ++s) {
    const int slot = (int)(s % STAGES);
    mbar_wait(&full[slot], (uint32_t)((s / STAGES) & 1));
    const float4* st = reinterpret_cast<const float4*>(ring + (size_t)slot * STAGE_FLOATS);
    for (int k = t; k < STAGE_FLOATS / 4; k += 32 * CW) {
      const float4 v = st[k];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 123.456f) out[0] = acc;
}

template <int BOX, int G4, int STAGES, int CW>
int launch_probe(const CUtensorMap& map, int32_t c0, const int32_t* idx, int64_t n_idx,
                 int ctas, float* out, cudaStream_t st) {
  auto* k = gather_tma_probe_kernel<BOX, G4, STAGES, CW>;
  const size_t smem = (size_t)STAGES * 4 * G4 * BOX * 4 + 2 * STAGES * 8;
  DG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)ctas, 32 * (CW + 1), smem, st>>>(map, c0, reinterpret_cast<const int4*>(idx),
                                                  n_idx / 4, out);
  DG_LAUNCHED();
  return DG_OK;
}

}  // namespace

extern "C" int dg_diag_gather_tma(const float* tab, int64_t ld, int64_t rows, int32_t col0,
                                  int32_t box_cols, const int32_t* idx, int64_t n_idx,
                                  int32_t variant, int32_t ctas, float* out, void* stream) {
  CUtensorMap map;
  int rc = dg::make_tensor_map_2d(&map, tab, rows, ld, ld, box_cols, 1, true);
  if (rc) return rc;
  if ((uintptr_t)idx & 15) return set_err(DG_ERR_ARG, "diag_gather_tma: idx must be 16-B aligned");
  cudaStream_t st = S(stream);
  // variant: ring depth / rows per stage / consumer warps (bytes in flight per CTA)
#define DG_P(box, g4, stages, cw) \
  return launch_probe<box, g4, stages, cw>(map, col0, idx, n_idx, ctas, out, st)
  switch (box_cols * 10 + variant) {
    case 640: DG_P(64, 4, 12, 4);     // 16 rows x 256 B x 12 = 192 KB / CTA
    case 641: DG_P(64, 2, 24, 4);     //  8 rows per stage, 24 stages
    case 642: DG_P(64, 4, 6, 4);      // 96 KB / CTA (2 CTAs/SM)
    case 643: DG_P(64, 8, 6, 8);      // 32 rows per stage
    case 1280: DG_P(128, 2, 12, 4);   // 512-B rows, 8 rows per stage, 192 KB
    case 1282: DG_P(128, 2, 6, 4);    // 96 KB / CTA
    case 160: DG_P(16, 8, 24, 4);     // 64-B rows, 32 rows x 64 B x 24 = 48 KB
    case 162: DG_P(16, 16, 24, 4);    // 96 KB
    default: return set_err(DG_ERR_ARG, "diag_gather_tma: no such box / variant");
  }
#undef DG_P
}
