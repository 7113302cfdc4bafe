// tma.cuh -- Blackwell (sm_100a) TMA + mbarrier helpers shared by the kernels
// that stage operands through shared memory with the tensor-memory
// accelerator: tensor maps (cuTensorMapEncodeTiled, resolved at run time
// through the runtime's driver entry point -- no link-time libcuda
// dependency), 2-D tile and tile::gather4 loads, mbarrier phase waits.
#ifndef DG_TMA_CUH
#define DG_TMA_CUH

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dg {

// 2-D fp32 tensor map over a row-major (rows x ld) matrix, box = box_cols x
// box_rows elements (box_rows = 1 for tile::gather4).  Returns 0 on success.
int make_tensor_map_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t ld,
                       int64_t cols, int box_cols, int box_rows, bool l2_promote_256);
// the same with the 128-byte swizzle (box_cols * 4 == 128): 16-B chunk c of
// smem row r lands at chunk c ^ (r % 8) -- conflict-free column reads
int make_tensor_map_2d_swz128(CUtensorMap* map, const void* base, int64_t rows, int64_t ld,
                              int64_t cols, int box_cols, int box_rows);

}  // namespace dg

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 4 rows (r0..r3) x box_cols columns starting at column c0 -> dst (row-major,
// contiguous); completion counted on `bar` in bytes.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t r0, int32_t r1, int32_t r2,
                                            int32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}

// a box_rows x box_cols tile at (c0, r0) -> dst
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t r0) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0)
      : "memory");
}

#endif  // DG_TMA_CUH
