/*
 * dgb200.h -- C ABI of the B200 sparsity-aware distributed SpMM library.
 *
 * The reference (`distgcn` 0.1.0, /root/reference/pkg) is pure Python/NumPy
 * with no FFI; these entry points are what its Python hot path would bind
 * (via ctypes) to move onto the GPU.  Each one names the reference
 * function(s) it replaces.  Plain pointers and sizes only; device pointers
 * are marked (device).  Every function returns DG_OK (0) or a negative
 * error code; dg_last_error() holds the message (thread-local).
 *
 * Streams are passed as `void*` (a cudaStream_t).  All calls are
 * asynchronous on that stream unless stated otherwise.  Memory passed in
 * (H, Z, halo buffers) is owned by the caller; plan objects own the
 * device copies of the sparse operand and the exchange lists and free them
 * in the matching *_destroy.
 */
#ifndef DGB200_H
#define DGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_OK 0
#define DG_ERR_CUDA -1
#define DG_ERR_ARG -2
#define DG_ERR_TIMEOUT -3
#define DG_MAX_LOCAL 64   /* ranks one process may host (virtual ranks per GPU) */
#define DG_MAX_GROUP 64   /* members of one reduction group */

const char* dg_last_error(void);
int dg_version(void);
/* number of kernels this library launched since load (bench's gpu_launches) */
int64_t dg_launch_count(void);
int dg_device_sync(void);

/* ---- device memory / peers (the reference's in-process mailbox,
 *      runtime.py:237-248, becomes symmetric device buffers) ----------- */
int dg_malloc(void** ptr, int64_t bytes);          /* zero-filled cudaMalloc */
int dg_free(void* ptr);
int dg_memset0(void* ptr, int64_t bytes, void* stream);
int dg_enable_peer(int peer_device);               /* from the current device */
int dg_ipc_get_handle(void* dev_ptr, uint8_t handle_out[64]);
int dg_ipc_open_handle(const uint8_t handle[64], void** dev_ptr_out);
int dg_ipc_close(void* dev_ptr);

/* ---- local SpMM: replaces sparse.local_spmm (sparse.py:208-223) and the
 *      per-block loops of spmm._kernel_1d_* / _kernel_15d (spmm.py:172-227).
 *
 * One plan covers the `n_ranks` ranks hosted by this process.  Rank r's
 * operand is its block row as CSR over an EXTENDED column space:
 * ext < n_local[r] reads row ext of the rank's own H block; ext >= n_local[r]
 * reads row (ext - n_local[r]) of its halo buffer (rows received from peers).
 * Entries stay in the reference's storage order (ascending global column),
 * which fixes the summation order: the aware and oblivious forms of a
 * variant -- and 1.5D with c = 1 vs 1D -- are bitwise identical.
 * Host arrays are copied; long rows are split into fixed chunks of at most
 * `max_chunk` nonzeros and reduced in a fixed order (deterministic).     */
typedef struct dg_spmm_plan dg_spmm_plan;
#define DG_PLAN_SKIP_EMPTY_ROWS 1  /* no work items for rows without entries (z untouched) */
#define DG_PLAN_DEVICE_SRC 2       /* col_ext / val are DEVICE arrays (row_ptr stays host):
                                      the entries are laid out on the GPU (graphs built in HBM) */
int dg_spmm_plan_create(dg_spmm_plan** plan, int n_ranks,
                        const int64_t* n_rows, const int64_t* n_local, const int64_t* nnz,
                        const int64_t* const* row_ptr, const int32_t* const* col_ext,
                        const float* const* val, int32_t max_chunk, int32_t flags);
/* As dg_spmm_plan_create, plus a processing order: row_order[r] (host, nullable; a
 * permutation of rank r's rows) is the order in which rows are scheduled, e.g. rows
 * grouped by graph community so the H rows gathered together stay L2-resident.  Items
 * are bucketed by length only inside windows of ~window_nnz entries (<= 0: chosen from
 * the graph -- DG_SPMM_WINDOW_NNZ when at least a quarter of the own-block entries are
 * processed within one window of their row, else one global window).  The order and the
 * window change no result: every row is still summed in its CSR storage order
 * (bit-identical output).  dg_spmm_plan_info reports the window in info[6]. */
#define DG_SPMM_WINDOW_NNZ (1LL << 20)
int dg_spmm_plan_create_ordered(dg_spmm_plan** plan, int n_ranks,
                                const int64_t* n_rows, const int64_t* n_local, const int64_t* nnz,
                                const int64_t* const* row_ptr, const int32_t* const* col_ext,
                                const float* const* val, int32_t max_chunk, int32_t flags,
                                const int32_t* const* row_order, int64_t window_nnz);
int dg_spmm_plan_destroy(dg_spmm_plan* plan);
/* Size the plan's fp64 split-row partial buffer for row pitches up to ld_max, so that
 * dg_spmm_run never allocates (it refuses to grow the buffer inside a stream capture). */
int dg_spmm_plan_reserve(dg_spmm_plan* plan, int64_t ld_max);
/* Fused forward epilogue (gcn.py:273-276): z[r] = (A_r [H_r; halo_r]) W and,
 * when h_relu is given, h_relu[r] = relu(z[r]) -- the product T never reaches HBM.  For
 * 13 <= f <= 16 (one float4 per lane of a 4-lane group), W is f x n_out (row pitch ld_w,
 * device), n_out <= 64, z / h_relu rows of pitch ld_z (>= n_out, padding written as 0).
 * Single-pass plans only (no split own/halo passes, no 1.5D partials).  T is summed
 * exactly as dg_spmm_run sums it; z = t W in fp32 in ascending k. */
int dg_spmm_run_fused(dg_spmm_plan* plan, const float* const* h_local,
                      const float* const* h_halo, float* const* z, float* const* h_relu,
                      int32_t f, int64_t ld_h, int64_t ld_z, const float* w, int64_t ld_w,
                      int32_t n_out, void* stream);
/* info[0]=items, [1]=split rows, [2]=chunks, [3]=total nnz, [4]=device bytes,
 * [5]=extended rows, [6]=length-bucketing window (entries) */
int dg_spmm_plan_info(const dg_spmm_plan* plan, int64_t info[8]);
/* z[r] (n_rows[r] x ld_z, device) = A_r @ [h_local[r]; h_halo[r]] (ld_h).
 * f <= ld_h, ld_h % 4 == 0, ld_z % 4 == 0.  acc: 0 = fp32 accumulate,
 * 1 = fp32 4-entry windows folded into fp64, 2 = two-level fp32 (32-entry
 * windows folded into an fp32 sum; <= (32 + len/32) ulp of the row's
 * sum of |terms|, <= 64 ulp per 1024-entry item; used for rows > 48 floats
 * (and 9..16-float rows of tables > 1 GB); other rows use mode 1).  slab_floats: feature-slab width (0 = auto: sized
 * so one slab of the gathered rows stays L2-resident).  beta = 1 adds the
 * product to z (the halo pass of a phase whose own-block pass overlapped
 * the exchange).                                                        */
int dg_spmm_run(dg_spmm_plan* plan, const float* const* h_local, const float* const* h_halo,
                float* const* z, int32_t f, int64_t ld_h, int64_t ld_z, int32_t acc,
                int32_t slab_floats, int32_t beta, void* stream);

/* ---- halo exchange: replaces the pack `h_block[NnzCols(dst, me)]`
 *      (spmm.py:185, 212), Comm.all_to_allv / isend / broadcast
 *      (runtime.py:311-435) and the receiver-side `_scatter`
 *      (spmm.py:166-169).  One fused gather + (peer) store kernel: every
 *      segment copies rows idx[k] (or src_row0 + k when idx is NULL) of the
 *      source rank's H into `count` consecutive rows of a destination halo
 *      buffer, which may live on a peer GPU (P2P / CUDA-IPC mapped).       */
typedef struct dg_xchg_plan dg_xchg_plan;
int dg_xchg_plan_create(dg_xchg_plan** plan, int n_segs, const int32_t* src_local,
                        const int64_t* count, const int32_t* const* idx /* host, device or NULL */,
                        const int64_t* src_row0, const int32_t* dst_buf,
                        const int64_t* dst_row0);
int dg_xchg_plan_destroy(dg_xchg_plan* plan);
/* dst_bufs[b] = base of halo buffer b (device; local or peer-mapped);
 * fence_sys != 0 ends the kernel with a system-scope fence (cross-process). */
int dg_xchg_run(dg_xchg_plan* plan, const float* const* h_src, int n_src,
                float* const* dst_bufs, int n_dst, int32_t f, int64_t ld, int32_t fence_sys,
                void* stream);
/* Same, with at most max_ctas CTAs in flight over all segments (0: no cap,
 * as dg_xchg_run).  An exchange overlapped with the own-block SpMM passes a
 * cap so the SpMM keeps most SMs.                                        */
int dg_xchg_run_ctas(dg_xchg_plan* plan, const float* const* h_src, int n_src,
                     float* const* dst_bufs, int n_dst, int32_t f, int64_t ld,
                     int32_t fence_sys, int32_t max_ctas, void* stream);

/* ---- group all-reduce: replaces Comm.all_reduce_sum (runtime.py:437-466).
 * For elements [lo, hi): s = src[0] + src[1] + ... + src[g-1] (ascending
 * member order, the reference's order), stored to dst[0..n_dst).  Every
 * member that reduces the same range in the same order gets bit-identical
 * values.  Sources may be peer-mapped (CUDA IPC / P2P over NVLink).       */
int dg_group_reduce(int g, const float* const* src, int n_dst, float* const* dst, int64_t lo,
                    int64_t hi, int32_t fence_sys, void* stream);

/* ---- cross-process barrier over peer-mapped flag words (device-side;
 *      one process per GPU).  flags[q] points at process q's flag array;
 *      each process writes `epoch` to slot `me` of every peer and waits for
 *      all slots of its own array to reach `epoch`.  Bounded by timeout_ns;
 *      on timeout sets *err_dev = 1 and traps: the context faults, so no
 *      later kernel computes on stale halos and the host's next
 *      synchronisation reports the error (fail closed, no hang).         */
int dg_barrier(uint64_t* const* flags, int n_procs, int me, uint64_t epoch,
               int64_t timeout_ns, int32_t* err_dev, void* stream);

/* ---- GCN loss: replaces gcn._xent_parts (gcn.py:98-120).  Masked
 *      softmax cross-entropy; grad = (softmax - onehot) / denom on masked
 *      rows, 0 elsewhere; stats_out[0] += loss sum, stats_out[1] += correct
 *      (first-index argmax, like np.argmax).  Deterministic (fixed-order
 *      block reduction).  Labels of masked rows must lie in [0, C) (the
 *      host validates them, as _xent_parts raises ValueError); unmasked
 *      rows may carry any label.  scratch: >= 2 * ceil(n / 8) + 2 doubles. */
int dg_xent(const float* logits, int64_t n, int32_t C, int64_t ld, const int64_t* labels,
            const uint8_t* mask, double denom, float* grad, int64_t ld_grad,
            double* scratch, uint32_t* counter, double* stats_out, void* stream);

/* ---- elementwise pieces of the GCN step (gcn.py:76-82, 276, 282-283) ---- */
int dg_relu(const float* z, float* h, int64_t rows, int32_t f, int64_t ld, void* stream);
/* g[i, :f] *= (zprev[i, :f] > 0) */
int dg_relu_grad_mul(float* g, int64_t ld_g, const float* zprev, int64_t ld_z,
                     int64_t rows, int32_t f, void* stream);
/* w -= lr * y  (n contiguous floats) */
int dg_sgd(float* w, const float* y, int64_t n, float lr, void* stream);

/* ---- dense transforms of the GCN step (gcn.py:274-282), fp32 SIMT,
 *      HBM-bound tall-skinny shapes (cuBLAS picks SIMT kernels ~4x off
 *      bandwidth for these).
 * dg_dense_rows: C[r, :] = A[r, :K] @ B (K x N; transB: B is N x K, i.e.
 *   W^T), N <= 64, K * roundup16(N) <= 16384.  Optional epilogues:
 *   C_relu = max(C, 0) (gcn.py:276); C *= 1[z_mask > 0] (gcn.py:282).
 *   Columns [N, ldc) of C are written as zeros.
 * dg_dense_tn: Y (K x ldy) = H[:, :K]^T @ M[:, :N], reduced over the n rows
 *   (gcn.py:280), deterministically: per-slice partials in fp64, summed in
 *   slice order.  work: >= dg_dense_tn_work(n, K, N) doubles.            */
int dg_dense_rows(const float* A, int64_t lda, int64_t n, int32_t K, const float* B, int64_t ldb,
                  int32_t N, int32_t transB, float* C, int64_t ldc, float* C_relu,
                  const float* z_mask, int64_t ld_mask, void* stream);
int64_t dg_dense_tn_work(int64_t n, int32_t K, int32_t N);
int dg_dense_tn(const float* H, int64_t ldh, int64_t n, int32_t K, const float* M, int64_t ldm,
                int32_t N, float* Y, int64_t ldy, double* work, int64_t work_len, void* stream);

/* ---- diagnostic: random-row gather bandwidth probe (the practical ceiling
 *      of the SpMM's H-row gathers; used by scripts/gather_roofline.py).
 *      `groups` groups of `lanes` lanes each sum `per_group` rows tab[idx[k]]
 *      of 16*lanes bytes.                                                  */
int dg_diag_gather(const float* tab, int64_t ld, const int32_t* idx, int64_t n_idx,
                   int32_t lanes, int64_t groups, int32_t per_group, float* out, void* stream);
/* Diagnostic: the same random-row gather through TMA tile::gather4 into a shared-memory
 * ring (one producer lane per CTA, mbarrier-tracked).  Rows idx[k] (n_idx a multiple of 4,
 * 16-B aligned) of a (rows x ld) fp32 table, box_cols floats from column col0; variant
 * selects ring depth / rows per stage (probe.cu); ctas CTAs. */
int dg_diag_gather_tma(const float* tab, int64_t ld, int64_t rows, int32_t col0,
                       int32_t box_cols, const int32_t* idx, int64_t n_idx, int32_t variant,
                       int32_t ctas, float* out, void* stream);

/* ---- host preprocessing: stable O(nnz + n) transpose, bit-identical to
 *      sparse.transpose_csr (sparse.py:237-247).  Host pointers.          */
int dg_host_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                      const int64_t* col, const double* val, int64_t* out_row_ptr,
                      int64_t* out_col, double* out_val);

/* ---- host preprocessing: symmetric permutation P A P^T (new id perm[i]),
 *      equal to partition.apply_partition (partition.py:231-254).          */
int dg_host_permute(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                    const int64_t* perm, int64_t* out_row_ptr, int64_t* out_col,
                    double* out_val);

/* ---- host preprocessing: the reference's partitioners, same visiting
 *      orders / tie-breaks / float64 comparisons (identical assignments).
 *      greedy_tv_partition (partition.py:257-339) over the symmetric
 *      pattern `p*` (no diagonal); volume_balanced_refine (partition.py:
 *      342-428) over A (`a*`), A^T (`at*`) and the pattern's row_ptr.     */
int dg_host_greedy_tv(int64_t n, const int64_t* pat_row_ptr, const int64_t* pat_col, int32_t k,
                      double epsilon, int32_t max_passes, int64_t* assignment, int32_t* relaxed);
int dg_host_gvb(int64_t n, const int64_t* a_row_ptr, const int64_t* a_col,
                const int64_t* at_row_ptr, const int64_t* at_col, const int64_t* pat_row_ptr,
                int32_t k, double lambda_max, double epsilon, int32_t max_passes,
                int64_t* assignment);

#ifdef __cplusplus
}
#endif
#endif /* DGB200_H */
