// common.cu -- error state, launch counter, device memory / CUDA-IPC
// plumbing and native host preprocessing of the libdgb200 C ABI.

#include "common.cuh"

namespace dg {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace dg

extern "C" {

const char* dg_last_error(void) { return dg::g_err.c_str(); }
int dg_version(void) { return 2; }
int64_t dg_launch_count(void) { return dg::g_launches.load(); }
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
// host preprocessing (native): symmetric permutation P A P^T
// (partition.apply_partition, partition.py:231-254: new ids perm[], entries
// ordered by (new row, new col) -- the (row, col) keys are unique, so the
// result equals the reference's lexsort exactly)
// ---------------------------------------------------------------------------

extern "C" int dg_host_permute(int64_t n, const int64_t* row_ptr, const int64_t* col,
                               const double* val, const int64_t* perm, int64_t* out_row_ptr,
                               int64_t* out_col, double* out_val) {
  if (n < 0) return set_err(DG_ERR_ARG, "permute: bad n");
  std::vector<int64_t> inv(n);
  for (int64_t i = 0; i < n; ++i) {
    if (perm[i] < 0 || perm[i] >= n) return set_err(DG_ERR_ARG, "permute: perm out of range");
    inv[perm[i]] = i;
  }
  out_row_ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t o = inv[r];
    out_row_ptr[r + 1] = out_row_ptr[r] + (row_ptr[o + 1] - row_ptr[o]);
  }
  std::vector<std::pair<int64_t, double>> tmp;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t o = inv[r];
    const int64_t lo = row_ptr[o], len = row_ptr[o + 1] - lo;
    tmp.resize(len);
    for (int64_t k = 0; k < len; ++k) tmp[k] = {perm[col[lo + k]], val[lo + k]};
    std::sort(tmp.begin(), tmp.end(),
              [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& b) {
                return a.first < b.first;
              });
    const int64_t d = out_row_ptr[r];
    for (int64_t k = 0; k < len; ++k) {
      out_col[d + k] = tmp[k].first;
      out_val[d + k] = tmp[k].second;
    }
  }
  return DG_OK;
}
