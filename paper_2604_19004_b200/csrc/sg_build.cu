// sg_build.cu — canonical CSR construction on the device: COO triplets ->
// CSR with duplicates summed (reference csr.py:52-80, from_triplets) and the
// exact transpose used by the AA^T mode (csr.py:90-97).
//
// Both are one stable 64-bit key sort (key = row * ncols + col; CUB onesweep
// radix sort over only the bits the key range needs, the original position as
// the payload so equal keys keep input order), then three streaming kernels:
// run heads + scan (unique positions), run reduction in input order (the
// reference's stable argsort + add.reduceat order), and row_ptr by binary
// search of each row's first key.  Every pass is a coalesced HBM sweep.
#include <cub/device/device_radix_sort.cuh>

#include "sg_internal.cuh"

namespace sg {

namespace {

__global__ void k_coo_keys(int64_t n, int64_t nrows, int64_t ncols, const int64_t* __restrict__ rows,
                           const int64_t* __restrict__ cols, unsigned long long* __restrict__ keys,
                           uint32_t* __restrict__ idx, int* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[i], c = cols[i];
    if (r < 0 || r >= nrows || c < 0 || c >= ncols) {
      *bad = 1;
      keys[i] = 0;
    } else {
      keys[i] = (unsigned long long)r * (unsigned long long)ncols + (unsigned long long)c;
    }
    idx[i] = (uint32_t)i;
  }
}

// transpose keys: entry j of row r, column c -> key c * nrows + r
__global__ void k_transpose_keys(int64_t nrows, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col, unsigned long long* __restrict__ keys,
                                 uint32_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrows; r += nw) {
    const int64_t s = row_ptr[r], e = row_ptr[r + 1];
    for (int64_t j = s + lane; j < e; j += 32) {
      keys[j] = (unsigned long long)col[j] * (unsigned long long)nrows + (unsigned long long)r;
      idx[j] = (uint32_t)j;
    }
  }
}

__global__ void k_run_heads(int64_t n, const unsigned long long* __restrict__ keys, int64_t* __restrict__ head) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per run head: sum the run's values in input order (stable sort
// payload), write the unique key's column and value at its scanned position
template <typename V>
__global__ void k_run_reduce(int64_t n, int64_t ncols, const unsigned long long* __restrict__ keys,
                             const uint32_t* __restrict__ idx, const int64_t* __restrict__ pos,
                             const V* __restrict__ vals, unsigned long long* __restrict__ ukeys,
                             int32_t* __restrict__ col_out, V* __restrict__ val_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    if (i > 0 && keys[i - 1] == k) continue;
    double s = (double)vals[idx[i]];
    for (int64_t j = i + 1; j < n && keys[j] == k; ++j) s += (double)vals[idx[j]];
    const int64_t p = pos[i];
    ukeys[p] = k;
    col_out[p] = (int32_t)(k % (unsigned long long)ncols);
    val_out[p] = (V)s;
  }
}

// row_ptr[r] = first unique key >= r * ncols (r = 0..nrows)
__global__ void k_row_ptr_search(int64_t nrows, int64_t ncols, int64_t nu,
                                 const unsigned long long* __restrict__ ukeys, int64_t* __restrict__ row_ptr) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long target = (unsigned long long)r * (unsigned long long)ncols;
    int64_t lo = 0, hi = nu;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < target) lo = mid + 1; else hi = mid;
    }
    row_ptr[r] = lo;
  }
}

// transpose emission: keys are unique, so position = sorted position
template <typename V>
__global__ void k_transpose_emit(int64_t n, int64_t nrows_a, const unsigned long long* __restrict__ keys,
                                 const uint32_t* __restrict__ idx, const V* __restrict__ vals,
                                 int32_t* __restrict__ t_col, V* __restrict__ t_val) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    t_col[i] = (int32_t)(keys[i] % (unsigned long long)nrows_a);
    t_val[i] = vals[idx[i]];
  }
}

int key_bits(unsigned long long max_key) {
  int b = 1;
  while (b < 64 && (max_key >> b) != 0) ++b;
  return b;
}

// workspace: keys[2][n] u64, idx[2][n] u32, pos[n+1] i64, partials, flag, cub temp
struct BuildWs {
  unsigned long long* k0;
  unsigned long long* k1;
  uint32_t* i0;
  uint32_t* i1;
  int64_t* pos;
  int64_t* partials;
  int* bad;
  void* cub_tmp;
  size_t cub_bytes;
};

size_t cub_sort_bytes(int64_t n) {
  size_t b = 0;
  cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, b, dk, dv, (int)std::max<int64_t>(n, 1), 0, 64);
  return b;
}

size_t build_bytes(int64_t n) {
  size_t b = 0;
  b += 2 * align256(8 * (size_t)n);
  b += 2 * align256(4 * (size_t)n);
  b += align256(8 * ((size_t)n + 1));
  b += align256(8 * ((size_t)scan_tiles(n + 1) + 2));
  b += align256(8);
  b += align256(cub_sort_bytes(n));
  return b + 256;
}

bool carve_build(void* ws, size_t ws_bytes, int64_t n, BuildWs& w) {
  const size_t need = build_bytes(n);
  if (ws == nullptr || ws_bytes < need) {
    set_error("build workspace too small: need " + std::to_string(need) + " bytes, got " +
              std::to_string(ws_bytes));
    return false;
  }
  uintptr_t p = (reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255);
  w.k0 = reinterpret_cast<unsigned long long*>(p);
  p += align256(8 * (size_t)n);
  w.k1 = reinterpret_cast<unsigned long long*>(p);
  p += align256(8 * (size_t)n);
  w.i0 = reinterpret_cast<uint32_t*>(p);
  p += align256(4 * (size_t)n);
  w.i1 = reinterpret_cast<uint32_t*>(p);
  p += align256(4 * (size_t)n);
  w.pos = reinterpret_cast<int64_t*>(p);
  p += align256(8 * ((size_t)n + 1));
  w.partials = reinterpret_cast<int64_t*>(p);
  p += align256(8 * ((size_t)scan_tiles(n + 1) + 2));
  w.bad = reinterpret_cast<int*>(p);
  p += align256(8);
  w.cub_tmp = reinterpret_cast<void*>(p);
  w.cub_bytes = cub_sort_bytes(n);
  return true;
}

// stable sort of (k0, i0); returns the buffers holding the sorted data
int sort_pairs(BuildWs& w, int64_t n, int end_bit, cudaStream_t s, unsigned long long** keys, uint32_t** idx) {
  cub::DoubleBuffer<unsigned long long> dk(w.k0, w.k1);
  cub::DoubleBuffer<uint32_t> dv(w.i0, w.i1);
  size_t bytes = w.cub_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(w.cub_tmp, bytes, dk, dv, (int)n, 0, end_bit, s);
  if (e != cudaSuccess) {
    set_error(std::string("radix sort: ") + cudaGetErrorString(e));
    return SG_ERR_CUDA;
  }
  count_launches(end_bit / 8 + 2);
  *keys = dk.Current();
  *idx = dv.Current();
  return SG_OK;
}

int grid_stride(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 16); }

}  // namespace

}  // namespace sg

using namespace sg;

extern "C" {

size_t sg_build_workspace_bytes(int64_t nnz) { return build_bytes(nnz < 0 ? 0 : nnz); }

int sg_coo_to_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                  const void* vals, int dtype, int64_t* row_ptr, int32_t* col_out, void* val_out,
                  int64_t* nnz_out_host, void* ws, size_t ws_bytes, void* stream) {
  if (nrows < 0 || ncols < 0 || nnz < 0 || nrows >= ((int64_t)1 << 31) || ncols >= ((int64_t)1 << 31) ||
      nnz >= ((int64_t)1 << 31) || !row_ptr || !nnz_out_host || (dtype != SG_F64 && dtype != SG_F32)) {
    set_error("sg_coo_to_csr: bad arguments");
    return SG_ERR_ARG;
  }
  BuildWs w;
  if (!carve_build(ws, ws_bytes, nnz, w)) return SG_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  *nnz_out_host = 0;
  if (nnz == 0 || ncols == 0) {
    if (nnz != 0) {
      set_error("sg_coo_to_csr: coordinate out of range");
      return SG_ERR_ARG;
    }
    cudaMemsetAsync(row_ptr, 0, 8 * ((size_t)nrows + 1), s);
    return check_cuda("sg_coo_to_csr memset", 0);
  }
  cudaMemsetAsync(w.bad, 0, sizeof(int), s);
  k_coo_keys<<<grid_stride(nnz), 256, 0, s>>>(nnz, nrows, ncols, rows, cols, w.k0, w.i0, w.bad);
  if (int rc = check_cuda("k_coo_keys")) return rc;
  unsigned long long *keys, *ukeys;
  uint32_t* idx;
  const int bits = key_bits((unsigned long long)nrows * (unsigned long long)ncols - 1ull);
  if (int rc = sort_pairs(w, nnz, bits, s, &keys, &idx)) return rc;
  k_run_heads<<<grid_stride(nnz), 256, 0, s>>>(nnz, keys, w.pos);
  if (int rc = check_cuda("k_run_heads")) return rc;
  if (int rc = scan_i64(nnz, w.pos, w.pos, w.partials, s)) return rc;
  // the other key buffer receives the unique keys
  ukeys = keys == w.k0 ? w.k1 : w.k0;
  if (dtype == SG_F64)
    k_run_reduce<double><<<grid_stride(nnz), 256, 0, s>>>(nnz, ncols, keys, idx, w.pos, (const double*)vals, ukeys,
                                                          col_out, (double*)val_out);
  else
    k_run_reduce<float><<<grid_stride(nnz), 256, 0, s>>>(nnz, ncols, keys, idx, w.pos, (const float*)vals, ukeys,
                                                         col_out, (float*)val_out);
  if (int rc = check_cuda("k_run_reduce")) return rc;
  int64_t nu = 0;
  int bad = 0;
  cudaMemcpyAsync(&nu, w.pos + nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&bad, w.bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_coo_to_csr sync", 0);
  if (bad) {
    set_error("sg_coo_to_csr: coordinate out of range");
    return SG_ERR_ARG;
  }
  k_row_ptr_search<<<grid_stride(nrows + 1), 256, 0, s>>>(nrows, ncols, nu, ukeys, row_ptr);
  if (int rc = check_cuda("k_row_ptr_search")) return rc;
  *nnz_out_host = nu;
  return SG_OK;
}

int sg_transpose(int64_t nrows, int64_t ncols, const int64_t* row_ptr, const int32_t* col, const void* val,
                 int dtype, int64_t* t_ptr, int32_t* t_col, void* t_val, void* ws, size_t ws_bytes,
                 void* stream) {
  if (nrows < 0 || ncols < 0 || !row_ptr || !t_ptr || (dtype != SG_F64 && dtype != SG_F32)) {
    set_error("sg_transpose: bad arguments");
    return SG_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nnz = 0;
  cudaMemcpyAsync(&nnz, row_ptr + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_transpose sync", 0);
  BuildWs w;
  if (!carve_build(ws, ws_bytes, nnz, w)) return SG_ERR_WORKSPACE;
  if (nnz == 0 || nrows == 0) {
    cudaMemsetAsync(t_ptr, 0, 8 * ((size_t)ncols + 1), s);
    return check_cuda("sg_transpose memset", 0);
  }
  k_transpose_keys<<<grid_stride(nrows * 32), 256, 0, s>>>(nrows, row_ptr, col, w.k0, w.i0);
  if (int rc = check_cuda("k_transpose_keys")) return rc;
  unsigned long long* keys;
  uint32_t* idx;
  const int bits = key_bits((unsigned long long)ncols * (unsigned long long)nrows - 1ull);
  if (int rc = sort_pairs(w, nnz, bits, s, &keys, &idx)) return rc;
  if (dtype == SG_F64)
    k_transpose_emit<double><<<grid_stride(nnz), 256, 0, s>>>(nnz, nrows, keys, idx, (const double*)val, t_col,
                                                              (double*)t_val);
  else
    k_transpose_emit<float><<<grid_stride(nnz), 256, 0, s>>>(nnz, nrows, keys, idx, (const float*)val, t_col,
                                                             (float*)t_val);
  if (int rc = check_cuda("k_transpose_emit")) return rc;
  // sorted keys are unique: row_ptr of A^T by binary search over them
  k_row_ptr_search<<<grid_stride(ncols + 1), 256, 0, s>>>(ncols, nrows, nnz, keys, t_ptr);
  return check_cuda("k_row_ptr_search");
}

}  // extern "C"
