// sg_internal.cuh — host-side helpers shared by the .cu translation units.
#pragma once
#include <cstdio>
#include <string>

#include "../../include/sgb200.h"
#include "sg_common.cuh"

namespace sg {

void set_error(const std::string& msg);

// Workspace carve-up (sizes in bytes, 256-aligned).  Every stage takes the
// same `ws` block; regions are reused between stages.
struct Workspace {
  uint8_t* bins;        // uint8[m]   per-row bin id
  int32_t* rowlist;     // int32[m]   rows grouped by bin
  int64_t* tmp;         // int64[m+1] flags / scan scratch
  int64_t* partials;    // int64[nb+2] scan block partials
  int64_t* bincnt;      // int64[256] bin histogram + cursors + tickets
  size_t bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline int64_t scan_tiles(int64_t n) { return (n + 4095) / 4096; }

inline size_t workspace_bytes(int64_t m) {
  size_t b = 0;
  b += align256((size_t)m);
  b += align256(4 * (size_t)m);
  b += align256(8 * ((size_t)m + 1));
  b += align256(8 * ((size_t)scan_tiles(m + 1) + 2));
  b += align256(8 * 256);
  return b + 256;
}

inline bool carve(void* ws, size_t ws_bytes, int64_t m, Workspace& w) {
  size_t need = workspace_bytes(m);
  if (ws == nullptr || ws_bytes < need) {
    set_error("workspace too small: need " + std::to_string(need) + " bytes, got " +
              std::to_string(ws_bytes));
    return false;
  }
  uintptr_t p = (reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255);
  w.bins = reinterpret_cast<uint8_t*>(p);
  p += align256((size_t)m);
  w.rowlist = reinterpret_cast<int32_t*>(p);
  p += align256(4 * (size_t)m);
  w.tmp = reinterpret_cast<int64_t*>(p);
  p += align256(8 * ((size_t)m + 1));
  w.partials = reinterpret_cast<int64_t*>(p);
  p += align256(8 * ((size_t)scan_tiles(m + 1) + 2));
  w.bincnt = reinterpret_cast<int64_t*>(p);
  w.bytes = need;
  return true;
}

// diagnostic launch counter (sg_launch_count); incremented by check_cuda
void count_launches(int n);

// per-kernel CUDA-event timer (sg_kernel_timer / sg_kernel_time): when
// enabled, ktimer_begin/ktimer_end bracket a launch with events recorded on
// the launching stream; a no-op otherwise
bool ktimer_on();
void ktimer_begin(const char* name, cudaStream_t s);
void ktimer_end(cudaStream_t s);

// returns SG_OK or SG_ERR_CUDA with the message recorded; `launches` is the
// number of kernels the caller just enqueued
inline int check_cuda(const char* where, int launches = 1) {
  count_launches(launches);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return SG_ERR_CUDA;
  }
  return SG_OK;
}

inline int grid_for(int64_t work_items, int per_block) {
  int64_t g = (work_items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return (int)g;
}

// exclusive scan used internally (defined in sg_analysis.cu)
int scan_i64(int64_t n, const int64_t* in, int64_t* out, int64_t* partials, cudaStream_t s);

// Partition rows 0..m-1 by bins[] (values < nbins) into w.rowlist; fills
// cnt_host[nbins] and off_host[nbins+1].  Synchronises the stream once.
int partition_rows(int64_t m, int nbins, Workspace& w, int64_t* cnt_host, int64_t* off_host,
                   cudaStream_t s);

}  // namespace sg
