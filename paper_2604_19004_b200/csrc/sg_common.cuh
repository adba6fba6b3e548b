// sg_common.cuh — shared device helpers for the sm_100a SpGEMM kernels.
//
// Data layout in HBM: CSR with int64 row_ptr, int32
// col_idx, fp64 (or fp32) values; per-row metadata arrays are int64.  All
// kernels are plain CUDA C++ for sm_100a: the path is an irregular, memory-
// bound gather/hash reduction, so no tensor cores are used.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define SG_WARP 32
#define SG_FULL 0xffffffffu

namespace sg {

// splitmix64 finaliser: the reference's hash64 (hll.py:34-49).
__device__ __forceinline__ uint64_t hash64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// HLL register index / rank (hll.py:64-76): idx = h & (m-1),
// rank = (64-p) - bit_length(h >> p) + 1 == clz64(h >> p) - p + 1.
__device__ __forceinline__ void hll_index_rank(uint32_t key, int p, uint32_t& idx,
                                               uint32_t& rank) {
  uint64_t h = hash64((uint64_t)key);
  idx = (uint32_t)(h & ((1ull << p) - 1));
  rank = (uint32_t)(__clzll((long long)(h >> p)) - p + 1);
}

// accumulator table hash (internal; output order never depends on it)
__device__ __forceinline__ uint32_t slot_hash(uint32_t col, int log2t) {
  return (col * 0x9E3779B1u) >> (32 - log2t);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(SG_FULL, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(SG_FULL, v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(SG_FULL, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// inclusive warp scan
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(SG_FULL, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total
// through *total.  `scratch` needs (blockDim/32 + 1) entries of T.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* scratch, T* total) {
  const int lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) scratch[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane < nw ? scratch[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) scratch[lane] = si - s;
    if (lane == nw - 1) scratch[nw] = si;
  }
  __syncthreads();
  T out = scratch[w] + inc - v;
  if (total) *total = scratch[nw];
  __syncthreads();
  return out;
}

// fp64 add into shared memory (sm_100a lowers this to a CAS loop; see
// SURVEY §2.2) and fire-and-forget fp64 add into global memory (REDG.ADD.F64).
__device__ __forceinline__ void smem_add(double* p, double v) { atomicAdd(p, v); }
__device__ __forceinline__ void gmem_red(double* p, double v) { atomicAdd(p, v); }
__device__ __forceinline__ void gmem_red(float* p, float v) { atomicAdd(p, v); }

// Output of C and the saved key bitmaps stream through L2 once: store them
// evict-first (st.global.cs) so the gathered B rows stay L2-resident.
__device__ __forceinline__ void st_stream(int32_t* p, int32_t v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(unsigned long long* p, unsigned long long v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream_v4(uint4* p, uint4 v) { __stcs(p, v); }

__device__ __forceinline__ uint32_t next_pow2_u32(uint32_t x) {
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}

}  // namespace sg
