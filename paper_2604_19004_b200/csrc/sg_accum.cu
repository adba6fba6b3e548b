// sg_accum.cu — the accumulators: symbolic counting, numeric Gustavson pass,
// fallback re-execution.  Hot path of the estimation-based SpGEMM.
//
// Reference semantics (all exact; only the summation order of values may
// differ, as it already does between the reference's own bins):
//   symbolic_pass            predict.py:39-84         -> count mode
//   accumulate_hash_like     accumulate.py:335-365    -> hash families, limit floor(0.8 cap)
//   accumulate_esc           accumulate.py:368-378    -> ESC family
//   accumulate_dense         accumulate.py:381-430    -> bitmap family, limit alloc
//   _fallback_phase          engine.py:312-328        -> bitmap family, no limit
//   _sort_hash_rows          engine.py:331-343        -> fused: rows leave sorted
//
// GPU accumulator families (chosen per row by a classify kernel, rows grouped
// into bins by a partition pass, one launch per non-empty bin):
//   ESC  warp per row, <= 64 products in shared memory, bitonic sort + segment sum
//   HW   warp per row, shared-memory open-addressing hash, T in [32, 2048]
//   HB   block per row, shared-memory hash, T in [2048, 32768]
//   BM   block per row, shared-memory bitmap over the row's column span (up to
//        2^20 columns per window; wider spans loop over windows); count =
//        popcount, output columns come out of the bitmap already sorted, values
//        are accumulated with fire-and-forget fp64 REDs into the row's output
//        slots at rank(col) — the paper's shared+global spill accumulator,
//        with the key side held as a bitmap.
// Product iteration is load balanced inside each row: A-row chunks are
// prefix-summed over their B-row lengths and every warp walks a contiguous
// range of products (CREDUX.OR finds segment owners), so a row with one hub
// B row keeps all warps busy.
#include <array>
#include <type_traits>
#include <map>
#include <mutex>
#include <algorithm>
#include <climits>

#include <cub/block/block_radix_sort.cuh>
#include <string>
#include <vector>
#include <cstdio>

#include "sg_internal.cuh"

namespace sg {

constexpr int64_t NOLIMIT = 0x7fffffffffffffffll;
#ifndef SG_UNR
#define SG_UNR 4
#endif

struct Csr {
  const int64_t* ptr;
  const int32_t* col;
  const void* val;
};

// -------------------------------------------------------------------------
// product iteration

// compacted non-empty A entries of one chunk (shared memory)
struct Entries {
  int64_t* S;   // first product index of the entry within the chunk (excl scan)
  int64_t* d;   // B position of product p of this entry is p + d (B row start - S)
  double* av;   // A value
};

__device__ __forceinline__ unsigned lanemask_le() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// One block of UNR x 32 products of a warp: per step, the lane's A value
// multiplier (already applied) is carried as `a`, the gathered column and B
// value are in registers; `valid` bit u marks steps with a product.
template <int UNR>
struct ProdBlock {
  int32_t col[UNR];
  double v[UNR];
  unsigned valid;
};

// Resolve the owners of products [p0, p0 + 32*UNR) (advancing c0) and issue
// their gathers.  Fast path (warp-uniform): the block lies inside one B-row
// segment, so lanes read consecutive elements and no owner search is needed.
template <bool VALUES, typename V, int UNR>
__device__ __forceinline__ void plan_load(const Entries& E, int nent, int64_t p0, int64_t pend, int& c0,
                                          const int32_t* __restrict__ b_col, const V* __restrict__ b_val,
                                          unsigned le, ProdBlock<UNR>& B) {
  const int lane = lane_id();
  const int64_t blk_end = min(p0 + 32 * UNR, pend);
  const int64_t seg_end = (c0 + 1 < nent) ? E.S[c0 + 1] : (int64_t)NOLIMIT;
  B.valid = 0;
  if (seg_end >= blk_end) {
    const int64_t base = E.d[c0] + p0 + lane;
    const double a = VALUES ? E.av[c0] : 0.0;
    const int nvalid = (int)(blk_end - p0) - lane;
    const int32_t* cp = b_col + base;
    const V* vp = b_val + base;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const bool ok = 32 * u < nvalid;
      B.col[u] = ok ? __ldg(cp + 32 * u) : 0;
      B.v[u] = (VALUES && ok) ? a * (double)__ldg(vp + 32 * u) : 0.0;
      B.valid |= ok ? (1u << u) : 0u;
    }
    if (seg_end == blk_end) ++c0;
    if (c0 >= nent) c0 = nent - 1;
    return;
  }
  int64_t jj[UNR];
  int cc[UNR];
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const int64_t q0 = p0 + 32 * u;
    const int ci = c0 + 1 + lane;
    const int64_t nxt = ci < nent ? E.S[ci] : (int64_t)NOLIMIT;
    const int64_t d = nxt - q0;
    const unsigned bit = (d >= 0 && d < 32) ? (1u << (unsigned)d) : 0u;
    const unsigned mask = __reduce_or_sync(SG_FULL, bit);
    const int c = c0 + __popc(mask & le);
    const int64_t p = q0 + lane;
    cc[u] = c;
    jj[u] = (p < pend) ? E.d[c] + p : -1;
    const int k = __popc(mask);
    const int64_t nk = __shfl_sync(SG_FULL, nxt, k);
    c0 = c0 + k + (nk == q0 + 32 ? 1 : 0);
    if (c0 >= nent) c0 = nent - 1;
  }
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const bool ok = jj[u] >= 0;
    B.col[u] = ok ? __ldg(b_col + jj[u]) : 0;
    B.v[u] = (VALUES && ok) ? E.av[cc[u]] * (double)__ldg(b_val + jj[u]) : 0.0;
    B.valid |= ok ? (1u << u) : 0u;
  }
}

template <int UNR, class Op>
__device__ __forceinline__ void run_ops(const ProdBlock<UNR>& B, Op& op) {
#pragma unroll
  for (int u = 0; u < UNR; ++u)
    if (B.valid & (1u << u)) op(B.col[u], B.v[u]);
}

// The calling warp processes products [pbeg, pend) of a chunk; op(col, val).
// Two-stage software pipeline: the gathers of block k+1 are in flight while
// the (shared-memory) ops of block k run, so each lane keeps 2*UNR L2 round
// trips outstanding instead of stalling on every block.
template <bool VALUES, typename V, class Op>
__device__ __forceinline__ void warp_products(const Entries& E, int nent, int64_t pbeg, int64_t pend,
                                              const int32_t* __restrict__ b_col,
                                              const V* __restrict__ b_val, Op& op) {
  if (pbeg >= pend) return;
  int lo = 0, hi = nent - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (E.S[mid] <= pbeg) lo = mid; else hi = mid - 1;
  }
  int c0 = lo;
  const unsigned le = lanemask_le();
  constexpr int UNR = SG_UNR;
  constexpr int STEP = 32 * UNR;
  ProdBlock<UNR> A, Bk;
  int64_t p = pbeg;
  if (VALUES) {
    // value passes are register-bound at 1024 threads: no prefetch stage
    for (; p < pend; p += STEP) {
      plan_load<VALUES, V, UNR>(E, nent, p, pend, c0, b_col, b_val, le, A);
      run_ops(A, op);
    }
    return;
  }
  plan_load<VALUES, V, UNR>(E, nent, p, pend, c0, b_col, b_val, le, A);
  p += STEP;
  for (;;) {
    const bool hasB = p < pend;
    if (hasB) {
      plan_load<VALUES, V, UNR>(E, nent, p, pend, c0, b_col, b_val, le, Bk);
      p += STEP;
    }
    run_ops(A, op);
    if (!hasB) break;
    const bool hasA = p < pend;
    if (hasA) {
      plan_load<VALUES, V, UNR>(E, nent, p, pend, c0, b_col, b_val, le, A);
      p += STEP;
    }
    run_ops(Bk, op);
    if (!hasA) break;
  }
}

// Block-wide product iteration over a chunk's compacted entries (E.S strictly
// increasing exclusive product prefix, E.d, E.av), products [0, P).
// Products are cut into 32-product groups; a group table built once per
// sub-chunk holds, per group, the entry owning its first product and a
// bitmask of the entries starting inside it, so a lane finds its product's
// entry with one broadcast load and a popcount -- no per-step owner search,
// no dependency between steps (every warp keeps UNR groups of gathers in
// flight).  Sub-chunks of GRP_MAX groups bound the table.
#ifndef SG_GROUPED
#define SG_GROUPED 1
#endif
constexpr int GRP_MAX = 512;
// one table per kernel that iterates (file-scope shared: not duplicated per
// template instantiation of block_products)
__shared__ int2 g_grp[GRP_MAX];

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint2 lds_v2u32(uint32_t a) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
  return r;
}
__device__ __forceinline__ int64_t lds_s64(uint32_t a) {
  int64_t r;
  asm volatile("ld.shared.s64 %0, [%1];" : "=l"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(a));
  return r;
}

template <bool VALUES, typename V, class Op>
__device__ __forceinline__ void block_products(const Entries& E, int nent, int64_t P,
                                               const int32_t* __restrict__ b_col,
                                               const V* __restrict__ b_val, Op& op, int2* grp = g_grp,
                                               int grp_max = GRP_MAX) {
  const uint32_t grp_s = smem_u32(grp), d_s = smem_u32(E.d), av_s = smem_u32(E.av);
  const int nw = blockDim.x >> 5, w = warp_id(), lane = lane_id();
  const unsigned le = lanemask_le();
#ifndef SG_UNR_KEYS
#define SG_UNR_KEYS 8
#endif
  // key passes carry a column per product (values passes a column and a
  // value): twice the gathers in flight at the same register budget
  constexpr int U = VALUES ? SG_UNR : SG_UNR_KEYS;
  for (int64_t base = 0; base < P; base += 32 * (int64_t)grp_max) {
    const int rem = (int)min((int64_t)32 * grp_max, P - base);  // products of this sub-chunk
    const int ng = (rem + 31) >> 5;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
      const int64_t q = base + 32 * (int64_t)g;
      int lo = 0, hi = nent - 1;  // last entry with S <= q
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (E.S[mid] <= q) lo = mid; else hi = mid - 1;
      }
      unsigned mask = 0;
      for (int c = lo + 1; c < nent; ++c) {
        const int64_t dd = E.S[c] - q;
        if (dd >= 32) break;
        mask |= 1u << (unsigned)dd;
      }
      grp[g] = make_int2(lo, (int)mask);
    }
    __syncthreads();
    const int32_t* bc = b_col + base;  // product p of the sub-chunk is at d + p
    const V* bv = b_val + base;
    for (int g0 = w * U; g0 < ng; g0 += nw * U) {
      int32_t col[U];
      double v[U];
      if ((g0 + U) * 32 <= rem) {
        // full step: U groups, every lane has a product (no predicates)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint2 gr = lds_v2u32(grp_s + (uint32_t)(g0 + u) * 8u);
          const uint32_t c = gr.x + (uint32_t)__popc(gr.y & le);
          const int64_t pos = lds_s64(d_s + c * 8u) + (int64_t)((g0 + u) * 32 + lane);
          col[u] = __ldg(bc + pos);
          if (VALUES) v[u] = lds_f64(av_s + c * 8u) * (double)__ldg(bv + pos);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) op(col[u], VALUES ? v[u] : 0.0);
      } else {
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int p = (g0 + u) * 32 + lane;
          ok[u] = p < rem;
          col[u] = 0;
          v[u] = 0.0;
          if (ok[u]) {
            const uint2 gr = lds_v2u32(grp_s + (uint32_t)(g0 + u) * 8u);
            const uint32_t c = gr.x + (uint32_t)__popc(gr.y & le);
            const int64_t pos = lds_s64(d_s + c * 8u) + (int64_t)p;
            col[u] = __ldg(bc + pos);
            if (VALUES) v[u] = lds_f64(av_s + c * 8u) * (double)__ldg(bv + pos);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u]) op(col[u], v[u]);
      }
    }
    __syncthreads();
  }
}

// Load one chunk of A entries for a warp (CH = 32), compacting empties.
// Returns the chunk's product total; nent receives the entry count.
template <bool VALUES, typename V>
__device__ __forceinline__ int64_t warp_load_chunk(int64_t t, int64_t t1, const int32_t* __restrict__ a_col,
                                                   const V* __restrict__ a_val,
                                                   const int64_t* __restrict__ b_ptr, Entries E, int& nent) {
  const int lane = lane_id();
  int64_t bs = 0, len = 0;
  double av = 0.0;
  if (t + lane < t1) {
    const int32_t k = a_col[t + lane];
    bs = b_ptr[k];
    len = b_ptr[k + 1] - bs;
    if (VALUES) av = (double)a_val[t + lane];
  }
  const int64_t incl = warp_incl_scan(len);
  const unsigned nz = __ballot_sync(SG_FULL, len > 0);
  const int pos = __popc(nz & lanemask_lt());
  __syncwarp();
  if (len > 0) {
    E.S[pos] = incl - len;
    E.d[pos] = bs - (incl - len);
    if (VALUES) E.av[pos] = av;
  }
  __syncwarp();
  nent = __popc(nz);
  return __shfl_sync(SG_FULL, incl, 31);
}

// Whole row with one warp.
template <bool VALUES, typename V, class Op>
__device__ __forceinline__ void warp_row(int64_t row, const int64_t* __restrict__ a_ptr,
                                         const int32_t* __restrict__ a_col, const V* __restrict__ a_val,
                                         const int64_t* __restrict__ b_ptr, const int32_t* __restrict__ b_col,
                                         const V* __restrict__ b_val, Entries E, Op& op,
                                         volatile int* stop) {
  const int64_t t1 = a_ptr[row + 1];
  for (int64_t t = a_ptr[row]; t < t1; t += 32) {
    int nent;
    const int64_t P = warp_load_chunk<VALUES, V>(t, t1, a_col, a_val, b_ptr, E, nent);
    if (P > 0) warp_products<VALUES, V>(E, nent, 0, P, b_col, b_val, op);
    __syncwarp();
    if (stop && __shfl_sync(SG_FULL, *stop, 0)) return;
  }
}

// Whole row with the whole block; chunks of blockDim A entries; every warp
// takes a contiguous product range of each chunk.  `stop` (shared) aborts
// between chunks.
template <bool VALUES, typename V, class Op>
__device__ __forceinline__ void block_row(int64_t row, const int64_t* __restrict__ a_ptr,
                                          const int32_t* __restrict__ a_col, const V* __restrict__ a_val,
                                          const int64_t* __restrict__ b_ptr, const int32_t* __restrict__ b_col,
                                          const V* __restrict__ b_val, Entries E, int64_t* scan_scratch,
                                          Op& op, volatile int* stop, int64_t max_len = NOLIMIT,
                                          int2* grp = g_grp, int grp_max = GRP_MAX) {
  const int nw = blockDim.x >> 5, w = warp_id();
  const int64_t t1 = a_ptr[row + 1];
  for (int64_t t = a_ptr[row]; t < t1; t += blockDim.x) {
    int64_t bs = 0, len = 0;
    double av = 0.0;
    if (t + threadIdx.x < t1) {
      const int32_t k = a_col[t + threadIdx.x];
      bs = b_ptr[k];
      len = b_ptr[k + 1] - bs;
      if (len > max_len) len = 0;  // entry filter (k_win_light: light B rows only)
      if (VALUES) av = (double)a_val[t + threadIdx.x];
    }
    // one scan of (len << 12 | nonempty): segment starts and compacted slots
    int64_t tot;
    const int64_t ex = block_excl_scan((len << 12) | (int64_t)(len > 0), scan_scratch, &tot);
    const int64_t S = ex >> 12, pos = ex & 4095, P = tot >> 12, nent64 = tot & 4095;
    if (len > 0) {
      E.S[pos] = S;
      E.d[pos] = bs - S;
      if (VALUES) E.av[pos] = av;
    }
    __syncthreads();
#if SG_GROUPED
    (void)nw;
    (void)w;
    block_products<VALUES, V>(E, (int)nent64, P, b_col, b_val, op, grp, grp_max);
#else
    const int64_t per = ((P + nw - 1) / nw + 31) & ~(int64_t)31;
    const int64_t pb = min(P, per * w), pe = min(P, per * (w + 1));
    warp_products<VALUES, V>(E, (int)nent64, pb, pe, b_col, b_val, op);
    __syncthreads();
#endif
    if (stop && *stop) return;
  }
}

struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct BlockSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// -------------------------------------------------------------------------
// row limit (reference overflow rule) and output type helpers

__device__ __forceinline__ int64_t row_limit(const int8_t* kind, const int64_t* cap, const int64_t* alloc,
                                             int64_t row) {
  if (!kind) return NOLIMIT;
  const int8_t k = kind[row];
  if (k == SG_KIND_HASH || k == SG_KIND_ENHANCED_HASH) return (int64_t)(0.8 * (double)cap[row]);
  if (k == SG_KIND_DENSE) return alloc[row];
  return NOLIMIT;
}

// bitonic sort of n = pow2 (key, val) pairs in shared memory by a group of
// `gsize` threads starting at thread `gtid`; `sync` is a group barrier.
template <class Sync>
__device__ __forceinline__ void bitonic_kv(int* keys, double* vals, int n, int gtid, int gsize, Sync sync) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int q = gtid; q < (n >> 1); q += gsize) {
        const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
        const int ixj = i | j;
        const int ki = keys[i], kj = keys[ixj];
        const bool up = (i & k) == 0;
        if ((ki > kj) == up) {
          keys[i] = kj;
          keys[ixj] = ki;
          if (vals) {
            const double t = vals[i];
            vals[i] = vals[ixj];
            vals[ixj] = t;
          }
        }
      }
      sync();
    }
  }
}

// -------------------------------------------------------------------------
// warp register sort of packed (col << LOG2T | slot) words: blocked layout,
// element e = lane * IPT + i; stages with partner distance < IPT stay in
// registers, the others exchange with __shfl_xor (no shared-memory traffic)

template <int IPT>
__device__ __forceinline__ void warp_bitonic_reg(uint32_t (&r)[IPT], int lane) {
  // Direction of stage k for element e = lane * IPT + i is ((e & k) == 0):
  // for k < IPT it depends on i only (compile-time), for k >= IPT on the
  // lane only (one test per stage), so no per-element index math remains.
#pragma unroll
  for (int k = 2; k <= 32 * IPT; k <<= 1) {
    const bool asc_lane = ((lane * IPT) & k) == 0;
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= IPT) {
        const int lm = j / IPT;
        const bool keep_min = ((lane & lm) == 0) == asc_lane;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t o = __shfl_xor_sync(SG_FULL, r[i], lm);
          r[i] = keep_min ? min(r[i], o) : max(r[i], o);
        }
      } else {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const int p = i ^ j;
          if (p > i) {
            const uint32_t a = r[i], b = r[p];
            const uint32_t lo = min(a, b), hi = max(a, b);
            if (k < IPT) {
              const bool asc = (i & k) == 0;  // compile-time
              r[i] = asc ? lo : hi;
              r[p] = asc ? hi : lo;
            } else {
              r[i] = asc_lane ? lo : hi;
              r[p] = asc_lane ? hi : lo;
            }
          }
        }
      }
    }
  }
}

// every column fits next to a LOG2T-bit slot index in 32 bits
template <int LOG2T>
__device__ __forceinline__ bool b_ncols_fit_u32(int64_t ncols) {
  return ncols <= ((int64_t)1 << (32 - LOG2T));
}

// packs the occupied slots of a warp hash table (keys[T], -1 = empty) to the
// front of keys as (col << LOG2T | slot), in slot order; returns the count
template <int LOG2T>
__device__ __forceinline__ int warp_compact_packed(int* keys, int lane) {
  constexpr int T = 1 << LOG2T;
  int n = 0;
  for (int s0 = 0; s0 < T; s0 += 32) {
    const int k = keys[s0 + lane];
    const bool occ = k != -1;
    const unsigned b = __ballot_sync(SG_FULL, occ);
    __syncwarp();
    if (occ) keys[n + __popc(b & lanemask_lt())] = (int)(((uint32_t)k << LOG2T) | (uint32_t)(s0 + lane));
    n += __popc(b);
    __syncwarp();
  }
  return n;
}

// sorts the n packed words at keys[0, n) and writes the row: columns and
// vals[slot] (n <= 32 * IPT)
template <int IPT, int LOG2T, typename V>
__device__ __forceinline__ void warp_sort_emit(int* keys, const double* vals, int n, int lane,
                                               int32_t* __restrict__ oc, V* __restrict__ ov) {
  uint32_t r[IPT];
  uint32_t* pk = reinterpret_cast<uint32_t*>(keys);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = lane * IPT + i;
    r[i] = e < n ? pk[e] : 0xFFFFFFFFu;
  }
  warp_bitonic_reg<IPT>(r, lane);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = lane * IPT + i;
    if (e < n) pk[e] = r[i];
  }
  __syncwarp();
  // striped (coalesced) emission
  for (int e = lane; e < n; e += 32) {
    const uint32_t p = pk[e];
    st_stream(oc + e, (int32_t)(p >> LOG2T));
    st_stream(ov + e, (V)vals[p & ((1u << LOG2T) - 1)]);
  }
}

// long rows (n > 512): bitonic sort of the packed words in shared memory
template <int LOG2T, typename V>
__device__ __forceinline__ void warp_sort_emit_packed_smem(int* keys, const double* vals, int n, int lane,
                                                           int32_t* __restrict__ oc, V* __restrict__ ov) {
  uint32_t* pk = reinterpret_cast<uint32_t*>(keys);
  const int pad = (int)next_pow2_u32((uint32_t)max(n, 1));  // <= T
  for (int i = n + lane; i < pad; i += 32) pk[i] = 0xFFFFFFFFu;
  __syncwarp();
  for (int k = 2; k <= pad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int q = lane; q < (pad >> 1); q += 32) {
        const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
        const int ixj = i | j;
        const uint32_t a = pk[i], b = pk[ixj];
        if ((a > b) == ((i & k) == 0)) {
          pk[i] = b;
          pk[ixj] = a;
        }
      }
      __syncwarp();
    }
  }
  for (int e = lane; e < n; e += 32) {
    const uint32_t p = pk[e];
    st_stream(oc + e, (int32_t)(p >> LOG2T));
    st_stream(ov + e, (V)vals[p & ((1u << LOG2T) - 1)]);
  }
}

// wide-column fallback: compact (key, val) in place and bitonic-sort them in
// shared memory; returns the count
template <int T, typename V>
__device__ __forceinline__ int warp_sort_emit_smem(int* keys, double* vals, int lane, int32_t* __restrict__ oc,
                                                   V* __restrict__ ov) {
  int n = 0;
  for (int s0 = 0; s0 < T; s0 += 32) {
    const int k = keys[s0 + lane];
    const double v = vals[s0 + lane];
    const bool occ = k != -1;
    const unsigned b = __ballot_sync(SG_FULL, occ);
    __syncwarp();
    if (occ) {
      const int pos = n + __popc(b & lanemask_lt());
      keys[pos] = k;
      vals[pos] = v;
    }
    n += __popc(b);
    __syncwarp();
  }
  const int pad = (int)next_pow2_u32((uint32_t)max(n, 1));
  for (int i = n + lane; i < pad; i += 32) keys[i] = INT_MAX;
  __syncwarp();
  bitonic_kv(keys, vals, pad, lane, 32, WarpSync{});
  for (int i = lane; i < n; i += 32) {
    st_stream(oc + i, keys[i]);
    st_stream(ov + i, (V)vals[i]);
  }
  return n;
}

// -------------------------------------------------------------------------
// HW: warp-per-row shared-memory hash

constexpr int HW_WARPS = 4;

// COUNT = false: no running count (the caller counts occupied slots after
// the row, overflow = count > limit; identical to the running rule)
template <int MODE, bool COUNT = true>
struct HashOp {
  int* keys;
  double* vals;
  int* cnt;
  int* ovf;
  int log2t;
  int64_t limit;
  __device__ __forceinline__ void operator()(int32_t col, double v) {
    const int T = 1 << log2t;
    uint32_t s = slot_hash((uint32_t)col, log2t);
    volatile int* vk = keys;
    for (int probe = 0; probe < T; ++probe) {
      int k = vk[s];
      if (k == col) {
        if (MODE) smem_add(&vals[s], v);
        return;
      }
      if (k == -1) {
        const int old = atomicCAS(&keys[s], -1, col);
        if (old == -1) {
          if (COUNT) {
            const int c = atomicAdd(cnt, 1);
            if ((int64_t)c >= limit) *ovf = 1;
          }
          if (MODE) smem_add(&vals[s], v);
          return;
        }
        if (old == col) {
          if (MODE) smem_add(&vals[s], v);
          return;
        }
      }
      s = (s + 1) & (T - 1);
    }
    *ovf = 1;
  }
};

template <int LOG2T, int MODE, typename V>
__global__ void __launch_bounds__(HW_WARPS * 32) k_hash_warp(int64_t nbin, const int32_t* __restrict__ rows,
                                                             Csr A, Csr B, const int8_t* kind, const int64_t* cap,
                                                             const int64_t* alloc, const int64_t* __restrict__ out_off,
                                                             int32_t* __restrict__ out_col, V* __restrict__ out_val,
                                                             int64_t* __restrict__ counts,
                                                             uint8_t* __restrict__ overflow, int64_t B_ncols) {
  constexpr int T = 1 << LOG2T;
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = warp_id(), lane = lane_id();
  // per-warp layout: S[33] bs[33] av[33] (int64/double), keys[T], vals[T], cnt, ovf
  constexpr size_t ENT = 3 * 33 * 8;
  constexpr size_t PER = ENT + (size_t)T * 4 + (MODE ? (size_t)T * 8 : 0) + 16;
  unsigned char* base = smem + (size_t)w * ((PER + 15) & ~size_t(15));
  Entries E{reinterpret_cast<int64_t*>(base), reinterpret_cast<int64_t*>(base) + 33,
            reinterpret_cast<double*>(base) + 66};
  double* vals = reinterpret_cast<double*>(base + ENT);
  int* keys = reinterpret_cast<int*>(base + ENT + (MODE ? (size_t)T * 8 : 0));
  int* cnt = keys + T;
  int* ovf = cnt + 1;
  const int64_t wid = (int64_t)blockIdx.x * HW_WARPS + w;
  if (wid >= nbin) return;
  const int64_t row = rows[wid];
  for (int i = lane; i < T; i += 32) {
    keys[i] = -1;
    if (MODE) vals[i] = 0.0;
  }
  if (lane == 0) {
    *cnt = 0;
    *ovf = 0;
  }
  __syncwarp();
  const int64_t limit = row_limit(kind, cap, alloc, row);
  HashOp<MODE, false> op{keys, vals, cnt, ovf, LOG2T, limit};
  warp_row<MODE == 1, V>(row, A.ptr, A.col, (const V*)A.val, B.ptr, B.col, (const V*)B.val, E, op, ovf);
  __syncwarp();
  int occ = 0;
  for (int s0 = 0; s0 < T; s0 += 32) occ += __popc(__ballot_sync(SG_FULL, keys[s0 + lane] != -1));
  if (MODE == 0) {
    // a full table (assisted sizing underestimated the row): -1 = recount
    if (lane == 0) counts[row] = *ovf ? -1 : occ;
    return;
  }
  if (*ovf || (int64_t)occ > limit) {
    if (lane == 0) {
      counts[row] = 0;
      overflow[row] = 1;
    }
    return;
  }
  const int64_t off = out_off[row];
  int n;
  if (b_ncols_fit_u32<LOG2T>(B_ncols)) {
    // pack (col << LOG2T | slot) to the front of keys, sort the packed words
    // in registers, then emit col = p >> LOG2T with vals[slot]
    n = warp_compact_packed<LOG2T>(keys, lane);
    const int ipt = (n + 31) >> 5;
    if (ipt <= 1) warp_sort_emit<1, LOG2T>(keys, vals, n, lane, out_col + off, out_val + off);
    else if (ipt <= 2) warp_sort_emit<2, LOG2T>(keys, vals, n, lane, out_col + off, out_val + off);
    else if (ipt <= 4) warp_sort_emit<4, LOG2T>(keys, vals, n, lane, out_col + off, out_val + off);
    else if (ipt <= 8) warp_sort_emit<8, LOG2T>(keys, vals, n, lane, out_col + off, out_val + off);
    else if (ipt <= 16) warp_sort_emit<16, LOG2T>(keys, vals, n, lane, out_col + off, out_val + off);
    else warp_sort_emit_packed_smem<LOG2T>(keys, vals, n, lane, out_col + off, out_val + off);
  } else {
    n = -1;
  }
  if (n < 0) n = warp_sort_emit_smem<T>(keys, vals, lane, out_col + off, out_val + off);
  if (lane == 0) {
    counts[row] = n;
    overflow[row] = 0;
  }
}

template <int LOG2T, int MODE>
constexpr size_t hw_smem() {
  return (size_t)HW_WARPS * (((3 * 33 * 8 + ((size_t)1 << LOG2T) * 4 + (MODE ? ((size_t)1 << LOG2T) * 8 : 0) + 16) + 15) &
                             ~size_t(15));
}

// -------------------------------------------------------------------------
// ESCR: warp-per-row register expand-sort-compress for short rows of low
// compression ratio (products ~ outputs, e.g. the rect config): the products
// are appended to a per-warp shared buffer, sorted as packed
// (col << 9 | product slot) words in registers (warp_bitonic_reg), and
// duplicate columns summed in slot order -- no hash table to clear, probe,
// compact or sort.  Needs products <= 512 and columns < 2^23.

constexpr int ESCR_WARPS = 4;
constexpr int ESCR_MAX = 512;

struct AppendOp {
  int* keys;
  double* vals;
  int* n;
  __device__ __forceinline__ void operator()(int32_t col, double v) {
    const unsigned act = __activemask();
    const int lane = lane_id();
    const int leader = __ffs(act) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(n, __popc(act));
    base = __shfl_sync(act, base, leader);
    const int pos = base + __popc(act & lanemask_lt());
    keys[pos] = col;
    vals[pos] = v;
  }
};

template <int IPT, typename V>
__device__ __forceinline__ int escr_sort_reduce(int* keys, const double* vals, int n, int lane,
                                                int32_t* __restrict__ oc, V* __restrict__ ov) {
  uint32_t r[IPT];
  uint32_t* pk = reinterpret_cast<uint32_t*>(keys);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = lane * IPT + i;
    r[i] = e < n ? (((uint32_t)keys[e] << 9) | (uint32_t)e) : 0xFFFFFFFFu;
  }
  __syncwarp();
  warp_bitonic_reg<IPT>(r, lane);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int e = lane * IPT + i;
    if (e < n) pk[e] = r[i];
  }
  __syncwarp();
  // striped pass: a run head sums its run (slot order) and writes at the
  // head's rank among heads
  int out = 0;
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int e = e0 + lane;
    const uint32_t k = e < n ? pk[e] : 0xFFFFFFFFu;
    const bool head = e < n && (e == 0 || (pk[e - 1] >> 9) != (k >> 9));
    const unsigned hb = __ballot_sync(SG_FULL, head);
    if (head) {
      double sum = vals[k & 511u];
      for (int j = e + 1; j < n && (pk[j] >> 9) == (k >> 9); ++j) sum += vals[pk[j] & 511u];
      const int pos = out + __popc(hb & lanemask_lt());
      st_stream(oc + pos, (int32_t)(k >> 9));
      st_stream(ov + pos, (V)sum);
    }
    out += __popc(hb);
  }
  return out;
}

template <typename V>
__global__ void __launch_bounds__(ESCR_WARPS * 32) k_escr(int64_t nbin, const int32_t* __restrict__ rows, Csr A,
                                                          Csr B, const int64_t* __restrict__ out_off,
                                                          int32_t* __restrict__ out_col, V* __restrict__ out_val,
                                                          int64_t* __restrict__ counts,
                                                          uint8_t* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = warp_id(), lane = lane_id();
  constexpr size_t ENT = 3 * 33 * 8;
  constexpr size_t PER = ENT + (size_t)ESCR_MAX * 12 + 16;
  unsigned char* base = smem + (size_t)w * PER;
  Entries E{reinterpret_cast<int64_t*>(base), reinterpret_cast<int64_t*>(base) + 33,
            reinterpret_cast<double*>(base) + 66};
  double* vals = reinterpret_cast<double*>(base + ENT);
  int* keys = reinterpret_cast<int*>(base + ENT + (size_t)ESCR_MAX * 8);
  int* n = keys + ESCR_MAX;
  const int64_t wid = (int64_t)blockIdx.x * ESCR_WARPS + w;
  if (wid >= nbin) return;
  const int64_t row = rows[wid];
  if (lane == 0) *n = 0;
  __syncwarp();
  AppendOp op{keys, vals, n};
  warp_row<true, V>(row, A.ptr, A.col, (const V*)A.val, B.ptr, B.col, (const V*)B.val, E, op, nullptr);
  __syncwarp();
  const int np = *n;
  const int64_t off = out_off[row];
  int cnt;
  const int ipt = (np + 31) >> 5;
  if (ipt <= 1) cnt = escr_sort_reduce<1, V>(keys, vals, np, lane, out_col + off, out_val + off);
  else if (ipt <= 2) cnt = escr_sort_reduce<2, V>(keys, vals, np, lane, out_col + off, out_val + off);
  else if (ipt <= 4) cnt = escr_sort_reduce<4, V>(keys, vals, np, lane, out_col + off, out_val + off);
  else if (ipt <= 8) cnt = escr_sort_reduce<8, V>(keys, vals, np, lane, out_col + off, out_val + off);
  else cnt = escr_sort_reduce<16, V>(keys, vals, np, lane, out_col + off, out_val + off);
  if (lane == 0) {
    counts[row] = cnt;
    overflow[row] = 0;
  }
}

constexpr size_t escr_smem() { return (size_t)ESCR_WARPS * (3 * 33 * 8 + (size_t)ESCR_MAX * 12 + 16); }

// -------------------------------------------------------------------------
// HB: block-per-row shared-memory hash

#ifndef SG_HB_RADIX
#define SG_HB_RADIX 5  // 4 passes over the 20 key bits of a 2^20-column span
#endif
template <int LOG2T, int MODE, typename V, int NT>
__global__ void __launch_bounds__(NT) k_hash_block(int64_t nbin, const int32_t* __restrict__ rows, Csr A, Csr B,
                                                   const int8_t* kind, const int64_t* cap, const int64_t* alloc,
                                                   const int64_t* __restrict__ span_lo,
                                                   const int64_t* __restrict__ span_hi,
                                                   const int64_t* __restrict__ out_off,
                                                   int32_t* __restrict__ out_col, V* __restrict__ out_val,
                                                   int64_t* __restrict__ counts, uint8_t* __restrict__ overflow) {
  constexpr int T = 1 << LOG2T;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t scr[NT / 32 + 2];
  __shared__ int cnt, ovf;
  double* vals = reinterpret_cast<double*>(smem);
  int* keys = reinterpret_cast<int*>(smem + (MODE ? (size_t)T * 8 : 0));
  unsigned char* ebase = smem + (MODE ? (size_t)T * 8 : 0) + (size_t)T * 4;
  Entries E{reinterpret_cast<int64_t*>(ebase), reinterpret_cast<int64_t*>(ebase) + (NT + 1),
            reinterpret_cast<double*>(ebase) + 2 * (NT + 1)};
  for (int64_t b = blockIdx.x; b < nbin; b += gridDim.x) {
    const int64_t row = rows[b];
    for (int i = threadIdx.x; i < T; i += NT) {
      keys[i] = -1;
      if (MODE) vals[i] = 0.0;
    }
    if (threadIdx.x == 0) {
      cnt = 0;
      ovf = 0;
    }
    __syncthreads();
    HashOp<MODE> op{keys, vals, &cnt, &ovf, LOG2T, row_limit(kind, cap, alloc, row)};
    block_row<MODE == 1, V>(row, A.ptr, A.col, (const V*)A.val, B.ptr, B.col, (const V*)B.val, E, scr, op, &ovf);
    __syncthreads();
    if (MODE == 0) {
      if (threadIdx.x == 0) counts[row] = ovf ? -1 : cnt;  // -1: recount (assisted sizing)
      __syncthreads();
      continue;
    }
    if (ovf) {
      if (threadIdx.x == 0) {
        counts[row] = 0;
        overflow[row] = 1;
      }
      __syncthreads();
      continue;
    }
    // in-place compaction in any order (the sort below orders it): chunks of
    // 2*NT slots are read into registers, then (one barrier later) written to
    // positions from a shared counter, one warp-aggregated atomic per warp;
    // the writes stay below the chunk's start + the occupied count, so never
    // reach an unread slot
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    for (int s0 = 0; s0 < T; s0 += 2 * NT) {
      const int k0 = keys[s0 + threadIdx.x], k1 = (s0 + NT + (int)threadIdx.x < T) ? keys[s0 + NT + threadIdx.x] : -1;
      const double v0 = vals[s0 + threadIdx.x];
      const double v1 = (s0 + NT + (int)threadIdx.x < T) ? vals[s0 + NT + threadIdx.x] : 0.0;
      __syncthreads();
      const unsigned m0 = __ballot_sync(SG_FULL, k0 != -1), m1 = __ballot_sync(SG_FULL, k1 != -1);
      const int lane = lane_id();
      int base = 0;
      if (lane == 0) base = atomicAdd(&cnt, __popc(m0) + __popc(m1));
      base = __shfl_sync(SG_FULL, base, 0);
      const unsigned lt = lanemask_lt();
      if (k0 != -1) {
        const int p = base + __popc(m0 & lt);
        keys[p] = k0;
        vals[p] = v0;
      }
      if (k1 != -1) {
        const int p = base + __popc(m0) + __popc(m1 & lt);
        keys[p] = k1;
        vals[p] = v1;
      }
    }
    __syncthreads();
    const int64_t n = cnt;
    // sort the n <= T/2 distinct columns: LSD radix sort (CUB block
    // primitive) on (col - span_lo) over only the bits the row's span needs,
    // values carried along; striped output -> coalesced stores
    {
      constexpr int ITEMS = (T / 2) / NT;
      using Sorter = cub::BlockRadixSort<uint32_t, NT, ITEMS, double, SG_HB_RADIX>;
      const int32_t lo32 = (int32_t)span_lo[row];
      const uint32_t span = (uint32_t)(span_hi[row] - span_lo[row] + 1);
      static_assert(sizeof(typename Sorter::TempStorage) <= ((size_t)1 << LOG2T) * 12, "sort storage");
      // keys < 2^bits; the padding items (blocked positions >= n) take the
      // largest key, and the stable sort keeps them after the n real ones
      const int bits = span <= 1 ? 1 : 32 - __clz(span - 1);
      const uint32_t pad = bits < 32 ? (1u << bits) - 1u : 0xffffffffu;
      uint32_t kk[ITEMS];
      double vv[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int idx = threadIdx.x * ITEMS + i;
        kk[i] = idx < n ? (uint32_t)(keys[idx] - lo32) : pad;
        vv[i] = idx < n ? vals[idx] : 0.0;
      }
      __syncthreads();
      auto& tmp = *reinterpret_cast<typename Sorter::TempStorage*>(smem);
      Sorter(tmp).SortBlockedToStriped(kk, vv, 0, bits);
      const int64_t off = out_off[row];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int idx = i * NT + threadIdx.x;
        if (idx < n) {
          st_stream(out_col + off + idx, (int32_t)kk[i] + lo32);
          st_stream(out_val + off + idx, (V)vv[i]);
        }
      }
    }
    if (threadIdx.x == 0) {
      counts[row] = n;
      overflow[row] = 0;
    }
    __syncthreads();
  }
}

template <int LOG2T, int MODE, int NT>
constexpr size_t hb_smem() {
  return ((size_t)1 << LOG2T) * (MODE ? 12 : 4) + (size_t)3 * (NT + 1) * 8;
}

// -------------------------------------------------------------------------
// ESC: warp per row, <= 64 products (accumulate.py:254-271, 368-378)

constexpr int ESC_WARPS = 8;


template <typename V>
__global__ void __launch_bounds__(ESC_WARPS * 32) k_esc(int64_t nbin, const int32_t* __restrict__ rows, Csr A, Csr B,
                                                        const int64_t* __restrict__ out_off,
                                                        int32_t* __restrict__ out_col, V* __restrict__ out_val,
                                                        int64_t* __restrict__ counts, uint8_t* __restrict__ overflow) {
  __shared__ int64_t ent[ESC_WARPS][3 * 33];
  __shared__ unsigned long long key[ESC_WARPS][64];
  __shared__ double val[ESC_WARPS][64];
  __shared__ double vsorted[ESC_WARPS][64];
  const int w = warp_id(), lane = lane_id();
  const int64_t wid = (int64_t)blockIdx.x * ESC_WARPS + w;
  if (wid >= nbin) return;
  const int64_t row = rows[wid];
  Entries E{ent[w], ent[w] + 33, reinterpret_cast<double*>(ent[w] + 66)};
  // gather products in stream order
  int np = 0;
  const int64_t t1 = A.ptr[row + 1];
  for (int64_t t = A.ptr[row]; t < t1; t += 32) {
    int nent;
    const int64_t P = warp_load_chunk<true, V>(t, t1, A.col, (const V*)A.val, B.ptr, E, nent);
    for (int64_t p0 = 0; p0 < P; p0 += 32) {
      // owner search (small chunks: linear)
      const int64_t p = p0 + lane;
      if (p < P) {
        int c = 0;
        while (c + 1 < nent && E.S[c + 1] <= p) ++c;
        const int64_t j = E.d[c] + p;
        const int pos = np + (int)p;
        if (pos < 64) {
          key[w][pos] = ((unsigned long long)(uint32_t)B.col[j] << 32) | (unsigned)pos;
          val[w][pos] = E.av[c] * (double)((const V*)B.val)[j];
        }
      }
    }
    np += (int)P;
    __syncwarp();
  }
  np = min(np, 64);
  for (int i = np + lane; i < 64; i += 32) key[w][i] = ~0ull;
  __syncwarp();
  // bitonic sort of 64 packed (col, product index) keys: stable by construction
  for (int k = 2; k <= 64; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int q = lane;  // 32 pairs
      const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
      const int ixj = i | j;
      const unsigned long long ki = key[w][i], kj = key[w][ixj];
      const bool up = (i & k) == 0;
      if ((ki > kj) == up) {
        key[w][i] = kj;
        key[w][ixj] = ki;
      }
      __syncwarp();
    }
  for (int i = lane; i < np; i += 32) vsorted[w][i] = val[w][(unsigned)(key[w][i] & 0xffffffffu)];
  __syncwarp();
  // heads and segmented sums (sequential within a run, stream order)
  int nhead = 0;
  const int64_t off = out_off[row];
  for (int base = 0; base < np; base += 32) {
    const int i = base + lane;
    bool head = false;
    if (i < np) head = (i == 0) || ((key[w][i] >> 32) != (key[w][i - 1] >> 32));
    const unsigned hb = __ballot_sync(SG_FULL, head);
    if (head) {
      double s = vsorted[w][i];
      for (int r = i + 1; r < np && (key[w][r] >> 32) == (key[w][i] >> 32); ++r) s += vsorted[w][r];
      const int pos = nhead + __popc(hb & lanemask_lt());
      st_stream(out_col + off + pos, (int32_t)(key[w][i] >> 32));
      st_stream(out_val + off + pos, (V)s);
    }
    nhead += __popc(hb);
  }
  if (lane == 0) {
    counts[row] = nhead;
    overflow[row] = 0;
  }
}

// -------------------------------------------------------------------------
// BM: block-per-row bitmap over the column span (windows of BW*64 columns)

template <typename V>
struct BitmapSetOp {
  unsigned long long* bm;
  int32_t wlo;
  uint32_t wspan;  // whi - wlo
  __device__ __forceinline__ void operator()(int32_t col, double) {
    const uint32_t x = (uint32_t)(col - wlo);
    if (x > wspan) return;
    // 32-bit ATOMS.OR is native on sm_100a (the 64-bit form is a CAS loop)
    atomicOr(reinterpret_cast<unsigned*>(bm) + (x >> 5), 1u << (x & 31));
  }
};



template <typename V>
struct BitmapAddOp {
  const unsigned long long* bm;
  const int* pre;
  int64_t wlo, whi;
  V* out;  // already offset to the window's first output slot
  __device__ __forceinline__ void operator()(int32_t col, double v) {
    if (col < wlo || col > whi) return;
    const int64_t x = col - wlo;
    const int w = (int)(x >> 6);
    const unsigned long long below = bm[w] & ((1ull << (x & 63)) - 1ull);
    gmem_red(out + pre[w] + __popcll(below), (V)v);
  }
};

// Exclusive prefix of word popcounts: pre[i] = set bits in words [0, i);
// returns the total.  Warps own contiguous word ranges and read them with
// consecutive lanes (no bank conflicts).
template <int NT>
__device__ __forceinline__ int64_t bitmap_prefix(const unsigned long long* bm, int* pre, int nwords,
                                                 int64_t* scr) {
  constexpr int NW = NT / 32;
  const int w = warp_id(), lane = lane_id();
  const int per = ((nwords + NW - 1) / NW + 31) & ~31;
  const int wb = min(nwords, per * w), we = min(nwords, per * (w + 1));
  int64_t s = 0;
  for (int i = wb + lane; i < we; i += 32) s += __popcll(bm[i]);
  s = warp_sum(s);
  int64_t tot;
  int64_t base = block_excl_scan(lane == 0 ? s : (int64_t)0, scr, &tot);
  base = __shfl_sync(SG_FULL, base, 0);
  for (int i0 = wb; i0 < we; i0 += 32) {
    const int i = i0 + lane;
    const int v = i < we ? __popcll(bm[i]) : 0;
    const int inc = warp_incl_scan(v);
    if (i < we) pre[i] = (int)(base + inc - v);
    base += __shfl_sync(SG_FULL, inc, 31);
  }
  __syncthreads();
  return tot;
}

// Write the column of every set bit of a 64-bit bitmap word, ascending.
// Plain (L2-allocating) stores: a warp fills each output line over several
// instructions, and evict-first partial lines would cost DRAM read-fills.
__device__ __forceinline__ void emit_bits(unsigned long long bits, int32_t colbase, int32_t* __restrict__ out) {
  unsigned lo = (unsigned)bits, hi = (unsigned)(bits >> 32);
  int k = 0;
  while (lo) {
    out[k++] = colbase + __ffs(lo) - 1;
    lo &= lo - 1;
  }
  while (hi) {
    out[k++] = colbase + 31 + __ffs(hi);
    hi &= hi - 1;
  }
}

// Numeric window geometry (shared by the count kernels that emit windows and
// the window accumulator): a window holds at most WIN_R distinct columns and
// spans at most WIN_WORDS*64 columns, so its bitmap, rank prefix and values
// all sit in shared memory.
#ifndef SG_WIN_WORDS
#define SG_WIN_WORDS 2048
#endif
constexpr int WIN_WORDS = SG_WIN_WORDS;  // 2048: 131,072 columns
#ifndef SG_WIN_R
#define SG_WIN_R 8192
#endif
constexpr int WIN_R = SG_WIN_R;  // values per window (8192: 64 KB fp64, two windows in flight per SM)
// Windows start on TILE_COLS-column tiles (absolute), so each selected B
// row's segment in a window is two lookups in the B tile index (no search).
constexpr int TILE_COLS = 4096;
constexpr int TILE_WORDS = TILE_COLS / 64;
constexpr int WIN_TILES = WIN_WORDS / TILE_WORDS;
constexpr int WIN_NT = 1024;

// bitmap origin of a windowed row: span_lo rounded down to a tile
__host__ __device__ __forceinline__ int64_t win_origin(int64_t lo) { return lo & ~(int64_t)(TILE_COLS - 1); }

// device view of sg_windows_t (include/sgb200.h)
struct Win {
  const int64_t* off;
  int2* wins;
  int32_t* nwin;
  const int64_t* bm_off;
  unsigned long long* bm_save;
  int32_t* pre_save;  // unused (ranks live in the 16-byte saved words)
  const int64_t* btile_off;
  const int32_t* btile;
};

// Symbolic-pass routing: rows counted with a shared-memory bitmap (and hence
// able to record numeric windows).  Long rows with a dense enough span, and
// every row too long for the largest count hash table.
// rows of more than SG_BM_COUNT_MIN products are counted with a bitmap even
// when it is sparse (span/64 > products); with SG_SPARSE_WIN they also get
// windows (cut by the count pass, no saved words) taken by k_bmr
#ifndef SG_BM_COUNT_MIN
#define SG_BM_COUNT_MIN 4096
#endif
#ifndef SG_SPARSE_WIN
#define SG_SPARSE_WIN 0
#endif
__host__ __device__ __forceinline__ bool count_uses_bitmap(int64_t p, int64_t span);
__host__ __device__ __forceinline__ bool count_bitmap_sparse(int64_t p, int64_t span) {
  return !count_uses_bitmap(p, span) && SG_BM_COUNT_MIN > 0 && p > SG_BM_COUNT_MIN && span <= ((int64_t)1 << 20);
}
__host__ __device__ __forceinline__ bool count_uses_bitmap(int64_t p, int64_t span) {
  if (p <= 1024) return false;
  if (span <= ((int64_t)1 << 20) && (span + 63) / 64 <= p) return true;
  return p > 16384;
}

__host__ __device__ __forceinline__ int64_t window_capacity(int64_t products, int64_t span) {
  if (products <= 0 || span <= 0) return 0;
  const int64_t d = products < span ? products : span;
  // two consecutive windows cut by the WIN_R rule hold > WIN_R keys together
  return 2 * d / WIN_R + (span + TILE_COLS) / TILE_COLS / WIN_TILES + 3;
}

// Count pass of a windowed row (one sweep): word ranks, the saved 16-byte
// {lo, rank, hi, rank} words and the rank at every tile start in ONE pass
// over the bitmap (warps own contiguous word ranges; a warp scan of the
// popcounts gives each word its rank).  tile_rank[t] = rank of tile t's first
// column relative to the sweep.  Returns the sweep's total.
template <int NT>
__device__ __forceinline__ int64_t prefix_save(const unsigned long long* bm, int nwords, int64_t rank_base,
                                               uint4* __restrict__ dst, int* tile_rank, int64_t* scr) {
  constexpr int NW = NT / 32;
  const int w = warp_id(), lane = lane_id();
  const int per = ((nwords + NW - 1) / NW + 31) & ~31;
  const int wb = min(nwords, per * w), we = min(nwords, per * (w + 1));
  int64_t s = 0;
  for (int i = wb + lane; i < we; i += 32) s += __popcll(bm[i]);
  s = warp_sum(s);
  int64_t tot;
  int64_t base = block_excl_scan(lane == 0 ? s : (int64_t)0, scr, &tot);
  base = __shfl_sync(SG_FULL, base, 0);
  for (int i0 = wb; i0 < we; i0 += 32) {
    const int i = i0 + lane;
    const unsigned long long wv = i < we ? bm[i] : 0ull;
    const int c = __popcll(wv);
    const int inc = warp_incl_scan(c);
    if (i < we) {
      const int64_t rel = base + inc - c;
      if (dst) {
        const uint32_t r = (uint32_t)(rank_base + rel), lo32 = (uint32_t)wv;
        st_stream_v4(dst + i, make_uint4(lo32, r, (uint32_t)(wv >> 32), r + (uint32_t)__popc(lo32)));
      }
      if ((i & (TILE_WORDS - 1)) == 0) tile_rank[i / TILE_WORDS] = (int)rel;
    }
    base += __shfl_sync(SG_FULL, inc, 31);
  }
  __syncthreads();
  return tot;
}

// k_bitmap shared layout: bitmap (BW words) | ranks | [group table] | entries.
// MODE 1 ranks every word; MODE 0 only the 4096-column tiles.
template <int BW, int MODE>
__host__ __device__ constexpr size_t bm_pre_bytes() {
  return MODE == 0 ? (((size_t)BW / TILE_WORDS * 4 + 15) & ~(size_t)15) : (size_t)BW * 4;
}
// own group table (groups) of the long-row count pass; 0: the shared g_grp
#ifndef SG_BM0_GRP
#define SG_BM0_GRP 4096
#endif
template <int BW, int MODE>
__host__ __device__ constexpr int bm_grp() {
  return (MODE == 0 && BW >= 16384) ? SG_BM0_GRP : 0;
}

template <int BW, int MODE, typename V, int NT>
__global__ void __launch_bounds__(NT) k_bitmap(int64_t nbin, const int32_t* __restrict__ rows, Csr A, Csr B,
                                               const int8_t* kind, const int64_t* cap, const int64_t* alloc,
                                               const int64_t* __restrict__ span_lo,
                                               const int64_t* __restrict__ span_hi,
                                               const int64_t* __restrict__ out_off,
                                               int32_t* __restrict__ out_col, V* __restrict__ out_val,
                                               int64_t* __restrict__ counts, uint8_t* __restrict__ overflow,
                                               Win win) {
  const int64_t* __restrict__ win_off = win.off;
  int2* __restrict__ wins = win.wins;
  int32_t* __restrict__ nwin = win.nwin;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t scr[NT / 32 + 2];
  // MODE 0 keeps only tile ranks (not word ranks); the long-row count pass
  // has its own group table of bm_grp() groups in dynamic shared memory, so
  // a long row's products run in sub-chunks of 32 * 4096 between barriers
  constexpr int OWN = bm_grp<BW, MODE>();
  constexpr size_t PRE = bm_pre_bytes<BW, MODE>();
  unsigned long long* bm = reinterpret_cast<unsigned long long*>(smem);
  int* pre = reinterpret_cast<int*>(smem + (size_t)BW * 8);
  int2* grp = OWN ? reinterpret_cast<int2*>(smem + (size_t)BW * 8 + PRE) : g_grp;
  constexpr int GRP = OWN ? OWN : GRP_MAX;
  unsigned char* ebase = smem + (size_t)BW * 8 + PRE + (size_t)OWN * 8;
  Entries E{reinterpret_cast<int64_t*>(ebase), reinterpret_cast<int64_t*>(ebase) + (NT + 1),
            reinterpret_cast<double*>(ebase) + 2 * (NT + 1)};
  constexpr int64_t WCOLS = (int64_t)BW * 64;
  __shared__ int64_t wst_rank, wst_tile;  // open numeric window (count pass)
  __shared__ int wst_n;                   // windows emitted so far
  for (int64_t b = blockIdx.x; b < nbin; b += gridDim.x) {
    const int64_t row = rows[b];
    const int64_t lo = span_lo[row], hi = span_hi[row];
    const int64_t limit = row_limit(kind, cap, alloc, row);
    int64_t total = 0;
    const int64_t wcap = (MODE == 0 && win_off) ? win_off[row + 1] - win_off[row] : 0;
    if (threadIdx.x == 0) {
      wst_n = 0;
      wst_rank = wst_tile = 0;
    }
    const bool multi = hi - lo + 1 > WCOLS;
    // count-only sweep first when a limit applies and the span needs windows
    bool over = false;
    if (MODE == 1 && limit != NOLIMIT && multi) {
      for (int64_t wlo = lo; wlo <= hi; wlo += WCOLS) {
        const int64_t whi = min(hi, wlo + WCOLS - 1);
        const int nwords = (int)((whi - wlo) / 64 + 1);
        for (int i = threadIdx.x; i < nwords; i += NT) bm[i] = 0ull;
        __syncthreads();
        BitmapSetOp<V> so{bm, (int32_t)wlo, (uint32_t)(whi - wlo)};
        block_row<false, V>(row, A.ptr, A.col, (const V*)A.val, B.ptr, B.col, (const V*)B.val, E, scr, so,
                            nullptr);
        int64_t c = 0;
        for (int i = threadIdx.x; i < nwords; i += NT) c += __popcll(bm[i]);
        int64_t tot;
        block_excl_scan(c, scr, &tot);
        total += tot;
      }
      over = total > limit;
      total = 0;
    }
    if (over) {
      if (threadIdx.x == 0) {
        counts[row] = 0;
        if (overflow) overflow[row] = 1;
      }
      __syncthreads();
      continue;
    }
    // windowed rows (count pass) keep their bitmap from a tile-aligned origin
    const int64_t org = (MODE == 0 && wcap > 0) ? win_origin(lo) : lo;
    for (int64_t wlo = org; wlo <= hi; wlo += WCOLS) {
      const int64_t whi = min(hi, wlo + WCOLS - 1);
      const int nwords = (int)((whi - wlo) / 64 + 1);
      for (int i = threadIdx.x; i < nwords; i += NT) bm[i] = 0ull;
      __syncthreads();
      BitmapSetOp<V> so{bm, (int32_t)wlo, (uint32_t)(whi - wlo)};
      block_row<false, V>(row, A.ptr, A.col, (const V*)A.val, B.ptr, B.col, (const V*)B.val, E, scr, so, nullptr,
                          NOLIMIT, grp, GRP);
      if (MODE == 0 && wcap == 0) {
        int64_t c = 0;
        for (int i = threadIdx.x; i < nwords; i += NT) c += __popcll(bm[i]);
        int64_t wtot;
        block_excl_scan(c, scr, &wtot);
        total += wtot;
        continue;
      }
      // MODE 0 (windowed rows): ranks, saved words and tile ranks in one
      // pass (pre[t] = rank of tile t); MODE 1: word ranks for the values
      const int64_t wtot =
          MODE == 0 ? prefix_save<NT>(bm, nwords, total,
                                      (win.bm_save && win.bm_off[row + 1] > win.bm_off[row])
                                          ? reinterpret_cast<uint4*>(win.bm_save) + win.bm_off[row] +
                                                ((wlo - org) >> 6)
                                          : nullptr,
                                      pre, scr)
                    : bitmap_prefix<NT>(bm, pre, nwords, scr);
      if (MODE == 0) {
        // emit numeric windows (tiles of TILE_WORDS words from the
        // tile-aligned origin):
        const int64_t gw0 = (wlo - org) >> 6;  // count windows are tile-aligned
        int2* wrow = wins + win_off[row];
        // (the row's bitmap was saved by prefix_save with the row rank of
        // every 32-bit half word, interleaved {lo, rank(lo), hi, rank(hi)}
        // (16 B per 64 columns): the window kernel bulk-copies a window's
        // words into shared memory as they are)
        // windows: greedy cuts over the row's tiles in column order -- a
        // window takes tiles while it holds <= WIN_R distinct columns over
        // <= WIN_TILES tiles; warp 0 walks 32 tiles per ballot, one ballot
        // per cut (the open window carries over to the next sweep)
        if (warp_id() == 0) {
          const int lane = lane_id();
          const int ntiles = (nwords + TILE_WORDS - 1) / TILE_WORDS;
          const int64_t tg0 = gw0 / TILE_WORDS;
          int n = wst_n;
          int64_t rs = wst_rank, ts = wst_tile;
          for (int ti0 = 0; ti0 < ntiles; ti0 += 32) {
            const int ti = ti0 + lane;
            const bool in = ti < ntiles;
            const int64_t r = in ? total + pre[ti] : 0;
            const int64_t rn = (ti + 1 < ntiles) ? total + pre[ti + 1] : total + wtot;
            const int64_t tg = tg0 + ti;
            int from = 0;
            for (;;) {
              const bool cut = in && lane >= from &&
                               (n == 0 || rn - rs > WIN_R || tg - ts + 1 > WIN_TILES);
              const unsigned m = __ballot_sync(SG_FULL, cut);
              if (!m) break;
              const int f = __ffs(m) - 1;
              if (lane == f && n < wcap) wrow[n] = make_int2((int)(org + (int64_t)TILE_COLS * tg), (int)r);
              rs = __shfl_sync(SG_FULL, r, f);
              ts = __shfl_sync(SG_FULL, tg, f);
              ++n;
              from = f + 1;
            }
          }
          if (lane == 0) {
            wst_n = n;
            wst_rank = rs;
            wst_tile = ts;
          }
        }
        __syncthreads();
        total += wtot;
        __syncthreads();
        continue;
      }
      if (!multi && total + wtot > limit) {
        over = true;
        break;
      }
      const int64_t base = out_off[row] + total;
      // emit sorted columns from the bitmap and clear the value slots
      for (int i = threadIdx.x; i < nwords; i += NT)
        emit_bits(bm[i], (int32_t)(wlo + (int64_t)i * 64), out_col + base + pre[i]);
      for (int64_t i = threadIdx.x; i < wtot; i += NT) out_val[base + i] = (V)0;
      __syncthreads();
      BitmapAddOp<V> ao{bm, pre, wlo, whi, out_val + base};
      block_row<true, V>(row, A.ptr, A.col, (const V*)A.val, B.ptr, B.col, (const V*)B.val, E, scr, ao, nullptr);
      total += wtot;
    }
    if (threadIdx.x == 0) {
      if (MODE == 0) {
        counts[row] = total;
        if (wcap > 0) nwin[row] = (int32_t)min((int64_t)wst_n, wcap);
      } else {
        counts[row] = over ? 0 : total;
        if (overflow) overflow[row] = over ? 1 : 0;
      }
    }
    __syncthreads();
  }
}

template <int BW, int MODE, int NT>
constexpr size_t bm_smem() {
  return (size_t)BW * 8 + bm_pre_bytes<BW, MODE>() + (size_t)bm_grp<BW, MODE>() * 8 + (size_t)3 * (NT + 1) * 8;
}

// -------------------------------------------------------------------------
// BMW: rank-window accumulator for long rows (multi-block per row).
//
// The count pass (k_bitmap, MODE 0) leaves, per long row, a list of windows
// (first column, rank of that column within the row) such that every window
// holds <= WIN_R distinct columns over <= WIN_WORDS*64 columns.  One CTA per
// (row, window) work item: restrict every selected B row to the window's
// column range (binary search), build the window bitmap (ATOMS.OR), rank
// prefix, accumulate values in shared memory at rank (fp64), then write the
// window's sorted slice of C with coalesced stores.  Windows of one row run
// on different SMs, so a 9.7M-product hub row is spread over ~80 CTAs.

__device__ __forceinline__ int64_t lower_bound_col(const int32_t* __restrict__ col, int64_t s, int64_t e,
                                                   int64_t c) {
  while (s < e) {
    const int64_t mid = (s + e) >> 1;
    if ((int64_t)__ldg(col + mid) < c) s = mid + 1; else e = mid;
  }
  return s;
}


template <bool VALUES, typename V, class Op>
__device__ __forceinline__ void block_chunk_products(const Entries& E, int nent, int64_t P,
                                                     const int32_t* __restrict__ b_col,
                                                     const V* __restrict__ b_val, Op& op) {
#if SG_GROUPED
  block_products<VALUES, V>(E, nent, P, b_col, b_val, op);
#else
  const int nw = blockDim.x >> 5, w = warp_id();
  const int64_t per = ((P + nw - 1) / nw + 31) & ~(int64_t)31;
  warp_products<VALUES, V>(E, nent, min(P, per * w), min(P, per * (w + 1)), b_col, b_val, op);
#endif
}

// The window's key set lives in shared memory as interleaved 32-bit words
// {bits, rank of the word's first column within the window} (uint2), so a
// product's rank is one LDS.64 + POPC; operations use 32-bit shared
// addresses (no generic-pointer conversions in the inner loop).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
  return r;
}

__device__ __forceinline__ void sts_u4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// fp64 add into shared memory: ptxas lowers it to LDS + DADD +
// ATOMS.CAST.SPIN.64 (store-conditional; no old value returned)
__device__ __forceinline__ void smem_add_f64(uint32_t a, double v) {
  asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

struct WinSetOp {
  uint32_t wp;  // shared address of the uint2 words
  int32_t c0;
  __device__ __forceinline__ void operator()(int32_t col, double) {
    const uint32_t x = (uint32_t)(col - c0);
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(wp + (x >> 5) * 8), "r"(1u << (x & 31)) : "memory");
  }
};


struct WinAddOp {
  uint32_t wp;    // shared address of the uint2 words
  uint32_t vals;  // shared address of the fp64 values
  int32_t c0;
  __device__ __forceinline__ uint32_t slot(int32_t col) const {
    const uint32_t x = (uint32_t)(col - c0);
    const uint2 p = lds_u2(wp + (x >> 5) * 8);
    return vals + (p.y + __popc(p.x & ((2u << (x & 31)) - 1u)) - 1u) * 8u;
  }
  __device__ __forceinline__ void operator()(int32_t col, double v) { smem_add_f64(slot(col), v); }
};

// Exclusive popcount prefix over n32 <= 2 * WIN_WORDS interleaved words in
// one pass: each lane owns up to 8 consecutive words of its warp's range.
template <int NT>
__device__ __forceinline__ void window_prefix32(uint2* wp, int n32, int64_t* scr) {
  constexpr int NW = NT / 32;
  const int w = warp_id(), lane = lane_id();
  const int per = (n32 + NW - 1) / NW;
  const int L = (per + 31) / 32;  // <= 8
  const int wb = min(n32, per * w), we = min(n32, per * (w + 1));
  int c[8];
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = wb + lane * L + i;
    c[i] = (i < L && idx < we) ? __popc(wp[idx].x) : 0;
    s += c[i];
  }
  const int inc = warp_incl_scan(s);
  int64_t tot;
  const int64_t wbase = block_excl_scan(lane == 31 ? (int64_t)inc : (int64_t)0, scr, &tot);
  int run = (int)__shfl_sync(SG_FULL, wbase, 31) + inc - s;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = wb + lane * L + i;
    if (i < L && idx < we) wp[idx].y = (uint32_t)run;
    run += c[i];
  }
  __syncthreads();
}

__device__ __forceinline__ void emit_bits32_smem(uint32_t bits, int32_t colbase, int* __restrict__ out) {
  int k = 0;
  while (bits) {
    out[k++] = colbase + __ffs(bits) - 1;
    bits &= bits - 1;
  }
}


#ifdef SG_PROF
// phase cycle counters of the window kernel (profiling build only: make prof)
__device__ unsigned long long g_phase[12];
__device__ unsigned long long g_kw[16];  // k_win: producer / consumer phase cycles
#define SG_PH(i)                                              \
  if (threadIdx.x == 0) {                                     \
    const long long _t = clock64();                           \
    atomicAdd(&g_phase[i], (unsigned long long)(_t - _tprev)); \
    _tprev = _t;                                              \
  }
#else
#define SG_PH(i)
#endif


// One numeric window, resolved before launch: a CTA needs a single load.
struct WinItem {
  int64_t out_base;  // C index of the window's first entry (row_ptr + rank)
  int64_t t0;        // A row start
  int64_t bm_word;   // saved-bitmap word of the window's first column (-1: none)
  int32_t t_len;     // A row length
  int32_t c0, c1;    // columns [c0, c1); c0 tile-aligned, c1 tile-aligned or row end
  int32_t cnt;       // distinct columns in the window
  int32_t last;      // window ends at the row's end (segment = rest of B row)
  int32_t rank0;     // row rank of the window's first column
};

// B tile index: for B rows with a table, tbl[tbl_off[k] + t] = offset in the
// row of the first column >= t*TILE_COLS (t = 0..ceil(ncols/TILE_COLS)).
struct BTile {
  const int64_t* off;  // int64[k]: table start, or -1
  const int32_t* tbl;
};

// Clip the B rows of a chunk of A entries to columns [c0, c1) (table lookup
// when indexed, binary search otherwise) and compact the non-empty segments.
template <bool VALUES, typename V>
__device__ __forceinline__ int64_t block_load_tiles(int64_t t, int64_t t1, int32_t c0, int32_t c1, bool last,
                                                    const int32_t* __restrict__ a_col, const V* __restrict__ a_val,
                                                    const int64_t* __restrict__ b_ptr,
                                                    const int32_t* __restrict__ b_col, BTile bt, Entries E,
                                                    int64_t* scr, int& nent) {
  int64_t bs = 0, len = 0;
  double av = 0.0;
  if (t + threadIdx.x < t1) {
    const int32_t k = a_col[t + threadIdx.x];
    const int64_t s = b_ptr[k], e = b_ptr[k + 1];
    if (e > s) {
      const int64_t to = bt.off ? bt.off[k] : -1;
      int64_t ss, ee;
      if (to >= 0) {
        ss = s + bt.tbl[to + c0 / TILE_COLS];
        ee = (last || (c1 % TILE_COLS)) ? e : s + bt.tbl[to + c1 / TILE_COLS];
        if (last) ee = e;
      } else {
        ss = lower_bound_col(b_col, s, e, c0);
        ee = last ? e : lower_bound_col(b_col, ss, e, c1);
      }
      bs = ss;
      len = ee - ss;
    }
    if (VALUES) av = (double)a_val[t + threadIdx.x];
  }
  // one scan of (len << 12 | nonempty): segment starts and compacted slots
  int64_t tot;
  const int64_t ex = block_excl_scan((len << 12) | (int64_t)(len > 0), scr, &tot);
  const int64_t S = ex >> 12, pos = ex & 4095, P = tot >> 12, n64 = tot & 4095;
  if (len > 0) {
    E.S[pos] = S;
    E.d[pos] = bs - S;
    if (VALUES) E.av[pos] = av;
  }
  __syncthreads();
  nent = (int)n64;
  return P;
}

template <int NT, int WORDS, int R>
constexpr size_t bmr_smem() {
  return (size_t)WORDS * 16 + (size_t)R * 8 + (size_t)3 * (NT + 1) * 8;
}

// Small windows (<= R/2 values over <= WORDS/2 words) run in half-size CTAs,
// two per SM, so one window's latency-bound setup / load phases overlap the
// other's value pass; the rest run one 1024-thread CTA per SM.
constexpr int SMALL_NT = WIN_NT / 2, SMALL_WORDS = WIN_WORDS / 2, SMALL_R = WIN_R / 2;

// One CTA per window (dynamic tickets; items are grouped by column range so
// concurrent CTAs gather the same B-row slabs and keep them in L2).  With the
// saved key bitmap and word ranks the window needs one value pass: rank =
// pre[w] + popc(bits below), fp64 add into shared memory, coalesced write.
template <typename V, int NT, int WORDS, int R, int CTAS>
__global__ void __launch_bounds__(NT, CTAS) k_bmr(int64_t nwork, const WinItem* __restrict__ work, Csr A, Csr B,
                                                   BTile bt, const unsigned long long* __restrict__ bm_save,
                                                   const int32_t* __restrict__ pre_save,
                                                   int32_t* __restrict__ out_col, V* __restrict__ out_val,
                                                   unsigned long long* __restrict__ ticket) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t scr[NT / 32 + 2];
  __shared__ int64_t item_next;
  uint2* wp = reinterpret_cast<uint2*>(smem);  // 2 * WORDS interleaved {bits, rank}
  double* vals = reinterpret_cast<double*>(smem + (size_t)WORDS * 16);
  unsigned char* ebase = smem + (size_t)WORDS * 16 + (size_t)R * 8;
  Entries E{reinterpret_cast<int64_t*>(ebase), reinterpret_cast<int64_t*>(ebase) + (NT + 1),
            reinterpret_cast<double*>(ebase) + 2 * (NT + 1)};
  const uint32_t wp_s = smem_addr(wp), vals_s = smem_addr(vals);
  const V* av = (const V*)A.val;
  const V* bv = (const V*)B.val;
  if (threadIdx.x == 0) item_next = (int64_t)atomicAdd(ticket, 1ull);
  __syncthreads();
  int64_t b = item_next;
#ifdef SG_PROF
  long long _tprev = clock64();
#endif
  while (b < nwork) {
    const WinItem it = work[b];
    const int32_t c0 = it.c0, c1 = it.c1;
    const int cnt = it.cnt;
    const int nwords = (int)(((int64_t)c1 - c0 + 63) >> 6);
    const bool saved = it.bm_word >= 0 && bm_save != nullptr;
    (void)pre_save;
    if (saved) {
      // saved {lo, rank, hi, rank} words (row ranks) -> window ranks
      const uint4* src = reinterpret_cast<const uint4*>(bm_save) + it.bm_word;
      const uint32_t r0 = (uint32_t)it.rank0;
      for (int i = threadIdx.x; i < nwords; i += NT) {
        const uint4 q = __ldcs(src + i);
        sts_u4(wp_s + (uint32_t)i * 16, q.x, q.y - r0, q.z, q.w - r0);
      }
    } else {
      for (int i = threadIdx.x; i < nwords; i += NT) sts_u4(wp_s + (uint32_t)i * 16, 0u, 0u, 0u, 0u);
    }
    for (int i = threadIdx.x; i < cnt; i += NT) vals[i] = 0.0;
    __syncthreads();
    SG_PH(0);
    WinSetOp so{wp_s, c0};
    WinAddOp ao{wp_s, vals_s, c0};
    const int64_t t0 = it.t0, t1 = it.t0 + it.t_len;
    const bool single = it.t_len <= NT;
    int nent = 0;
    int64_t P = 0;
    if (single) {
      P = block_load_tiles<true, V>(t0, t1, c0, c1, it.last, A.col, av, B.ptr, B.col, bt, E, scr, nent);
      SG_PH(1);
#ifdef SG_PROF
      if (threadIdx.x == 0) atomicAdd(&g_phase[8], (unsigned long long)P);
#endif
    }
    if (!saved) {
      // no saved keys: key pass, rank prefix, column emission (staging
      // buffer overlays the value slots, then zero them again)
      if (single) {
        block_chunk_products<false, V>(E, nent, P, B.col, bv, so);
        __syncthreads();
      } else {
        for (int64_t t = t0; t < t1; t += NT) {
          P = block_load_tiles<false, V>(t, t1, c0, c1, it.last, A.col, av, B.ptr, B.col, bt, E, scr, nent);
          block_chunk_products<false, V>(E, nent, P, B.col, bv, so);
          __syncthreads();
        }
      }
      window_prefix32<NT>(wp, 2 * nwords, scr);
      int* colbuf = reinterpret_cast<int*>(vals);
      for (int i = threadIdx.x; i < 2 * nwords; i += NT) {
        const uint2 p = wp[i];
        emit_bits32_smem(p.x, c0 + 32 * i, colbuf + p.y);
      }
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += NT) st_stream(out_col + it.out_base + i, colbuf[i]);
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += NT) vals[i] = 0.0;
      __syncthreads();
    }
    SG_PH(2);
    // the next ticket's round trip overlaps this window's value pass; it is
    // published after the pass (item_next was last read before the setup
    // barrier above)
    unsigned long long nb = 0;
    if (threadIdx.x == 0) nb = atomicAdd(ticket, 1ull);
    if (single) {
      block_chunk_products<true, V>(E, nent, P, B.col, bv, ao);
      __syncthreads();
    } else {
      for (int64_t t = t0; t < t1; t += NT) {
        P = block_load_tiles<true, V>(t, t1, c0, c1, it.last, A.col, av, B.ptr, B.col, bt, E, scr, nent);
        block_chunk_products<true, V>(E, nent, P, B.col, bv, ao);
        __syncthreads();
      }
    }
    SG_PH(4);
    if (threadIdx.x == 0) item_next = (int64_t)nb;
    for (int i = threadIdx.x; i < cnt; i += NT) st_stream(out_val + it.out_base + i, (V)vals[i]);
    __syncthreads();
    SG_PH(5);
#ifdef SG_PROF
    if (threadIdx.x == 0) {
      atomicAdd(&g_phase[9], 1ull);
      atomicAdd(&g_phase[10], (unsigned long long)nwords);
      atomicAdd(&g_phase[11], (unsigned long long)cnt);
    }
#endif
    b = item_next;
  }
}

// -------------------------------------------------------------------------
// KW: warp-specialised window accumulator for long rows with saved bitmaps.
//
// One persistent 1024-thread CTA per SM, two windows in flight:
//   producer warps (KW_PW) take window tickets, bulk-copy the window's saved
//     {bits, rank} words into one of two bitmap buffers (cp.async.bulk, an
//     mbarrier counts the bytes), clip every A entry's B row to the window
//     (B tile index) and publish the non-empty segments in chunks (segment
//     table {B offset - product start, A value} + a 32-product group table);
//   consumer warps (KW_CW) take 4-group steps of the current chunk from a
//     shared counter (no block barrier anywhere), find each product's segment
//     with one broadcast load + popcount, gather (col, val) from B, rank the
//     column in the window bitmap and add a*b into the window's fp64 values
//     in shared memory; the warp that finishes a window last stores its
//     values (coalesced, streaming) and zeroes them.
// Chunks (two slots) and windows (two value / bitmap buffers) are handed
// over with mbarriers, so clipping, bitmap loads and value stores of one
// window overlap the value pass of the other.  Replaces the
// setup -> clip -> values -> store phases of k_bmr behind block barriers.
// Reference: the long-row part of _numeric_phase / _fallback_phase
// (engine.py:252-328), fallback_accumulate (accumulate.py:274-279).

#ifdef SG_PROF
#define KW_T0() const long long _kt0 = clock64()
#define KW_ACC(acc) (acc) += (unsigned long long)(clock64() - _kt0)
#else
#define KW_T0()
#define KW_ACC(acc)
#endif
constexpr int KW_NT = 1024;
#ifndef SG_KW_PW
#define SG_KW_PW 8
#endif
#ifndef SG_KW_SEG
#define SG_KW_SEG 256
#endif
#ifndef SG_KW_NCH
#define SG_KW_NCH 4
#endif
constexpr int KW_PW = SG_KW_PW;              // producer warps
constexpr int KW_CW = KW_NT / 32 - KW_PW;    // consumer warps
constexpr int KW_NP = KW_PW * 32;            // producer threads (one A entry each per batch)
constexpr int KW_SEG = SG_KW_SEG;            // segments per chunk
constexpr int KW_GRP = SG_KW_SEG;            // 32-product groups per chunk
constexpr int KW_NCH = SG_KW_NCH;            // chunk slots (the producer runs up to KW_NCH chunks ahead)
constexpr int KW_PMAX = 32 * KW_GRP;         // products per chunk
#ifndef SG_KW_U
#define SG_KW_U 4
#endif
#ifndef SG_KW_SLEEP
#define SG_KW_SLEEP 200
#endif
constexpr int KW_U = SG_KW_U;                // groups per consumer step

enum : int { KW_FIRST = 1, KW_LAST = 2, KW_END = 4 };

struct KwChunk {
  int64_t d[KW_SEG];       // B position of chunk product p of segment c = d[c] + p
  double av[KW_SEG];       // A value of segment c
  int32_t S[KW_SEG + 2];   // chunk-relative first product of segment c
  int2 grp[KW_GRP];        // group g: {segment of product 32g, segment starts in (32g, 32g+32)}
  int64_t out_base;        // C index of the window's first entry
  int32_t P, ng, wslot, flags, c0, cnt, rank0, nwords;
  uint32_t next;           // consumer step counter
};

// fp64 window values leave through a bulk shared->global copy and are
// re-zeroed by a bulk copy from this zero buffer: a slot holds WIN_R values
// from element 0 or 1 (C's first value's address mod 16), so the body of the
// copy is 16-byte aligned on both sides
constexpr int KW_VSLOT = WIN_R + 2;
#ifndef SG_KW_NWS
#define SG_KW_NWS 2
#endif
constexpr int KW_NWS = SG_KW_NWS;  // window slots in flight per CTA
__device__ __align__(16) double g_kw_zero[KW_VSLOT];

struct KwShared {
  double vals[KW_NWS][KW_VSLOT];
  uint4 bm[KW_NWS][WIN_WORDS];
  KwChunk ch[KW_NCH];
  // win_done[s]: every consumer thread arrives once it is done with the
  // slot's window (products and column emission); the producer then stores
  // the window's values and loads the slot's next window
  unsigned long long full[KW_NCH], empty[KW_NCH], bm_full[KW_NWS], win_done[KW_NWS];
  unsigned col_next[KW_NWS];  // column-emission work counter of each window slot
  WinItem items[4];        // producer's work-item ring (loaded two windows ahead)
  int pscan[2][KW_PW + 1];
  int pexcl[KW_NP + 1];
  int64_t ticket;
};
static_assert(sizeof(KwShared) <= 227 * 1024, "k_win shared memory");


__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1; }" ::"r"(
                   smem_u32(b)),
               "r"(bytes)
               : "memory");
}
// wait for the completion of the phase with the given parity (backing off
// so that waiting warps leave the issue slots to the working ones)
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  const uint32_t a = smem_u32(b);
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(SG_KW_SLEEP);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void pbar() { asm volatile("bar.sync 1, %0;" ::"n"(KW_NP) : "memory"); }
__device__ __forceinline__ int pbar_popc(bool p) {
  int r;
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, 0; bar.red.popc.u32 %0, 1, %2, q; }"
               : "=r"(r)
               : "r"((unsigned)p), "n"(KW_NP)
               : "memory");
  return r;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// Per A entry of a windowed row, resolved once per call instead of once per
// (entry, window): B row start and length, its tile-index row, the A value.
// Heavy entries (B rows of >= lh entries) go to k_win, light ones to
// k_win_light; each list is compacted per row at the row's A offset.
struct KwEnt {
  int64_t bs;   // B row start
  int64_t to;   // B tile index row (-1: none, binary search)
  double av;    // A value
  int32_t len;  // B row length
  int32_t pad;
};

template <typename V, int NT>
__global__ void __launch_bounds__(NT) k_win_entries(int64_t m, const int32_t* __restrict__ nwin, Csr A,
                                                    const int64_t* __restrict__ b_ptr, BTile bt, int lh,
                                                    KwEnt* __restrict__ hent, int32_t* __restrict__ hcnt,
                                                    KwEnt* __restrict__ lent, int32_t* __restrict__ lcnt) {
  __shared__ int64_t scr[NT / 32 + 2];
  const V* av = (const V*)A.val;
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    if (nwin[row] <= 0) {
      if (threadIdx.x == 0) hcnt[row] = lcnt[row] = 0;  // no windows: nothing for k_win / k_win_light
      continue;
    }
    const int64_t t0 = A.ptr[row], t1 = A.ptr[row + 1];
    int64_t nh = 0, nl = 0;
    for (int64_t t = t0; t < t1; t += NT) {
      KwEnt e{0, -1, 0.0, 0, 0};
      int kind = 0;  // 1 heavy, 2 light
      if (t + threadIdx.x < t1) {
        const int32_t k = A.col[t + threadIdx.x];
        e.bs = b_ptr[k];
        e.len = (int32_t)(b_ptr[k + 1] - e.bs);
        e.to = bt.off ? bt.off[k] : -1;
        e.av = (double)av[t + threadIdx.x];
        kind = e.len <= 0 ? 0 : (e.len >= lh ? 1 : 2);  // empty B rows contribute nothing
      }
      int64_t tot;
      const int64_t ex = block_excl_scan((int64_t)(kind == 1) | ((int64_t)(kind == 2) << 32), scr, &tot);
      if (kind == 1) hent[t0 + nh + (ex & 0xffffffffll)] = e;
      if (kind == 2) lent[t0 + nl + (ex >> 32)] = e;
      nh += tot & 0xffffffffll;
      nl += tot >> 32;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      hcnt[row] = (int32_t)nh;
      lcnt[row] = (int32_t)nl;
    }
  }
}

// a heavy entry's B row clipped to the window [c0, c1): (start, length)
__device__ __forceinline__ void kw_clip(const KwEnt& en, const int32_t* __restrict__ b_col, BTile bt, int32_t c0,
                                        int32_t c1, bool last, int64_t& bs, int& len) {
  const int64_t s = en.bs, e = en.bs + en.len;
  int64_t ss, ee;
  if (en.to >= 0) {
    ss = s + bt.tbl[en.to + c0 / TILE_COLS];
    ee = last ? e : s + bt.tbl[en.to + c1 / TILE_COLS];
  } else {
    ss = lower_bound_col(b_col, s, e, c0);
    ee = last ? e : lower_bound_col(b_col, ss, e, c1);
  }
  bs = ss;
  len = (int)(ee - ss);
}

// fp64 window values leave through the copy engine (SG_KW_BULK=0: plain
// stores by the producer threads -- e.g. for compute-sanitizer initcheck,
// which does not see the copy engine's global writes)
#ifndef SG_KW_BULK
#define SG_KW_BULK 1
#endif
template <typename V>
__host__ __device__ constexpr bool kw_bulk() {
  return sizeof(V) == 8 && SG_KW_BULK;
}

// Store the values of the window that held slot ws (all consumer warps have
// arrived on win_done[ws]) and leave the slot zeroed (float) or to be zeroed
// by the next bulk load (fp64).  fp64: tid 0 hands them to the copy engine --
// one bulk shared->global copy of the 16-byte aligned body, head / tail
// element apart -- and waits until the copy has read the slot.
template <typename V>
__device__ __forceinline__ void kw_store_window(KwShared& sh, unsigned ws, V* __restrict__ out_val,
                                                int64_t out_base, int cnt, int tid) {
  const uint32_t vs = smem_u32(&sh.vals[ws][0]);
  V* dst = out_val + out_base;
  if constexpr (kw_bulk<V>()) {
    if (tid == 0) {
      const uint32_t vshift = (uint32_t)((reinterpret_cast<uintptr_t>(dst) >> 3) & 1u);  // see KW_VSLOT
      const int head = (int)vshift < cnt ? (int)vshift : 0;
      const int body = (cnt - head) & ~1;
      if (head) st_stream(dst, (V)lds_f64(vs + 8u));
      if (head + body < cnt) st_stream(dst + head + body, (V)lds_f64(vs + (vshift + head + body) * 8u));
      if (body > 0) {
        bulk_s2g(dst + head, vs + (vshift + head) * 8u, (unsigned)body * 8u);
        bulk_commit_wait_read();  // the slot may be re-zeroed once read
      }
    }
  } else {
    for (int i = tid; i < cnt; i += KW_NP) {
      st_stream(dst + i, (V)lds_f64(vs + i * 8u));
      sts_f64(vs + i * 8u, 0.0);
    }
  }
}

template <typename V>
__device__ __forceinline__ void kw_producer(KwShared& sh, int64_t nwork, const WinItem* __restrict__ work,
                                            const Csr& A, const Csr& B, const BTile& bt,
                                            const uint4* __restrict__ bm16, const KwEnt* __restrict__ hent,
                                            V* __restrict__ out_val, unsigned long long* ticket) {
  (void)A;
  (void)ticket;
  const int tid = threadIdx.x;  // 0 .. KW_NP-1
  const int lane = lane_id(), pw = warp_id();
  unsigned wseq = 0, cseq = 0;
  int nprod = 0, nseg = 0;
  KwChunk* ch = nullptr;

  unsigned long long pc_free = 0, pc_empty = 0, pc_append = 0, pc_pub = 0, pc_clip = 0;
  (void)pc_free; (void)pc_empty; (void)pc_append; (void)pc_pub; (void)pc_clip;
  auto acquire = [&]() {
    const unsigned cs = cseq % KW_NCH;
    KW_T0();
    mbar_wait(&sh.empty[cs], ((cseq / KW_NCH) & 1u) ^ 1u);
    KW_ACC(pc_empty);
    ch = &sh.ch[cs];
    nprod = nseg = 0;
  };
  bool copy_pending = false;
  const WinItem* copy_item = nullptr;
  unsigned copy_slot = 0, copy_wseq = 0;
  int64_t prev_base[KW_NWS];  // C offset / values of the window last loaded into each slot
  int prev_cnt[KW_NWS];
  // wait until the consumers are done with the window in slot ws (its u-th
  // use), then store its values
  auto release = [&](unsigned ws, unsigned u) {
    mbar_wait(&sh.win_done[ws], u & 1u);
    kw_store_window<V>(sh, ws, out_val, prev_base[ws], prev_cnt[ws], tid);
    if (!kw_bulk<V>()) pbar();
  };
  auto publish = [&](int flags, const WinItem& it, unsigned wslot) {
    if (copy_pending) {
      KW_T0();
      if (copy_wseq >= KW_NWS) release(copy_slot, copy_wseq / KW_NWS - 1u);
      KW_ACC(pc_free);
      prev_base[copy_slot] = copy_item->out_base;
      prev_cnt[copy_slot] = copy_item->cnt;
      if (tid == 0) {
        sh.col_next[copy_slot] = 0;
        const unsigned nwords = (unsigned)(((int64_t)copy_item->c1 - copy_item->c0 + 63) >> 6);
        // fp64: the slot's values [0, shift + cnt) re-zeroed by the copy engine
        const unsigned zb = kw_bulk<V>() ? ((1u + (unsigned)copy_item->cnt) * 8u + 15u) & ~15u : 0u;
        mbar_arrive_tx(&sh.bm_full[copy_slot], nwords * 16u + zb);
        bulk_g2s(&sh.bm[copy_slot][0], bm16 + copy_item->bm_word, nwords * 16u, &sh.bm_full[copy_slot]);
        if (zb) bulk_g2s(&sh.vals[copy_slot][0], g_kw_zero, zb, &sh.bm_full[copy_slot]);
      }
      copy_pending = false;
    }
    // group table of the chunk: owner of every group's first product and
    // the segment starts inside the group (S strictly increasing)
    KW_T0();
    const int ng = (nprod + 31) >> 5;
    if (tid == 0) ch->S[nseg] = nprod;
    pbar();
    for (int g = tid; g < ng; g += KW_NP) {
      const int q = 32 * g;
      int lo = 0, hi = nseg - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ch->S[mid] <= q) lo = mid; else hi = mid - 1;
      }
      unsigned mask = 0;
      for (int c = lo + 1; c < nseg; ++c) {
        const int dd = ch->S[c] - q;
        if (dd >= 32) break;
        mask |= 1u << dd;
      }
      ch->grp[g] = make_int2(lo, (int)mask);
    }
    if (tid == 0) {
      ch->P = nprod;
      ch->ng = ng;
      ch->wslot = (int)wslot;
      ch->flags = flags;
      ch->c0 = it.c0;
      ch->cnt = it.cnt;
      ch->rank0 = it.rank0;
      ch->nwords = (int)(((int64_t)it.c1 - it.c0 + 63) >> 6);
      ch->out_base = it.out_base;
      ch->next = 0;
    }
    // every producer thread arrives once its own table entries are written
    // (the full barrier counts KW_NP arrivals): no second block barrier
    mbar_arrive(&sh.full[cseq % KW_NCH]);
    ++cseq;
    KW_ACC(pc_pub);
  };
  // one batch of KW_NP entries into the chunk(s): scan, append, publish full
  // chunks.  (bs, len, a) is this thread's clipped segment.
  unsigned spar = 0;  // parity of the double-buffered warp totals
  auto append = [&](int64_t bs, int len, double a, int& flags, const WinItem& it, unsigned wslot) {
    KW_T0();
    const int pk = (len << 9) | (len > 0 ? 1 : 0);  // (length, non-empty)
    const int inc = warp_incl_scan(pk);
    int* ps = sh.pscan[spar];
    spar ^= 1u;
    if (lane == 31) ps[pw] = inc;
    pbar();
    int wbase = 0, btot = 0;
#pragma unroll
    for (int w = 0; w < KW_PW; ++w) {
      const int x = ps[w];
      wbase += w < pw ? x : 0;
      btot += x;
    }
    const int excl = wbase + inc - pk;
    if (nprod + (btot >> 9) <= KW_PMAX && nseg + (btot & 511) <= KW_SEG) {
      // common case: the whole batch fits the open chunk -- one barrier
      if (len > 0) {
        const int c = nseg + (excl & 511);
        const int S = nprod + (excl >> 9);
        ch->S[c] = S;
        ch->d[c] = bs - S;
        ch->av[c] = a;
      }
      nprod += btot >> 9;
      nseg += btot & 511;
      KW_ACC(pc_append);
      return;
    }
    sh.pexcl[tid] = excl;
    if (tid == KW_NP - 1) sh.pexcl[KW_NP] = excl + pk;
    pbar();
    int from = 0;
    while (from < KW_NP) {
      const int base = sh.pexcl[from];
      const int rel_in = excl + pk - base;  // inclusive, relative to `from`
      const bool fits = tid >= from && nprod + (rel_in >> 9) <= KW_PMAX && nseg + (rel_in & 511) <= KW_SEG;
      const int nfit = pbar_popc(fits);
      if (fits && len > 0) {
        const int rel_ex = excl - base;
        const int c = nseg + (rel_ex & 511);
        const int S = nprod + (rel_ex >> 9);
        ch->S[c] = S;
        ch->d[c] = bs - S;
        ch->av[c] = a;
      }
      const int tot = sh.pexcl[from + nfit] - base;
      nprod += tot >> 9;
      nseg += tot & 511;
      from += nfit;
      if (from < KW_NP) {  // chunk full: publish it, continue in the next slot
        publish(flags, it, wslot);
        flags = 0;
        acquire();
      }
    }
    pbar();  // pexcl / pscan reuse
    KW_ACC(pc_append);
  };
  auto clip_of = [&](const WinItem& it, int64_t t, int64_t t1, int64_t& bs, int& len, double& a) {
    bs = 0;
    len = 0;
    a = 0.0;
    if (t < t1) {
      const KwEnt en = hent[t];
      kw_clip(en, B.col, bt, it.c0, it.c1, it.last != 0, bs, len);
      a = en.av;
    }
  };

  // Static round-robin over the work items (neighbouring items are alike:
  // same column bucket).  The producer walks the flattened sequence of
  // entry batches (KW_NP entries of one window; every window has >= 1) as a
  // three-stage software pipeline: at each step the entry records of the
  // batch two ahead are loaded, the batch one ahead is clipped (B tile index
  // loads in flight), and the current batch -- clipped one step ago -- is
  // scanned and appended.  The dependent global round trips (entry record,
  // then tile index) thus overlap two steps of barrier / shared-memory work.
  // Work items live in a 4-entry shared ring, loaded three windows ahead.
  const int64_t G = gridDim.x;
  const int64_t b0 = blockIdx.x;
  const int64_t nmine = b0 < nwork ? (nwork - 1 - b0) / G + 1 : 0;  // windows of this CTA
  auto load_item = [&](int64_t k) {  // 12 threads copy one 48-byte item into the ring
    const int64_t bb = b0 + k * G;
    if (tid < 12 && k < nmine)
      reinterpret_cast<int32_t*>(&sh.items[k & 3])[tid] = reinterpret_cast<const int32_t*>(work + bb)[tid];
  };
  for (int64_t k = 0; k < 3; ++k) load_item(k);
  pbar();
  // batch cursor: window k (of this CTA), first entry offset tb within it
  struct Cur {
    int64_t k;
    int tb;
  };
  auto advance = [&](Cur c) {
    const WinItem& w = sh.items[c.k & 3];
    if (c.tb + KW_NP < w.t_len) return Cur{c.k, c.tb + KW_NP};
    return Cur{c.k + 1, 0};
  };
  auto load_ent = [&](Cur c, KwEnt& e) {
    e = KwEnt{0, -1, 0.0, 0, 0};
    if (c.k < nmine) {
      const WinItem& w = sh.items[c.k & 3];
      if (c.tb + tid < w.t_len) e = hent[w.t0 + c.tb + tid];
    }
  };
  auto clip_ent = [&](Cur c, const KwEnt& e, int64_t& bs, int& len, double& a) {
    bs = 0;
    len = 0;
    a = 0.0;
    if (c.k < nmine && e.len > 0) {
      const WinItem& w = sh.items[c.k & 3];
      kw_clip(e, B.col, bt, w.c0, w.c1, w.last != 0, bs, len);
      a = e.av;
    }
  };
  Cur c0{0, 0}, c1 = c0, c2 = c0;
  KwEnt e1, e2;
  int64_t bs0 = 0;
  int len0 = 0;
  double a0 = 0.0;
  if (nmine > 0) {
    c1 = advance(c0);
    c2 = c1.k < nmine ? advance(c1) : c1;
    KwEnt e0;
    load_ent(c0, e0);
    load_ent(c1, e1);
    clip_ent(c0, e0, bs0, len0, a0);
  }
  int flags = 0;
  int64_t kcur = -1;
  while (c0.k < nmine) {
    // new window: fresh chunk, bitmap copy pending until its first publish,
    // ring slot of the window three ahead refilled
    if (c0.k != kcur) {
      kcur = c0.k;
      load_item(kcur + 3);
      copy_pending = true;
      copy_item = &sh.items[kcur & 3];
      copy_slot = wseq % KW_NWS;
      copy_wseq = wseq;
      acquire();
      flags = KW_FIRST;
    }
    load_ent(c2, e2);                  // stage 0: records of the batch two ahead
    int64_t bs1;
    int len1;
    double a1;
    {
      KW_T0();
      clip_ent(c1, e1, bs1, len1, a1);  // stage 1: tile-index loads in flight
      KW_ACC(pc_clip);
    }
    const WinItem it = sh.items[c0.k & 3];
    const unsigned wslot = wseq % KW_NWS;
    append(bs0, len0, a0, flags, it, wslot);  // stage 2
    if (c1.k != c0.k) {  // c0 was the window's last batch
      publish(flags | KW_LAST, it, wslot);
      ++wseq;
    }
    c0 = c1;
    bs0 = bs1;
    len0 = len1;
    a0 = a1;
    c1 = c2;
    e1 = e2;
    c2 = c2.k < nmine ? advance(c2) : c2;
  }
  acquire();
  WinItem none{};
  publish(KW_END, none, 0);
  // the last window of each slot
  for (unsigned w = wseq >= KW_NWS ? wseq - KW_NWS : 0; w < wseq; ++w) release(w % KW_NWS, w / KW_NWS);
  if (kw_bulk<V>() && tid == 0) bulk_wait_all();  // value stores complete before exit
#ifdef SG_PROF
  if (tid == 0) {
    atomicAdd(&g_kw[0], pc_free);
    atomicAdd(&g_kw[1], pc_empty);
    atomicAdd(&g_kw[2], pc_append);
    atomicAdd(&g_kw[3], pc_pub);
    atomicAdd(&g_kw[4], pc_clip);
    atomicAdd(&g_kw[5], (unsigned long long)wseq);
  }
#endif
}

template <typename V>
__device__ __forceinline__ void kw_consumer(KwShared& sh, const Csr& B, int32_t* __restrict__ out_col,
                                            V* __restrict__ out_val) {
  const int lane = lane_id();
  const unsigned le = lanemask_le();
  const int32_t* __restrict__ b_col = B.col;
  const V* __restrict__ b_val = (const V*)B.val;
  unsigned cseq = 0;
  unsigned wuse[KW_NWS];
#pragma unroll
  for (int j = 0; j < KW_NWS; ++j) wuse[j] = 0u;
  unsigned long long cc_full = 0, cc_bm = 0, cc_grp = 0, cc_col = 0, cc_store = 0;
  (void)cc_full; (void)cc_bm; (void)cc_grp; (void)cc_col; (void)cc_store;
  for (;;) {
    const unsigned cs = cseq % KW_NCH;
    {
      KW_T0();
      mbar_wait(&sh.full[cs], (cseq / KW_NCH) & 1u);
      KW_ACC(cc_full);
    }
    KwChunk& ch = sh.ch[cs];
    const int flags = ch.flags;
    if (flags & KW_END) break;
    const int ng = ch.ng, P = ch.P, ws = ch.wslot, c0 = ch.c0, cnt = ch.cnt, rank0 = ch.rank0,
              nwords = ch.nwords;
    const int64_t out_base = ch.out_base;
    if (flags & KW_FIRST) {
      KW_T0();
      mbar_wait(&sh.bm_full[ws], wuse[ws] & 1u);
      ++wuse[ws];
      KW_ACC(cc_bm);
    }
#ifdef SG_PROF
    const long long _kg = clock64();
#endif
    // (see KW_VSLOT) values from slot element 1 when C's first value is not 16-byte aligned
    const uint32_t vshift =
        kw_bulk<V>() ? (uint32_t)((reinterpret_cast<uintptr_t>(out_val + out_base) >> 3) & 1u) : 0u;
    WinAddOp op{smem_u32(&sh.bm[ws][0]), smem_u32(&sh.vals[ws][0]) + (vshift - (uint32_t)rank0) * 8u, c0};
    const uint32_t grp_s = smem_u32(&ch.grp[0]), d_s = smem_u32(&ch.d[0]), av_s = smem_u32(&ch.av[0]);
    for (;;) {
      unsigned g0 = 0;
      if (lane == 0) g0 = atomicAdd(&ch.next, (unsigned)KW_U);
      g0 = __shfl_sync(SG_FULL, g0, 0);
      if ((int)g0 >= ng) break;
      int32_t col[KW_U];
      double v[KW_U];
      if (((int)g0 + KW_U) * 32 <= P) {
#pragma unroll
        for (int u = 0; u < KW_U; ++u) {
          const uint2 gr = lds_v2u32(grp_s + (g0 + u) * 8u);
          const uint32_t c = gr.x + (uint32_t)__popc(gr.y & le);
          const int64_t pos = lds_s64(d_s + c * 8u) + (int64_t)(((int)g0 + u) * 32 + lane);
          col[u] = __ldg(b_col + pos);
          v[u] = lds_f64(av_s + c * 8u) * (double)__ldg(b_val + pos);
        }
#pragma unroll
        for (int u = 0; u < KW_U; ++u) op(col[u], v[u]);
      } else {
        bool ok[KW_U];
#pragma unroll
        for (int u = 0; u < KW_U; ++u) {
          const int p = ((int)g0 + u) * 32 + lane;
          ok[u] = p < P;
          col[u] = 0;
          v[u] = 0.0;
          if (ok[u]) {
            const uint2 gr = lds_v2u32(grp_s + (g0 + u) * 8u);
            const uint32_t c = gr.x + (uint32_t)__popc(gr.y & le);
            const int64_t pos = lds_s64(d_s + c * 8u) + (int64_t)p;
            col[u] = __ldg(b_col + pos);
            v[u] = lds_f64(av_s + c * 8u) * (double)__ldg(b_val + pos);
          }
        }
#pragma unroll
        for (int u = 0; u < KW_U; ++u)
          if (ok[u]) op(col[u], v[u]);
      }
    }
#ifdef SG_PROF
    cc_grp += (unsigned long long)(clock64() - _kg);
#endif
    __syncwarp();
    if (flags & KW_LAST) __threadfence_block();
    if (lane == 0) mbar_arrive(&sh.empty[cs]);
    if (flags & KW_LAST) {
      // C's columns of the window, straight from the bitmap in shared memory
      // (its 32-bit halves carry their row rank): every consumer warp that is
      // done with the window takes 128-half-word slices until none are left
      KW_T0();
      if (out_col) {
        const uint32_t bmw = smem_u32(&sh.bm[ws][0]);
        const int nh = 2 * nwords;
        int32_t* oc = out_col + out_base - rank0;
        for (;;) {
          unsigned j = 0;
          if (lane == 0) j = atomicAdd(&sh.col_next[ws], 128u);
          j = __shfl_sync(SG_FULL, j, 0);
          if ((int)j >= nh) break;
          const int hend = min((int)j + 128, nh);
          for (int h = (int)j + lane; h < hend; h += 32) {
            const uint2 p = lds_u2(bmw + (uint32_t)h * 8u);
            unsigned bits = p.x;
            int32_t* o = oc + p.y;
            const int32_t cb = c0 + 32 * h;
            while (bits) {
              st_stream(o++, cb + __ffs(bits) - 1);
              bits &= bits - 1;
            }
          }
        }
      }
      KW_ACC(cc_col);
      __threadfence_block();
      fence_proxy_async_smem();  // this warp's bitmap reads / value adds -> the bulk copies
      mbar_arrive(&sh.win_done[ws]);  // every lane: its own reads are ordered before the release
      KW_ACC(cc_store);
    }
    ++cseq;
  }
#ifdef SG_PROF
  if (lane == 0) {
    atomicAdd(&g_kw[8], cc_full);
    atomicAdd(&g_kw[9], cc_bm);
    atomicAdd(&g_kw[10], cc_grp);
    atomicAdd(&g_kw[11], cc_col);
    atomicAdd(&g_kw[12], cc_store);
    atomicAdd(&g_kw[13], (unsigned long long)cseq);
  }
#endif
}

// Light entries of the windowed rows: products of B rows shorter than lh
// (which k_win skips) are added straight into C's values with fire-and-forget
// fp64 REDs at the column's row rank, read from the row's saved bitmap (L2).
// R-MAT-20: B rows < 256 carry 4.4% of the long-row products but 57% of the
// long rows' A entries, i.e. of the window kernel's clipping work.
template <typename V>
struct LightOp {
  const uint2* bm;  // the row's saved {bits, rank} pairs, one per 32 columns
  int32_t org;      // column of the row's first saved bit
  V* out;           // C values of the row
  __device__ __forceinline__ void operator()(int32_t col, double v) {
    const uint32_t x = (uint32_t)(col - org);
    const uint2 p = __ldg(bm + (x >> 5));
    gmem_red(out + (p.y + __popc(p.x & ((2u << (x & 31)) - 1u)) - 1u), (V)v);
  }
};

// The light entries' products are combined per row in a shared-memory hash
// (column -> fp64 sum, open addressing) and the table is flushed -- one RED
// per distinct column at its row rank -- whenever it could overflow within
// the next round of entries, and at the row's end.  Hot columns (hub
// columns receive thousands of light products per dense row) are thereby
// summed in shared memory instead of serialising at one L2 address.
constexpr int KL_NT = 512, KL_LOG2T = 13, KL_T = 1 << KL_LOG2T;

template <typename V>
__global__ void __launch_bounds__(KL_NT, 2) k_win_light(int64_t m, const int32_t* __restrict__ lcnt, Csr A, Csr B,
                                                        const int64_t* __restrict__ span_lo,
                                                        const int64_t* __restrict__ bm_off,
                                                        const uint4* __restrict__ bm16,
                                                        const int64_t* __restrict__ row_ptr,
                                                        const KwEnt* __restrict__ lent, V* __restrict__ out_val) {
  extern __shared__ __align__(16) unsigned char smem[];
  int* keys = reinterpret_cast<int*>(smem);
  double* vals = reinterpret_cast<double*>(smem + KL_T * 4);
  __shared__ int cnt;
  constexpr int NW = KL_NT / 32;
  const int w = warp_id(), lane = lane_id();
  const int32_t* __restrict__ b_col = B.col;
  const V* __restrict__ b_val = (const V*)B.val;
  for (int i = threadIdx.x; i < KL_T; i += KL_NT) keys[i] = -1;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    const int n = lcnt[row];
    if (n <= 0) continue;
    const uint2* bm = reinterpret_cast<const uint2*>(bm16 + bm_off[row]);
    const int32_t org = (int32_t)win_origin(span_lo[row]);
    V* out = out_val + row_ptr[row];
    const KwEnt* le = lent + A.ptr[row];
    auto flush = [&]() {
      __syncthreads();
      for (int i = threadIdx.x; i < KL_T; i += KL_NT) {
        const int k = keys[i];
        if (k != -1) {
          const uint32_t x = (uint32_t)(k - org);
          const uint2 q = __ldg(bm + (x >> 5));
          gmem_red(out + (q.y + __popc(q.x & ((2u << (x & 31)) - 1u)) - 1u), (V)vals[i]);
          keys[i] = -1;
        }
      }
      if (threadIdx.x == 0) cnt = 0;
      __syncthreads();
    };
    // rounds of NW entries (one per warp, lanes over its B row: < lh <= 256
    // products, so a round adds at most NW * 255 keys)
    for (int j0 = 0; j0 < n; j0 += NW) {
      if (cnt > 3 * KL_T / 4 - NW * 256) flush();  // keeps the load factor <= 3/4
      const int j = j0 + w;
      if (j < n) {
        const KwEnt en = le[j];
        for (int q = lane; q < en.len; q += 32) {
          const int32_t col = __ldg(b_col + en.bs + q);
          const double v = en.av * (double)__ldg(b_val + en.bs + q);
          uint32_t s = slot_hash((uint32_t)col, KL_LOG2T);
          for (;;) {
            int k = reinterpret_cast<volatile int*>(keys)[s];
            if (k == -1) {
              const int old = atomicCAS(&keys[s], -1, col);
              if (old == -1) {
                atomicAdd(&cnt, 1);
                k = col;
              } else {
                k = old;
              }
            }
            if (k == col) {
              smem_add(&vals[s], v);
              break;
            }
            s = (s + 1) & (KL_T - 1);
          }
        }
      }
      __syncthreads();
    }
    flush();
  }
}

template <typename V>
__global__ void __launch_bounds__(KW_NT, 1) k_win(int64_t nwork, const WinItem* __restrict__ work, Csr A, Csr B,
                                                  BTile bt, const uint4* __restrict__ bm16,
                                                  const KwEnt* __restrict__ hent, int32_t* __restrict__ out_col,
                                                  V* __restrict__ out_val, unsigned long long* __restrict__ ticket) {
  extern __shared__ __align__(128) unsigned char kw_smem[];
  KwShared& sh = *reinterpret_cast<KwShared*>(kw_smem);
  for (int i = threadIdx.x; i < KW_NWS * KW_VSLOT; i += KW_NT) (&sh.vals[0][0])[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int j = 0; j < KW_NCH; ++j) {
      mbar_init(&sh.full[j], KW_NP);
      mbar_init(&sh.empty[j], KW_CW);
    }
    for (int j = 0; j < KW_NWS; ++j) {
      mbar_init(&sh.bm_full[j], 1);
      mbar_init(&sh.win_done[j], KW_CW * 32);
      sh.col_next[j] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp_id() < KW_PW)
    kw_producer<V>(sh, nwork, work, A, B, bt, bm16, hent, out_val, ticket);
  else
    kw_consumer<V>(sh, B, out_col, out_val);
}


// Work items: one per used window, grouped into NBUCKET column-range buckets
// (bucket = c0 * NBUCKET / ncols) so the dynamic ticket order sweeps B's
// columns once.
constexpr int NBUCKET = 64;

__device__ __forceinline__ int win_bucket(int32_t c0, int64_t ncols) {
  return (int)min((int64_t)NBUCKET - 1, ((int64_t)c0 * NBUCKET) / max(ncols, (int64_t)1));
}

// window class: 0 = full CTA, 1 = small (fits a half-size CTA)
__device__ __forceinline__ int win_class(int64_t cnt, int32_t c0, int32_t c1) {
  return (cnt <= SMALL_R && ((int64_t)c1 - c0 + 63) / 64 <= SMALL_WORDS) ? 1 : 0;
}

// walks the used windows of row i: f(c0, c1, last, cnt, rank0)
template <class F>
__device__ __forceinline__ void for_each_window(const int2* wr, int n, int64_t rowcnt, int32_t hi1, F f) {
  int j = 0;
  while (j < n && wr[j].x < 0) ++j;
  while (j < n) {
    const int2 me = wr[j];
    int k = j + 1;
    while (k < n && wr[k].x < 0) ++k;
    const int32_t c1 = k < n ? wr[k].x : hi1;
    const int64_t cnt = (k < n ? (int64_t)wr[k].y : rowcnt) - me.y;
    f(me.x, c1, k >= n, cnt, me.y);
    j = k;
  }
}

// window class: 2 = the row's words were saved (k_win), else the k_bmr
// geometry class (win_class)
__global__ void k_win_counts(int64_t m, int64_t ncols, const int64_t* __restrict__ win_off,
                             const int2* __restrict__ wins, const int32_t* __restrict__ nwin,
                             const int64_t* __restrict__ span_hi, const int64_t* __restrict__ out_off,
                             const int64_t* __restrict__ bm_off, unsigned long long* __restrict__ bucket_cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int n = nwin[i];
  if (n <= 0) return;
  const bool saved = bm_off && bm_off[i + 1] > bm_off[i];
  for_each_window(wins + win_off[i], n, out_off[i + 1] - out_off[i], (int32_t)(span_hi[i] + 1),
                  [&](int32_t c0, int32_t c1, bool, int64_t cnt, int32_t) {
                    const int cls = saved ? 2 : win_class(cnt, c0, c1);
                    atomicAdd(&bucket_cnt[cls * NBUCKET + win_bucket(c0, ncols)], 1ull);
                  });
}

__global__ void k_win_scatter(int64_t m, int64_t ncols, const int64_t* __restrict__ a_ptr,
                              const int64_t* __restrict__ span_lo, const int64_t* __restrict__ span_hi,
                              const int64_t* __restrict__ win_off, const int2* __restrict__ wins,
                              const int32_t* __restrict__ nwin, const int64_t* __restrict__ out_off,
                              const int64_t* __restrict__ bm_off, const int32_t* __restrict__ heavy_cnt,
                              unsigned long long* __restrict__ cursor, WinItem* __restrict__ work) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int n = nwin[i];
  if (n <= 0) return;
  const int64_t org = win_origin(span_lo[i]);
  const bool saved = bm_off && bm_off[i + 1] > bm_off[i];
  for_each_window(wins + win_off[i], n, out_off[i + 1] - out_off[i], (int32_t)(span_hi[i] + 1),
                  [&](int32_t c0, int32_t c1, bool last, int64_t cnt, int32_t rank0) {
                    WinItem it;
                    it.c0 = c0;
                    it.c1 = c1;
                    it.last = last ? 1 : 0;
                    it.cnt = (int32_t)cnt;
                    it.out_base = out_off[i] + rank0;
                    it.t0 = a_ptr[i];
                    // k_win walks the row's heavy entry table (same A offset)
                    it.t_len = (saved && heavy_cnt) ? heavy_cnt[i] : (int32_t)(a_ptr[i + 1] - a_ptr[i]);
                    it.bm_word = saved ? bm_off[i] + ((int64_t)c0 - org) / 64 : -1;
                    it.rank0 = rank0;
                    const int cls = saved ? 2 : win_class(cnt, c0, c1);
                    const unsigned long long slot = atomicAdd(&cursor[cls * NBUCKET + win_bucket(c0, ncols)], 1ull);
                    work[slot] = it;
                  });
}

// B tile index: row-length histogram (log2 classes) to pick which rows get a
// table within the memory budget, then one warp per indexed row walks its
// columns once and records the tile boundaries.
__global__ void k_brow_hist(int64_t k, const int64_t* __restrict__ b_ptr, unsigned long long* __restrict__ hist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const int64_t len = b_ptr[i + 1] - b_ptr[i];
  if (len > 0) atomicAdd(&hist[63 - __clzll((unsigned long long)len)], 1ull);
}

__global__ void k_btile_flags(int64_t k, const int64_t* __restrict__ b_ptr, int64_t min_len, int64_t per_row,
                              int64_t* __restrict__ sizes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  sizes[i] = (b_ptr[i + 1] - b_ptr[i] >= min_len) ? per_row : 0;
}

__global__ void k_btile_build(int64_t k, const int64_t* __restrict__ b_ptr, const int32_t* __restrict__ b_col,
                              int64_t ntiles, const int64_t* __restrict__ tbl_scan, int64_t* __restrict__ tbl_off,
                              int32_t* __restrict__ tbl) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  if (row >= k) return;
  const bool has = tbl_scan[row + 1] > tbl_scan[row];
  if (lane == 0) tbl_off[row] = has ? tbl_scan[row] : -1;
  if (!has) return;
  int32_t* t = tbl + tbl_scan[row];
  const int64_t s = b_ptr[row], len = b_ptr[row + 1] - s;
  int prev = -1;  // tile of the previous element (warp-uniform after each step)
  for (int64_t j0 = 0; j0 < len; j0 += 32) {
    const int64_t j = j0 + lane;
    const int tj = j < len ? (int)(b_col[s + j] / TILE_COLS) : (int)ntiles;
    int tp = __shfl_up_sync(SG_FULL, tj, 1);
    if (lane == 0) tp = prev;
    // element j is the first column >= t*TILE_COLS for every t in (tp, tj]
    if (j < len)
      for (int x = tp + 1; x <= tj; ++x) t[x] = (int32_t)j;
    const int last_lane = (int)min((int64_t)31, len - 1 - j0);
    prev = __shfl_sync(SG_FULL, tj, last_lane);
  }
  // tiles after the row's last column point past the end
  if (prev < ntiles)
    for (int x = prev + 1 + lane; x <= ntiles; x += 32) t[x] = (int32_t)len;
}

__global__ void k_win_capacity(int64_t m, const int64_t* __restrict__ products, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ hi, const uint8_t* __restrict__ select,
                               int64_t* __restrict__ cap, int64_t* __restrict__ words) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t p = products[i];
  const int64_t span = hi[i] - lo[i] + 1;
  // symbolic pass: only rows the count classifier sends to a bitmap kernel;
  // fallback count pass (select given): every selected long row
  const bool sel = select == nullptr ? count_uses_bitmap(p, span) : (select[i] && p > 256);
  const bool thin = SG_SPARSE_WIN && select == nullptr && count_bitmap_sparse(p, span);  // windows, no words
  cap[i] = (sel || thin) ? window_capacity(p, span) : 0;
  if (words) words[i] = sel ? (hi[i] - win_origin(lo[i])) / 64 + 1 : 0;
}

// -------------------------------------------------------------------------
// classification

// bin ids shared by all modes
enum Bin : uint8_t {
  BIN_NONE = 0,
  BIN_ESC = 1,
  BIN_HW0 = 2,  // T = 32 << (bin - BIN_HW0), up to 2048 (bins 2..8)
  BIN_HB0 = 9,  // T = 4096 << (bin - BIN_HB0), up to 32768 (bins 9..12); numeric uses 2048..16384 via HB_N0
  BIN_BM0 = 13, // BW = 256, 2048, 16384 (bins 13..15)
  BIN_HBN = 16, // numeric HB T = 2048 (bin 16)
  BIN_ESCR = 17, // numeric register expand-sort-compress, <= 512 products, low CR (bin 17)
  NBINS = 18
};

__device__ __forceinline__ uint8_t bm_bin(int64_t span) {
  const int64_t words = (span + 63) / 64;
  if (words <= 256) return BIN_BM0;
  if (words <= 2048) return BIN_BM0 + 1;
  return BIN_BM0 + 2;
}

__device__ __forceinline__ int log2_pow2(int64_t t) { return 63 - __clzll((unsigned long long)t); }

__device__ __forceinline__ int64_t pow2_at_least(int64_t x) {
  return x <= 1 ? 1 : (int64_t)1 << (64 - __clzll((unsigned long long)(x - 1)));
}

// mode 0 (symbolic)
// Assisted symbolic binning: hash rows are sized by
// products / crc, crc the conservative sampled CR (predict.py:111-118),
// instead of by products; a row whose table fills is flagged (-1) by the count
// kernel and recounted with product sizing (rerun = 1 classifies only those).
__global__ void k_classify_count(int64_t m, const int64_t* __restrict__ products, const int64_t* __restrict__ lo,
                                 const int64_t* __restrict__ hi, uint8_t* __restrict__ bins,
                                 int64_t* __restrict__ counts, double crc, int rerun, int64_t skip_max) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t p = products[i];
  uint8_t b;
  if (rerun && counts[i] != -1) {
    b = BIN_NONE;
  } else if (!rerun && p > 0 && p <= skip_max && p <= 1024) {
    b = BIN_NONE;  // short row left to a staged numeric pass: -2 = not counted
    counts[i] = -2;
  } else if (p == 0) {
    b = BIN_NONE;
    counts[i] = 0;
  } else {
    const int64_t span = hi[i] - lo[i] + 1;
    const int64_t est = (crc > 1.0 && !rerun) ? max((int64_t)1, (int64_t)ceil((double)p / crc)) : p;
    const int64_t T = max(pow2_at_least(2 * est), (int64_t)32);
    if (count_uses_bitmap(p, span) || count_bitmap_sparse(p, span)) {
      b = bm_bin(span);
    } else if (est <= 1024) {
      b = (uint8_t)(BIN_HW0 + log2_pow2(T) - 5);
    } else {
      b = (uint8_t)(BIN_HB0 + log2_pow2(max(T, (int64_t)4096)) - 12);
    }
  }
  bins[i] = b;
}

__global__ void k_count_negative(int64_t m, const int64_t* __restrict__ counts, unsigned long long* __restrict__ n) {
  int c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    c += counts[i] == -1;
  c = __reduce_add_sync(SG_FULL, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(n, (unsigned long long)c);
}

// mode 1 (numeric phase)
__global__ void k_classify_numeric(int64_t m, const int8_t* __restrict__ kind, const int64_t* __restrict__ cap,
                                   const int64_t* __restrict__ alloc, const int64_t* __restrict__ products,
                                   const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                                   uint8_t* __restrict__ bins, int64_t* __restrict__ counts,
                                   uint8_t* __restrict__ overflow, const int32_t* __restrict__ nwin,
                                   const int64_t* __restrict__ exact, int64_t escr_max) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t p = products[i];
  const int8_t k = kind[i];
  uint8_t b;
  const int64_t ex = exact ? exact[i] : -1;
  // rows with numeric windows (exact counts known) go to the window kernel
  if (p == 0 || k == SG_KIND_FALLBACK || (nwin && nwin[i] > 0)) {
    b = BIN_NONE;
    counts[i] = 0;
    overflow[i] = 0;
  } else {
    const int64_t span = hi[i] - lo[i] + 1;
    const int64_t limit = row_limit(kind, cap, alloc, i);
    if (k == SG_KIND_ESC && p <= 64) {
      b = BIN_ESC;
    } else if (p <= escr_max && p <= ESCR_MAX && k != SG_KIND_DENSE && (limit == NOLIMIT || p <= limit)) {
      b = BIN_ESCR;  // holds every product: cannot overflow while p <= limit
    } else if (k == SG_KIND_DENSE) {
      b = bm_bin(span);
    } else if (ex >= 0 && limit != NOLIMIT && ex > limit) {
      // known overflow (exact count over the tier limit): rerun in fallback
      b = BIN_NONE;
      counts[i] = 0;
      overflow[i] = 1;
    } else {
      // with an exact count the table holds exactly those keys
      const int64_t need = ex >= 0 ? max(ex, (int64_t)1) : min(limit == NOLIMIT ? p : limit + 1, p);
      const int64_t T = max(pow2_at_least(2 * need), (int64_t)32);
      if (T <= 1024 && p <= 4096)
        b = (uint8_t)(BIN_HW0 + log2_pow2(T) - 5);
      else if (T <= 2048)
        b = BIN_HBN;
      else if (T <= 16384)
        b = (uint8_t)(BIN_HB0 + log2_pow2(T) - 12);
      else
        b = bm_bin(span);
    }
  }
  bins[i] = b;
}

// fallback rows: bitmap family by span
__global__ void k_classify_fallback(int64_t nrows, const int64_t* __restrict__ rows, const int64_t* __restrict__ lo,
                                    const int64_t* __restrict__ hi, uint8_t* __restrict__ bins) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int64_t r = rows[i];
  bins[i] = bm_bin(hi[r] - lo[r] + 1);
}

// -------------------------------------------------------------------------
// launch helpers

template <class K>
static int set_smem(K kern, size_t bytes) {
  // the 48 KB default limit counts static shared memory too (the product
  // iterator's group table and scratch): opt in well before it
  if (bytes > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return SG_ERR_CUDA;
    }
  }
  return SG_OK;
}

static int num_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return sms;
}

struct Launch {
  Csr A, B;
  const int8_t* kind;
  const int64_t* cap;
  const int64_t* alloc;
  const int64_t* lo;
  const int64_t* hi;
  const int64_t* out_off;
  int32_t* out_col;
  void* out_val;
  int64_t* counts;
  uint8_t* overflow;
  cudaStream_t s;
  Win win{nullptr, nullptr, nullptr, nullptr, nullptr};  // count mode: record numeric windows
  int64_t b_ncols = INT64_MAX;
};

template <int LOG2T, int MODE, typename V>
static int launch_hw(const Launch& L, const int32_t* rows, int64_t n) {
  constexpr size_t sm = hw_smem<LOG2T, MODE>();
  auto kern = k_hash_warp<LOG2T, MODE, V>;
  if (int rc = set_smem(kern, sm)) return rc;
  ktimer_begin(MODE == 0 ? "k_hash_warp:count" : "k_hash_warp", L.s);
  kern<<<grid_for(n, HW_WARPS), HW_WARPS * 32, sm, L.s>>>(n, rows, L.A, L.B, L.kind, L.cap, L.alloc, L.out_off,
                                                         L.out_col, (V*)L.out_val, L.counts, L.overflow, L.b_ncols);
  ktimer_end(L.s);
  return check_cuda("k_hash_warp");
}

template <int LOG2T, int MODE, typename V, int NT>
static int launch_hb(const Launch& L, const int32_t* rows, int64_t n) {
  constexpr size_t sm = hb_smem<LOG2T, MODE, NT>();
  auto kern = k_hash_block<LOG2T, MODE, V, NT>;
  if (int rc = set_smem(kern, sm)) return rc;
  int g = (int)std::min<int64_t>(n, (int64_t)num_sms() * 16);
  ktimer_begin(MODE == 0 ? "k_hash_block:count" : "k_hash_block", L.s);
  kern<<<g, NT, sm, L.s>>>(n, rows, L.A, L.B, L.kind, L.cap, L.alloc, L.lo, L.hi, L.out_off, L.out_col,
                           (V*)L.out_val, L.counts, L.overflow);
  ktimer_end(L.s);
  return check_cuda("k_hash_block");
}

template <int BW, int MODE, typename V, int NT>
static int launch_bm(const Launch& L, const int32_t* rows, int64_t n) {
  constexpr size_t sm = bm_smem<BW, MODE, NT>();
  auto kern = k_bitmap<BW, MODE, V, NT>;
  if (int rc = set_smem(kern, sm)) return rc;
  int g = (int)std::min<int64_t>(n, (int64_t)num_sms() * 32);
  ktimer_begin(MODE == 0 ? "k_bitmap:count" : "k_bitmap", L.s);
  kern<<<g, NT, sm, L.s>>>(n, rows, L.A, L.B, L.kind, L.cap, L.alloc, L.lo, L.hi, L.out_off, L.out_col,
                           (V*)L.out_val, L.counts, L.overflow,
                           MODE == 0 ? L.win : Win{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr});
  ktimer_end(L.s);
  return check_cuda("k_bitmap");
}

template <int MODE, typename V>
static int launch_bin(int bin, const Launch& L, const int32_t* rows, int64_t n) {
  if (n == 0) return SG_OK;
  switch (bin) {
    case BIN_ESC:
      if (MODE == 1) {
        k_esc<V><<<grid_for(n, ESC_WARPS), ESC_WARPS * 32, 0, L.s>>>(n, rows, L.A, L.B, L.out_off, L.out_col,
                                                                     (V*)L.out_val, L.counts, L.overflow);
        return check_cuda("k_esc");
      }
      return SG_ERR_ARG;
    case BIN_ESCR:
      if (MODE == 1) {
        constexpr size_t sm = escr_smem();
        auto kern = k_escr<V>;
        if (int rc = set_smem(kern, sm)) return rc;
        kern<<<grid_for(n, ESCR_WARPS), ESCR_WARPS * 32, sm, L.s>>>(n, rows, L.A, L.B, L.out_off, L.out_col,
                                                                    (V*)L.out_val, L.counts, L.overflow);
        return check_cuda("k_escr");
      }
      return SG_ERR_ARG;
    case BIN_HW0 + 0: return launch_hw<5, MODE, V>(L, rows, n);
    case BIN_HW0 + 1: return launch_hw<6, MODE, V>(L, rows, n);
    case BIN_HW0 + 2: return launch_hw<7, MODE, V>(L, rows, n);
    case BIN_HW0 + 3: return launch_hw<8, MODE, V>(L, rows, n);
    case BIN_HW0 + 4: return launch_hw<9, MODE, V>(L, rows, n);
    case BIN_HW0 + 5: return launch_hw<10, MODE, V>(L, rows, n);
    case BIN_HW0 + 6:
      if (MODE == 0) return launch_hw<11, 0, V>(L, rows, n);
      return SG_ERR_ARG;
    case BIN_HBN: return launch_hb<11, MODE, V, 256>(L, rows, n);
    case BIN_HB0 + 0: return launch_hb<12, MODE, V, 512>(L, rows, n);
    case BIN_HB0 + 1: return launch_hb<13, MODE, V, 512>(L, rows, n);
    case BIN_HB0 + 2:  // numeric T = 16384 fills the SM's shared memory: one CTA with every thread
      return MODE == 1 ? launch_hb<14, MODE, V, 1024>(L, rows, n) : launch_hb<14, MODE, V, 512>(L, rows, n);
    case BIN_HB0 + 3:
      if (MODE == 0) return launch_hb<15, 0, V, 1024>(L, rows, n);
      return SG_ERR_ARG;
    case BIN_BM0 + 0: return launch_bm<256, MODE, V, 256>(L, rows, n);
    case BIN_BM0 + 1: return launch_bm<2048, MODE, V, 256>(L, rows, n);
    case BIN_BM0 + 2: return launch_bm<16384, MODE, V, 1024>(L, rows, n);
  }
  set_error("launch_bin: unexpected bin " + std::to_string(bin));
  return SG_ERR_ARG;
}

// bins in launch order: heaviest families first so they start early
static const int kOrder[] = {BIN_BM0 + 2, BIN_HB0 + 3, BIN_HB0 + 2, BIN_HB0 + 1, BIN_HB0 + 0, BIN_BM0 + 1,
                             BIN_HBN,     BIN_BM0 + 0, BIN_HW0 + 6, BIN_HW0 + 5, BIN_HW0 + 4, BIN_HW0 + 3,
                             BIN_HW0 + 2, BIN_HW0 + 1, BIN_HW0 + 0, BIN_ESC, BIN_ESCR};

// Bins are independent: launch them on a few forked streams so the small
// bins fill the tail of the big ones, then join back into the caller's stream.
// Side streams for independent bin launches: created once per device and
// reused (stream creation per call costs tens of microseconds); each fork
// waits on the main stream and joins back with events.
struct Fork {
  static constexpr int N = 4;
  cudaStream_t main;
  cudaStream_t side[N];
  cudaEvent_t ev[N + 1];
  int used = 0;
  explicit Fork(cudaStream_t s) : main(s) {
    static std::mutex mu;
    static std::map<int, std::array<cudaStream_t, N>> streams;
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = streams.find(dev);
      if (it == streams.end()) {
        std::array<cudaStream_t, N> a;
        for (int i = 0; i < N; ++i) cudaStreamCreateWithFlags(&a[i], cudaStreamNonBlocking);
        it = streams.emplace(dev, a).first;
      }
      for (int i = 0; i < N; ++i) side[i] = it->second[i];
    }
    for (int i = 0; i <= N; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    cudaEventRecord(ev[N], s);
  }
  // the i-th launch's stream (the first waits for the main stream lazily)
  cudaStream_t at(int i) {
    const int k = i % N;
    if (k >= used) {
      cudaStreamWaitEvent(side[k], ev[N], 0);
      used = k + 1;
    }
    return side[k];
  }
  ~Fork() {
    for (int i = 0; i < used; ++i) {
      cudaEventRecord(ev[i], side[i]);
      cudaStreamWaitEvent(main, ev[i], 0);
    }
    for (int i = 0; i <= N; ++i) cudaEventDestroy(ev[i]);
  }
};

template <int MODE, typename V>
static int run_bins(const Launch& L, int64_t m, Workspace& w, const int32_t* rowmap_unused) {
  int64_t cnt[NBINS], off[NBINS + 1];
  if (int rc = partition_rows(m, NBINS, w, cnt, off, L.s)) return rc;
  if (getenv("SG_PRINT_BINS")) {  // analysis hook: rows per accumulator bin
    fprintf(stderr, "bins(mode %d):", MODE);
    for (int b = 0; b < NBINS; ++b)
      if (cnt[b]) fprintf(stderr, " %d:%lld", b, (long long)cnt[b]);
    fprintf(stderr, "\n");
  }
  int nonempty = 0;
  for (int b : kOrder) nonempty += cnt[b] != 0;
  Fork f(L.s);
  int k = 0;
  for (int b : kOrder) {
    if (cnt[b] == 0) continue;
    Launch Lb = L;
    Lb.s = nonempty > 1 ? f.at(k++) : L.s;
    if (int rc = launch_bin<MODE, V>(b, Lb, w.rowlist + off[b], cnt[b])) return rc;
  }
  return SG_OK;
}

// fallback rows are given as a list; map through it
__global__ void k_gather_rows(int64_t n, const int32_t* __restrict__ idx, const int64_t* __restrict__ rows,
                              int32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)rows[idx[i]];
}

}  // namespace sg

using namespace sg;

template <typename V, int NT, int WORDS, int R, int CTAS>
static int launch_bmr(int64_t n, const WinItem* work, const Csr& A, const Csr& B, const BTile& bt, const Win& W,
                      int32_t* out_col, void* out_val, unsigned long long* ticket, cudaStream_t s) {
  constexpr size_t sm = bmr_smem<NT, WORDS, R>();
  auto kern = k_bmr<V, NT, WORDS, R, CTAS>;
  if (int rc = set_smem(kern, sm)) return rc;
  const int grid = (int)std::min<int64_t>(n, (int64_t)num_sms() * CTAS);
  kern<<<grid, NT, sm, s>>>(n, work, A, B, bt, W.bm_save, W.pre_save, out_col, (V*)out_val, ticket);
  return check_cuda("k_bmr");
}

// B rows shorter than this go through k_win_light (0: every entry in k_win)
static int light_len() {
  static int v = [] {
    const char* e = getenv("SG_LIGHT_LEN");
    return e ? std::min(atoi(e), 256) : 0;  // k_win_light's table bound assumes < 256 products per entry
  }();
  return v;
}


// window scratch: WinItems, then the heavy and light entry tables (indexed by
// A position) and their per-row counts
struct WinScratch {
  WinItem* work;
  KwEnt* hent;
  KwEnt* lent;
  int32_t* hcnt;
  int32_t* lcnt;
};
static size_t win_scratch_bytes(int64_t m, int64_t nnz_a, int64_t nwin) {
  return align256((size_t)nwin * sizeof(WinItem)) + 2 * align256((size_t)nnz_a * sizeof(KwEnt)) +
         2 * align256((size_t)m * 4) + 256;
}
static WinScratch win_scratch(void* buf, int64_t m, int64_t nnz_a, int64_t nwin) {
  unsigned char* p = reinterpret_cast<unsigned char*>(((uintptr_t)buf + 255) & ~(uintptr_t)255);
  WinScratch w;
  w.work = reinterpret_cast<WinItem*>(p);
  p += align256((size_t)nwin * sizeof(WinItem));
  w.hent = reinterpret_cast<KwEnt*>(p);
  p += align256((size_t)nnz_a * sizeof(KwEnt));
  w.lent = reinterpret_cast<KwEnt*>(p);
  p += align256((size_t)nnz_a * sizeof(KwEnt));
  w.hcnt = reinterpret_cast<int32_t*>(p);
  p += align256((size_t)m * 4);
  w.lcnt = reinterpret_cast<int32_t*>(p);
  return w;
}

template <typename V>
static int launch_kwin(int64_t n, const WinItem* work, const Csr& A, const Csr& B, const BTile& bt, const Win& W,
                       const KwEnt* hent, int32_t* out_col, void* out_val, unsigned long long* ticket,
                       cudaStream_t s) {
  constexpr size_t sm = sizeof(KwShared);
  auto kern = k_win<V>;
  if (int rc = set_smem(kern, sm)) return rc;
  const int grid = (int)std::min<int64_t>(n, (int64_t)num_sms());
  kern<<<grid, KW_NT, sm, s>>>(n, work, A, B, bt, reinterpret_cast<const uint4*>(W.bm_save), hent, out_col,
                               (V*)out_val, ticket);
  return check_cuda("k_win");
}

template <typename V>
static int launch_light(int64_t m, const Csr& A, const Csr& B, const Win& W, const int64_t* span_lo,
                        const int64_t* row_ptr, const WinScratch& ws, void* out_val, cudaStream_t s) {
  constexpr int NT = KL_NT;
  constexpr size_t sm = (size_t)KL_T * 12;
  auto kern = k_win_light<V>;
  if (int rc = set_smem(kern, sm)) return rc;
  const int grid = (int)std::min<int64_t>(m, (int64_t)num_sms() * 2);
  ktimer_begin("k_win_light", s);
  kern<<<grid, NT, sm, s>>>(m, ws.lcnt, A, B, span_lo, W.bm_off, reinterpret_cast<const uint4*>(W.bm_save), row_ptr,
                            ws.lent, (V*)out_val);
  ktimer_end(s);
  return check_cuda("k_win_light");
}

extern "C" {

static Win to_win(const sg_windows_t* w) {
  if (!w) return Win{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const bool sv = w->bm_save != nullptr;  // 16-byte {lo, rank, hi, rank} words (pre_save unused)
  return Win{w->win_off, reinterpret_cast<int2*>(w->wins), w->nwin, w->bm_off,
             sv ? reinterpret_cast<unsigned long long*>(w->bm_save) : nullptr, sv ? w->pre_save : nullptr,
             w->btile_off, w->btile};
}

int sg_symbolic(int64_t m, int64_t b_ncols, const int64_t* a_ptr, const int32_t* a_col, const int64_t* b_ptr,
                const int32_t* b_col, const int64_t* products, const int64_t* span_lo, const int64_t* span_hi,
                int64_t* counts, const sg_windows_t* win, double assist_cr, int64_t skip_max_products, void* ws,
                size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, m, w)) return SG_ERR_WORKSPACE;
  if (m == 0) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const double crc = assist_cr > 1.0 ? assist_cr : 1.0;
  k_classify_count<<<grid_for(m, 256), 256, 0, s>>>(m, products, span_lo, span_hi, w.bins, counts, crc, 0,
                                                    skip_max_products);
  if (int rc = check_cuda("k_classify_count")) return rc;
  Launch L{{a_ptr, a_col, nullptr}, {b_ptr, b_col, nullptr}, nullptr, nullptr, nullptr, span_lo, span_hi,
           nullptr, nullptr, nullptr, counts, nullptr, s};
  L.win = to_win(win);
  L.b_ncols = b_ncols;
  if (int rc = run_bins<0, double>(L, m, w, nullptr)) return rc;
  if (crc == 1.0) return SG_OK;
  // recount the rows whose assisted table filled up, with product sizing
  unsigned long long* nneg = reinterpret_cast<unsigned long long*>(w.bincnt) + 120;
  cudaMemsetAsync(nneg, 0, sizeof(unsigned long long), s);
  k_count_negative<<<std::min(grid_for(m, 256), num_sms() * 8), 256, 0, s>>>(m, counts, nneg);
  if (int rc = check_cuda("k_count_negative")) return rc;
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, nneg, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_symbolic sync", 0);
  if (h == 0) return SG_OK;
  k_classify_count<<<grid_for(m, 256), 256, 0, s>>>(m, products, span_lo, span_hi, w.bins, counts, 1.0, 1, 0);
  if (int rc = check_cuda("k_classify_count")) return rc;
  L.win = Win{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // bitmap rows are done
  return run_bins<0, double>(L, m, w, nullptr);
}

int sg_numeric(int64_t m, int64_t b_ncols, int dtype, const int64_t* a_ptr, const int32_t* a_col,
               const void* a_val, const int64_t* b_ptr, const int32_t* b_col, const void* b_val,
               const int8_t* kind, const int64_t* cap, const int64_t* alloc, const int64_t* products,
               const int64_t* span_lo, const int64_t* span_hi, const int64_t* out_off, int32_t* out_col,
               void* out_val, int64_t* counts, uint8_t* overflow, const int32_t* skip_nwin,
               const int64_t* exact, int64_t escr_max, void* ws, size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, m, w)) return SG_ERR_WORKSPACE;
  if (m == 0) return SG_OK;
  (void)b_ncols;
  cudaStream_t s = (cudaStream_t)stream;
  k_classify_numeric<<<grid_for(m, 256), 256, 0, s>>>(m, kind, cap, alloc, products, span_lo, span_hi, w.bins,
                                                      counts, overflow, skip_nwin, exact,
                                                      b_ncols < ((int64_t)1 << 23) ? escr_max : 0);
  if (int rc = check_cuda("k_classify_numeric")) return rc;
  Launch L{{a_ptr, a_col, a_val}, {b_ptr, b_col, b_val}, kind, cap, alloc, span_lo, span_hi,
           out_off, out_col, out_val, counts, overflow, s};
  L.b_ncols = b_ncols;
  if (dtype == SG_F64) return run_bins<1, double>(L, m, w, nullptr);
  if (dtype == SG_F32) return run_bins<1, float>(L, m, w, nullptr);
  set_error("sg_numeric: bad dtype");
  return SG_ERR_ARG;
}

int sg_fallback(int mode, int64_t nrows, const int64_t* rows, int64_t b_ncols, int dtype, const int64_t* a_ptr,
                const int32_t* a_col, const void* a_val, const int64_t* b_ptr, const int32_t* b_col,
                const void* b_val, const int64_t* products, const int64_t* span_lo, const int64_t* span_hi,
                const int64_t* out_off, int32_t* out_col, void* out_val, int64_t* counts,
                const sg_windows_t* win, void* ws, size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, nrows, w)) return SG_ERR_WORKSPACE;
  if (nrows == 0) return SG_OK;
  (void)products;
  cudaStream_t s = (cudaStream_t)stream;
  k_classify_fallback<<<grid_for(nrows, 256), 256, 0, s>>>(nrows, rows, span_lo, span_hi, w.bins);
  if (int rc = check_cuda("k_classify_fallback")) return rc;
  int64_t cnt[NBINS], off[NBINS + 1];
  if (int rc = partition_rows(nrows, NBINS, w, cnt, off, s)) return rc;
  // rowlist holds indices into `rows`; translate to row ids in place via tmp
  int32_t* mapped = reinterpret_cast<int32_t*>(w.tmp);
  k_gather_rows<<<grid_for(nrows, 256), 256, 0, s>>>(nrows, w.rowlist, rows, mapped);
  if (int rc = check_cuda("k_gather_rows")) return rc;
  Launch L{{a_ptr, a_col, a_val}, {b_ptr, b_col, b_val}, nullptr, nullptr, nullptr, span_lo, span_hi,
           out_off, out_col, out_val, counts, nullptr, s};
  L.b_ncols = b_ncols;
  if (mode == 0) L.win = to_win(win);
  if (getenv("SG_PRINT_BINS")) {  // analysis hook: rows per accumulator bin
    fprintf(stderr, "fallback bins(mode %d):", mode);
    for (int b = 0; b < NBINS; ++b)
      if (cnt[b]) fprintf(stderr, " %d:%lld", b, (long long)cnt[b]);
    fprintf(stderr, "\n");
  }
  int nonempty = 0;
  for (int b : kOrder) nonempty += cnt[b] != 0;
  Fork f(s);
  int kk = 0;
  for (int b : kOrder) {
    if (cnt[b] == 0) continue;
    Launch Lb = L;
    Lb.s = nonempty > 1 ? f.at(kk++) : s;
    int rc;
    if (mode == 0)
      rc = launch_bin<0, double>(b, Lb, mapped + off[b], cnt[b]);
    else if (dtype == SG_F64)
      rc = launch_bin<1, double>(b, Lb, mapped + off[b], cnt[b]);
    else
      rc = launch_bin<1, float>(b, Lb, mapped + off[b], cnt[b]);
    if (rc) return rc;
  }
  return SG_OK;
}

int sg_window_capacity(int64_t m, const int64_t* products, const int64_t* span_lo, const int64_t* span_hi,
                       const uint8_t* select, int64_t* win_off, int64_t* bm_off, int64_t* totals_host, void* ws,
                       size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, m, w)) return SG_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  // capacities into win_off[0..m) and word counts into bm_off[0..m), then
  // both are scanned in place (the scan reads each tile before writing it)
  if (m > 0) {
    k_win_capacity<<<grid_for(m, 256), 256, 0, s>>>(m, products, span_lo, span_hi, select, win_off, bm_off);
    if (int rc = check_cuda("k_win_capacity")) return rc;
  }
  if (int rc = scan_i64(m, win_off, win_off, w.partials, s)) return rc;
  if (bm_off)
    if (int rc = scan_i64(m, bm_off, bm_off, w.partials, s)) return rc;
  cudaMemcpyAsync(totals_host, win_off + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (bm_off) cudaMemcpyAsync(totals_host + 1, bm_off + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_window_capacity sync", 0);
  if (!bm_off) totals_host[1] = 0;
  return SG_OK;
}

int sg_window_numeric(int64_t m, int64_t b_ncols, int dtype, const int64_t* a_ptr, const int32_t* a_col,
                      const void* a_val, const int64_t* b_ptr, const int32_t* b_col, const void* b_val,
                      const int64_t* span_lo, const int64_t* span_hi, const sg_windows_t* win,
                      const int64_t* out_off, int32_t* out_col, void* out_val, void* work_buf, int64_t work_cap,
                      void* ws, size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, m, w)) return SG_ERR_WORKSPACE;
  if (m == 0 || win == nullptr) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const Win W = to_win(win);
  // (class, bucket) histogram -> exclusive offsets -> cursors.  Work array:
  // [k_bmr small class | k_bmr large class | saved words (k_win)]
  constexpr int NCLS = 3;
  const int64_t* bm_off = W.bm_save ? W.bm_off : nullptr;
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(w.bincnt);
  cudaMemsetAsync(cnt, 0, NCLS * NBUCKET * sizeof(unsigned long long), s);
  k_win_counts<<<grid_for(m, 256), 256, 0, s>>>(m, b_ncols, W.off, W.wins, W.nwin, span_hi, out_off, bm_off, cnt);
  if (int rc = check_cuda("k_win_counts")) return rc;
  unsigned long long h[NCLS * NBUCKET];
  cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_window_numeric sync", 0);
  int64_t nwork = 0, nsmall = 0, nrebuild = 0;
  unsigned long long cur[NCLS * NBUCKET];
  for (int c : {1, 0, 2}) {
    for (int i = 0; i < NBUCKET; ++i) {
      cur[c * NBUCKET + i] = (unsigned long long)nwork;
      nwork += (int64_t)h[c * NBUCKET + i];
    }
    if (c == 1) nsmall = nwork;
    if (c == 0) nrebuild = nwork;
  }
  if (nwork == 0) return SG_OK;
  int64_t nnz_a = 0;
  cudaMemcpyAsync(&nnz_a, a_ptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_window_numeric nnz", 0);
  if (win_scratch_bytes(m, nnz_a, nwork) > (size_t)work_cap) {
    set_error("sg_window_numeric: work buffer too small (sg_window_work_bytes)");
    return SG_ERR_WORKSPACE;
  }
  const WinScratch wsc = win_scratch(work_buf, m, nnz_a, nwork);
  WinItem* work = wsc.work;
  const Csr A{a_ptr, a_col, a_val}, B{b_ptr, b_col, b_val};
  const BTile bt{W.btile_off, W.btile};
  const int lh = W.bm_save ? light_len() : 0;
  if (W.bm_save) {
    // heavy / light entry tables of the windowed rows (k_win, k_win_light)
    auto ek = dtype == SG_F64 ? k_win_entries<double, 256> : k_win_entries<float, 256>;
    ek<<<(int)std::min<int64_t>(m, (int64_t)num_sms() * 16), 256, 0, s>>>(m, W.nwin, A, b_ptr, bt, lh, wsc.hent,
                                                                           wsc.hcnt, wsc.lent, wsc.lcnt);
    if (int rc = check_cuda("k_win_entries")) return rc;
  }
  cudaMemcpyAsync(cnt, cur, sizeof(cur), cudaMemcpyHostToDevice, s);
  k_win_scatter<<<grid_for(m, 256), 256, 0, s>>>(m, b_ncols, a_ptr, span_lo, span_hi, W.off, W.wins, W.nwin,
                                                 out_off, bm_off, W.bm_save ? wsc.hcnt : nullptr, cnt, work);
  if (int rc = check_cuda("k_win_scatter")) return rc;
  if (const char* dump = getenv("SG_DUMP_WINDOWS")) {
    // analysis hook: the window work items as raw 48-byte records
    std::vector<WinItem> hw((size_t)nwork);
    cudaMemcpyAsync(hw.data(), work, (size_t)nwork * sizeof(WinItem), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (FILE* f = fopen(dump, "wb")) {
      fwrite(hw.data(), sizeof(WinItem), hw.size(), f);
      fclose(f);
    }
  }
  // tickets live after the cursors (the host copy above must finish first)
  unsigned long long* tickets = cnt + NCLS * NBUCKET;
  cudaMemsetAsync(tickets, 0, 3 * sizeof(unsigned long long), s);
  if (nwork > nrebuild) {
    // saved words: the warp-specialised window kernel, heavy entries only
    ktimer_begin("k_win", s);
    int rc = dtype == SG_F64 ? launch_kwin<double>(nwork - nrebuild, work + nrebuild, A, B, bt, W, wsc.hent, out_col,
                                                   out_val, tickets, s)
                             : launch_kwin<float>(nwork - nrebuild, work + nrebuild, A, B, bt, W, wsc.hent, out_col,
                                                  out_val, tickets, s);
    if (rc) return rc;
    ktimer_end(s);
    // then the light entries add on top of the stored window values
    if (lh > 1) {
      rc = dtype == SG_F64 ? launch_light<double>(m, A, B, W, span_lo, out_off, wsc, out_val, s)
                           : launch_light<float>(m, A, B, W, span_lo, out_off, wsc, out_val, s);
      if (rc) return rc;
    }
  }
  // windows without saved words (no room for them, or thin rows): k_bmr
  // rebuilds their keys
  if (nrebuild > 0) ktimer_begin("k_bmr", s);
  if (nsmall > 0) {
    int rc = dtype == SG_F64
                 ? launch_bmr<double, SMALL_NT, SMALL_WORDS, SMALL_R, 2>(nsmall, work, A, B, bt, W, out_col, out_val,
                                                                           tickets + 1, s)
                 : launch_bmr<float, SMALL_NT, SMALL_WORDS, SMALL_R, 2>(nsmall, work, A, B, bt, W, out_col, out_val,
                                                                          tickets + 1, s);
    if (rc) return rc;
  }
  if (nrebuild > nsmall) {
    int rc = dtype == SG_F64 ? launch_bmr<double, WIN_NT, WIN_WORDS, WIN_R, 1>(nrebuild - nsmall, work + nsmall, A, B,
                                                                                bt, W, out_col, out_val, tickets + 2, s)
                             : launch_bmr<float, WIN_NT, WIN_WORDS, WIN_R, 1>(nrebuild - nsmall, work + nsmall, A, B,
                                                                               bt, W, out_col, out_val, tickets + 2, s);
    if (rc) return rc;
  }
  if (nrebuild > 0) ktimer_end(s);
  // `cur` (host) is read by the async copy above: keep it alive until done
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_window_numeric end", 0);
  return SG_OK;
}

int64_t sg_window_work_bytes(int64_t m, int64_t nnz_a, int64_t nwindows) {
  return (int64_t)win_scratch_bytes(m, nnz_a, nwindows);
}

int sg_btile_plan(int64_t k, int64_t b_ncols, const int64_t* b_ptr, int64_t budget_bytes, int64_t* tbl_scan,
                  int64_t* totals_host, void* ws, size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, k, w)) return SG_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ntiles = (b_ncols + TILE_COLS - 1) / TILE_COLS;
  const int64_t per_row = ntiles + 1;
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(w.bincnt);
  cudaMemsetAsync(hist, 0, 64 * sizeof(unsigned long long), s);
  if (k > 0) {
    k_brow_hist<<<grid_for(k, 256), 256, 0, s>>>(k, b_ptr, hist);
    if (int rc = check_cuda("k_brow_hist")) return rc;
  }
  unsigned long long hh[64];
  cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_btile_plan sync", 0);
  // smallest power-of-two length class whose rows (and all longer ones) fit the budget
  int cls = 63;
  int64_t rows = 0;
  for (int c = 63; c >= 0; --c) {  // down to single-entry rows while the budget lasts
    if ((rows + (int64_t)hh[c]) * per_row * 4 > budget_bytes) break;
    rows += (int64_t)hh[c];
    cls = c;
  }
  const int64_t min_len = (int64_t)1 << cls;
  if (k > 0) {
    k_btile_flags<<<grid_for(k, 256), 256, 0, s>>>(k, b_ptr, rows ? min_len : INT64_MAX, per_row, tbl_scan);
    if (int rc = check_cuda("k_btile_flags")) return rc;
  }
  if (int rc = scan_i64(k, tbl_scan, tbl_scan, w.partials, s)) return rc;
  cudaMemcpyAsync(totals_host, tbl_scan + k, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_btile_plan end", 0);
  totals_host[1] = rows ? min_len : -1;
  return SG_OK;
}

int sg_btile_build(int64_t k, int64_t b_ncols, const int64_t* b_ptr, const int32_t* b_col, const int64_t* tbl_scan,
                   int64_t* tbl_off, int32_t* tbl, void* stream) {
  if (k == 0) return SG_OK;
  const int64_t ntiles = (b_ncols + TILE_COLS - 1) / TILE_COLS;
  k_btile_build<<<grid_for(k * 32, 256), 256, 0, (cudaStream_t)stream>>>(k, b_ptr, b_col, ntiles, tbl_scan,
                                                                         tbl_off, tbl);
  return check_cuda("k_btile_build");
}

#ifdef SG_PROF
int sg_debug_kw_cycles(unsigned long long* out16) {
  cudaMemcpyFromSymbol(out16, g_kw, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_kw, z, sizeof(z));
  return check_cuda("sg_debug_kw_cycles", 0);
}

int sg_debug_phase_cycles(unsigned long long* out12) {
  cudaMemcpyFromSymbol(out12, g_phase, sizeof(unsigned long long) * 12);
  unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  return check_cuda("sg_debug_phase_cycles", 0);
}
#endif

}  // extern "C"
