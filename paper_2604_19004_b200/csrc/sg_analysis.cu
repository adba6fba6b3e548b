// sg_analysis.cu — analysis, sketching, planning, scan, selection, compaction.
//
// Stage kernels of the estimation-based SpGEMM that are not accumulators:
//   row statistics      analysis.py:96-128
//   HLL sketch build    analysis.py:131-146, hll.py:34-76
//   HLL merge+estimate  analysis.py:149-169, predict.py:87-103, hll.py:79-86
//   row planning        accumulate.py:104-181
//   prefix sums         engine.py:256-258, 349-350
//   fallback selection  engine.py:202-203
//   compaction          engine.py:346-368
// All are HBM-bound integer/byte work: coalesced loads, warp/sub-warp per row,
// grids sized by rows.
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "sg_internal.cuh"

namespace sg {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
static std::atomic<unsigned long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

struct KTimed {
  std::string name;
  cudaEvent_t a, b;
};
static std::mutex g_kt_mu;
static std::atomic<bool> g_kt_on{false};
static std::vector<KTimed> g_kt;
static thread_local int g_kt_open = -1;

bool ktimer_on() { return g_kt_on.load(std::memory_order_relaxed); }

void ktimer_begin(const char* name, cudaStream_t s) {
  if (!ktimer_on()) return;
  KTimed t{name, nullptr, nullptr};
  cudaEventCreate(&t.a);
  cudaEventCreate(&t.b);
  cudaEventRecord(t.a, s);
  std::lock_guard<std::mutex> g(g_kt_mu);
  g_kt_open = (int)g_kt.size();
  g_kt.push_back(t);
}

void ktimer_end(cudaStream_t s) {
  if (!ktimer_on() || g_kt_open < 0) return;
  std::lock_guard<std::mutex> g(g_kt_mu);
  cudaEventRecord(g_kt[g_kt_open].b, s);
  g_kt_open = -1;
}

static void ktimer_clear() {
  std::lock_guard<std::mutex> g(g_kt_mu);
  for (auto& t : g_kt) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  g_kt.clear();
}

// ---------------------------------------------------------------------------
// row statistics: G lanes per A row

// A rows longer than RS_LONG entries (R-MAT hub rows: tens of thousands)
// take a whole block each instead of G lanes: blocks sweep the rows 256 at a
// time, collect the long ones and reduce each with all their threads.
constexpr int64_t RS_LONG = 512;
constexpr int RS_NT = 256;

__global__ void __launch_bounds__(RS_NT) k_row_stats_long(int64_t m, int64_t b_ncols,
                                                          const int64_t* __restrict__ a_ptr,
                                                          const int32_t* __restrict__ a_col,
                                                          const int64_t* __restrict__ b_ptr,
                                                          const int32_t* __restrict__ b_col,
                                                          int64_t* __restrict__ products,
                                                          int64_t* __restrict__ span_lo,
                                                          int64_t* __restrict__ span_hi,
                                                          unsigned long long* __restrict__ totals) {
  __shared__ int64_t list[RS_NT];
  __shared__ int nlist;
  __shared__ int64_t red[3][RS_NT / 32];
  const int w = threadIdx.x >> 5, lane = lane_id();
  for (int64_t base = (int64_t)blockIdx.x * RS_NT; base < m; base += (int64_t)gridDim.x * RS_NT) {
    if (threadIdx.x == 0) nlist = 0;
    __syncthreads();
    const int64_t r = base + threadIdx.x;
    if (r < m && a_ptr[r + 1] - a_ptr[r] > RS_LONG) list[atomicAdd(&nlist, 1)] = r;
    __syncthreads();
    const int n = nlist;
    __syncthreads();  // (nlist is reset by the next sweep step)
    for (int i = 0; i < n; ++i) {
      const int64_t row = list[i];
      int64_t prod = 0, lo = b_ncols, hi = -1;
      const int64_t e = a_ptr[row + 1];
      for (int64_t t = a_ptr[row] + threadIdx.x; t < e; t += RS_NT) {
        const int32_t k = a_col[t];
        const int64_t bs = b_ptr[k], be = b_ptr[k + 1];
        if (be > bs) {
          prod += be - bs;
          lo = min(lo, (int64_t)b_col[bs]);
          hi = max(hi, (int64_t)b_col[be - 1]);
        }
      }
      prod = warp_sum(prod);
      lo = warp_min(lo);
      hi = warp_max(hi);
      if (lane == 0) {
        red[0][w] = prod;
        red[1][w] = lo;
        red[2][w] = hi;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int j = 1; j < RS_NT / 32; ++j) {
          prod += red[0][j];
          lo = min(lo, red[1][j]);
          hi = max(hi, red[2][j]);
        }
        products[row] = prod;
        span_lo[row] = prod ? lo : b_ncols;
        span_hi[row] = prod ? hi : -1;
        if (prod) {
          atomicAdd(&totals[0], (unsigned long long)prod);
          atomicMax(&totals[1], (unsigned long long)prod);
        }
      }
      __syncthreads();
    }
  }
}

template <int G>
__global__ void __launch_bounds__(256) k_row_stats(int64_t m, int64_t b_ncols,
                                                   const int64_t* __restrict__ a_ptr,
                                                   const int32_t* __restrict__ a_col,
                                                   const int64_t* __restrict__ b_ptr,
                                                   const int32_t* __restrict__ b_col,
                                                   int64_t* __restrict__ products,
                                                   int64_t* __restrict__ span_lo,
                                                   int64_t* __restrict__ span_hi,
                                                   unsigned long long* __restrict__ totals) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / G;
  const int sub = (int)(gid % G);
  int64_t prod = 0, lo = b_ncols, hi = -1;
  bool mine_row = row < m;
  if (mine_row) {
    const int64_t e = a_ptr[row + 1];
    mine_row = e - a_ptr[row] <= RS_LONG;  // long rows: k_row_stats_long
  }
  if (mine_row) {
    const int64_t e = a_ptr[row + 1];
    for (int64_t t = a_ptr[row] + sub; t < e; t += G) {
      const int32_t k = a_col[t];
      const int64_t bs = b_ptr[k], be = b_ptr[k + 1];
      if (be > bs) {
        prod += be - bs;
        lo = min(lo, (int64_t)b_col[bs]);
        hi = max(hi, (int64_t)b_col[be - 1]);
      }
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    prod += __shfl_xor_sync(SG_FULL, prod, o, G);
    lo = min(lo, (int64_t)__shfl_xor_sync(SG_FULL, lo, o, G));
    hi = max(hi, (int64_t)__shfl_xor_sync(SG_FULL, hi, o, G));
  }
  if (mine_row && sub == 0) {
    products[row] = prod;
    span_lo[row] = prod ? lo : b_ncols;
    span_hi[row] = prod ? hi : -1;
  }
  // block partials -> one atomic per warp
  int64_t mine = (mine_row && sub == 0) ? prod : 0;
  int64_t s = warp_sum(mine);
  int64_t mx = warp_max(mine);
  if (lane_id() == 0) {
    if (s) atomicAdd(&totals[0], (unsigned long long)s);
    if (mx) atomicMax(&totals[1], (unsigned long long)mx);
  }
}

// ---------------------------------------------------------------------------
// HLL: one warp per B row, registers in shared memory (ATOMS.MAX)

constexpr int HLL_WARPS = 8;

__global__ void __launch_bounds__(HLL_WARPS * 32) k_hll_build(int64_t k, const int64_t* __restrict__ b_ptr,
                                                              const int32_t* __restrict__ b_col, int p,
                                                              uint8_t* __restrict__ regs) {
  __shared__ uint32_t r[HLL_WARPS][128];
  const int w = warp_id(), lane = lane_id();
  const int m = 1 << p;
  const int64_t row = (int64_t)blockIdx.x * HLL_WARPS + w;
  if (row >= k) return;
  for (int i = lane; i < m; i += 32) r[w][i] = 0;
  __syncwarp();
  const int64_t e = b_ptr[row + 1];
  for (int64_t j = b_ptr[row] + lane; j < e; j += 32) {
    uint32_t idx, rank;
    hll_index_rank((uint32_t)b_col[j], p, idx, rank);
    atomicMax(&r[w][idx], rank);
  }
  __syncwarp();
  uint8_t* out = regs + row * m;
  for (int i = lane; i < m; i += 32) out[i] = (uint8_t)r[w][i];
}

// merge + estimate: one warp per selected A row; lane l owns registers
// [l*R, l*R+R) with R = m/32.
template <int R>
__global__ void __launch_bounds__(256) k_hll_estimate(int64_t nsel, const int64_t* __restrict__ rows,
                                                      const int64_t* __restrict__ a_ptr,
                                                      const int32_t* __restrict__ a_col,
                                                      const uint8_t* __restrict__ regs,
                                                      const double* __restrict__ lin, double alpha_mm,
                                                      double* __restrict__ est) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  if (wid >= nsel) return;
  const int64_t row = rows ? rows[wid] : wid;
  const int64_t s = a_ptr[row], e = a_ptr[row + 1];
  if (e == s) {
    if (lane == 0) est[wid] = 0.0;
    return;
  }
  constexpr int M = 32 * R;
  uint32_t mx[R];
#pragma unroll
  for (int i = 0; i < R; ++i) mx[i] = 0;
  for (int64_t t = s; t < e; ++t) {
    const uint8_t* sk = regs + (int64_t)a_col[t] * M + lane * R;
    if (R == 1) {
      mx[0] = max(mx[0], (uint32_t)sk[0]);
    } else if (R == 2) {
      uint16_t v = *reinterpret_cast<const uint16_t*>(sk);
      mx[0] = max(mx[0], (uint32_t)(v & 0xff));
      mx[R - 1] = max(mx[R - 1], (uint32_t)(v >> 8));
    } else {
      uint32_t v = *reinterpret_cast<const uint32_t*>(sk);
#pragma unroll
      for (int i = 0; i < R; ++i) mx[i] = max(mx[i], (v >> (8 * i)) & 0xff);
    }
  }
  double sum = 0.0;
  int zeros = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    sum += ldexp(1.0, -(int)mx[i]);
    zeros += mx[i] == 0;
  }
  // all terms are dyadic with rank <= 46 in practice, so the sum is exact and
  // order-independent (bit-identical to numpy's sum)
  sum = warp_sum(sum);
  zeros = warp_sum(zeros);
  if (lane == 0) {
    const double raw = alpha_mm / sum;
    est[wid] = (raw <= 2.5 * M && zeros > 0) ? lin[zeros] : raw;
  }
}

// ---------------------------------------------------------------------------
// plan_rows: thread per row, identical integer rules

__device__ __forceinline__ int search_left(const int64_t* a, int n, int64_t v) {
  int j = 0;
  while (j < n && a[j] < v) ++j;
  return j;
}

__global__ void k_plan(int64_t m, int pred_kind, const void* __restrict__ pred,
                       const int64_t* __restrict__ products, const int64_t* __restrict__ span_lo,
                       const int64_t* __restrict__ span_hi, sg_tiers_t t, int8_t* __restrict__ kind,
                       int64_t* __restrict__ cap, int64_t* __restrict__ alloc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t prod = products[i];
  const bool live = prod > 0;
  int64_t target;
  if (pred_kind == SG_PRED_UPPER) {
    target = prod;
  } else if (pred_kind == SG_PRED_EXACT) {
    target = (int64_t)ceil((double)((const int64_t*)pred)[i] * t.coef);
  } else {
    target = (int64_t)ceil(((const double*)pred)[i] * t.coef);
  }
  target = max(target, (int64_t)1);
  const int64_t span = live ? span_hi[i] - span_lo[i] + 1 : 0;
  const int64_t BIG = 0x7fffffffffffffffll;
  const int nh = t.n_hash, nd = t.n_dense;
  const int hj = search_left(t.hash_caps, nh, target);
  const bool hfit = hj < nh;
  const bool efit = target <= t.enh_cap;
  const int64_t hrank = hfit ? hj : (efit ? nh - 1 : BIG);
  const bool is_enh = !hfit && efit;
  const bool have_h = hfit || efit;
  const int dj = search_left(t.dense_spans, nd, span);
  const bool dfit = (dj < nd) && live;
  const int64_t drank = dfit ? dj : BIG;
  const bool use_d = dfit && (!have_h || drank < hrank || (drank == hrank && !is_enh));
  const bool use_h = live && !use_d && have_h;
  const bool use_f = live && !use_d && !use_h;
  int8_t kd = SG_KIND_HASH;
  int64_t cp = 0, al = 0;
  if (use_h) {
    kd = is_enh ? SG_KIND_ENHANCED_HASH : SG_KIND_HASH;
    cp = is_enh ? t.enh_cap : t.hash_caps[min(hj, nh - 1)];
  } else if (use_d) {
    kd = SG_KIND_DENSE;
    cp = t.dense_spans[min(dj, nd - 1)];
  } else if (use_f) {
    kd = SG_KIND_FALLBACK;
  }
  if (pred_kind == SG_PRED_UPPER) {
    if (live && prod < t.esc_max) {
      kd = SG_KIND_ESC;
      cp = prod;
    }
    al = live ? prod : 0;
  } else if (pred_kind == SG_PRED_EXACT) {
    if (live) al = ((const int64_t*)pred)[i];
    if (use_f) al = prod;
  } else {
    if (use_h) al = cp;
    if (use_d) {
      const int lg = target <= 1 ? 0 : 64 - __clzll((unsigned long long)(target - 1));
      const int64_t p2 = (int64_t)1 << lg;
      al = min(cp, max(p2, t.hash_caps[0]));
    }
    if (use_f) al = prod;
  }
  if (!live) {
    kd = SG_KIND_HASH;
    cp = t.hash_caps[0];
    al = 0;
  }
  kind[i] = kd;
  cap[i] = cp;
  alloc[i] = al;
}

// ---------------------------------------------------------------------------
// exclusive scan (int64), 4096-element tiles, three kernels

constexpr int SCAN_T = 1024, SCAN_IPT = 4;

__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(int64_t n, const int64_t* __restrict__ in,
                                                        int64_t* __restrict__ partials) {
  __shared__ int64_t sc[SCAN_T / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_IPT;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    int64_t j = base + (int64_t)i * SCAN_T + threadIdx.x;
    if (j < n) s += in[j];
  }
  s = warp_sum(s);
  if (lane_id() == 0) sc[warp_id()] = s;
  __syncthreads();
  if (warp_id() == 0) {
    int64_t v = lane_id() < SCAN_T / 32 ? sc[lane_id()] : 0;
    v = warp_sum(v);
    if (lane_id() == 0) partials[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(SCAN_T) k_scan_partials(int64_t nb, int64_t* __restrict__ partials) {
  __shared__ int64_t sc[SCAN_T / 32 + 1];
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += SCAN_T) {
    int64_t j = b0 + threadIdx.x;
    int64_t v = j < nb ? partials[j] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan(v, sc, &tot);
    if (j < nb) partials[j] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) partials[nb] = carry;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_down(int64_t n, const int64_t* __restrict__ in,
                                                      int64_t* __restrict__ out,
                                                      const int64_t* __restrict__ partials) {
  __shared__ int64_t sc[SCAN_T / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_IPT + (int64_t)threadIdx.x * SCAN_IPT;
  int64_t v[SCAN_IPT];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    s += v[i];
  }
  int64_t ex = block_excl_scan(s, sc, (int64_t*)nullptr) + partials[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = partials[gridDim.x];
}

int scan_i64(int64_t n, const int64_t* in, int64_t* out, int64_t* partials, cudaStream_t s) {
  if (n == 0) {
    cudaMemsetAsync(out, 0, sizeof(int64_t), s);
    return check_cuda("scan(n=0)", 0);
  }
  const int64_t nb = (n + SCAN_T * SCAN_IPT - 1) / (SCAN_T * SCAN_IPT);
  k_scan_reduce<<<(unsigned)nb, SCAN_T, 0, s>>>(n, in, partials);
  k_scan_partials<<<1, SCAN_T, 0, s>>>(nb, partials);
  k_scan_down<<<(unsigned)nb, SCAN_T, 0, s>>>(n, in, out, partials);
  return check_cuda("scan", 3);
}

// ---------------------------------------------------------------------------
// bin partition: block-aggregated histogram + scatter

constexpr int PART_T = 256;

__global__ void __launch_bounds__(PART_T) k_bin_hist(int64_t m, int nbins, const uint8_t* __restrict__ bins,
                                                     unsigned long long* __restrict__ cnt) {
  __shared__ unsigned int h[64];
  for (int i = threadIdx.x; i < nbins; i += PART_T) h[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * PART_T + threadIdx.x; i < m; i += (int64_t)gridDim.x * PART_T)
    atomicAdd(&h[bins[i]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < nbins; i += PART_T)
    if (h[i]) atomicAdd(&cnt[i], (unsigned long long)h[i]);
}

__global__ void __launch_bounds__(PART_T) k_bin_scatter(int64_t m, int nbins, const uint8_t* __restrict__ bins,
                                                        unsigned long long* __restrict__ cursor,
                                                        int32_t* __restrict__ rowlist) {
  __shared__ unsigned int h[64];
  __shared__ unsigned long long base[64];
  const int64_t chunk0 = (int64_t)blockIdx.x * PART_T * 16;
  for (int i = threadIdx.x; i < nbins; i += PART_T) h[i] = 0;
  __syncthreads();
  unsigned int rank[16];
  uint8_t bv[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    int64_t i = chunk0 + (int64_t)r * PART_T + threadIdx.x;
    bv[r] = i < m ? bins[i] : 0xff;
    rank[r] = bv[r] != 0xff ? atomicAdd(&h[bv[r]], 1u) : 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbins; i += PART_T)
    base[i] = h[i] ? atomicAdd(&cursor[i], (unsigned long long)h[i]) : 0;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    int64_t i = chunk0 + (int64_t)r * PART_T + threadIdx.x;
    if (bv[r] != 0xff) rowlist[base[bv[r]] + rank[r]] = (int32_t)i;
  }
}

int partition_rows(int64_t m, int nbins, Workspace& w, int64_t* cnt_host, int64_t* off_host,
                   cudaStream_t s) {
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(w.bincnt);
  cudaMemsetAsync(cnt, 0, 64 * sizeof(unsigned long long), s);
  if (m > 0) {
    int g = grid_for(m, PART_T * 16);
    k_bin_hist<<<g, PART_T, 0, s>>>(m, nbins, w.bins, cnt);
  }
  unsigned long long h[64];
  cudaMemcpyAsync(h, cnt, nbins * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("partition sync");
  off_host[0] = 0;
  for (int b = 0; b < nbins; ++b) {
    cnt_host[b] = (int64_t)h[b];
    off_host[b + 1] = off_host[b] + cnt_host[b];
  }
  unsigned long long cur[64];
  for (int b = 0; b < nbins; ++b) cur[b] = (unsigned long long)off_host[b];
  cudaMemcpyAsync(cnt, cur, nbins * sizeof(unsigned long long), cudaMemcpyHostToDevice, s);
  if (m > 0) {
    int g = grid_for(m, PART_T * 16);
    k_bin_scatter<<<g, PART_T, 0, s>>>(m, nbins, w.bins, cnt, w.rowlist);
  }
  // the host staging array `cur` must outlive the async copy
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("partition scatter");
  return check_cuda("partition", m > 0 ? 2 : 0);
}

// ---------------------------------------------------------------------------
// fallback-row selection and compaction

__device__ __forceinline__ bool is_fallback_row(int64_t i, const int8_t* kind, const int64_t* products,
                                                const uint8_t* overflow, const int32_t* exclude) {
  const bool fb = (overflow && overflow[i]) || (kind[i] == SG_KIND_FALLBACK && products[i] > 0);
  return fb && !(exclude && exclude[i] > 0);
}

__global__ void k_fb_flags(int64_t m, const int8_t* __restrict__ kind, const int64_t* __restrict__ products,
                           const uint8_t* __restrict__ overflow, const int32_t* __restrict__ exclude,
                           int64_t* __restrict__ flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  flags[i] = is_fallback_row(i, kind, products, overflow, exclude) ? 1 : 0;
}

__global__ void k_fb_scatter(int64_t m, const int8_t* __restrict__ kind, const int64_t* __restrict__ products,
                             const uint8_t* __restrict__ overflow, const int32_t* __restrict__ exclude,
                             const int64_t* __restrict__ pos, int64_t* __restrict__ rows_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (is_fallback_row(i, kind, products, overflow, exclude)) rows_out[pos[i]] = i;
}

template <typename V>
__global__ void __launch_bounds__(256) k_compact(int64_t m, const int64_t* __restrict__ counts,
                                                 const uint8_t* __restrict__ skip,
                                                 const int64_t* __restrict__ src_off,
                                                 const int64_t* __restrict__ dst_off,
                                                 const int32_t* __restrict__ src_col,
                                                 const V* __restrict__ src_val, int32_t* __restrict__ dst_col,
                                                 V* __restrict__ dst_val) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= m) return;
  if (skip && skip[row]) return;
  const int64_t c = counts[row];
  if (c == 0) return;
  const int64_t s = src_off[row], d = dst_off[row];
  if (s == d && src_col == dst_col) return;
  for (int64_t i = lane_id(); i < c; i += 32) {
    dst_col[d + i] = src_col[s + i];
    dst_val[d + i] = src_val[s + i];
  }
}


// ---------------------------------------------------------------------------
// estimation error of the per-row predictions (engine.py:218-226): over rows
// with a non-empty C row, rel = |pred - truth| / truth; mean and population
// std.  Two deterministic passes: fixed per-block partials (grid-stride), then
// one block folds them in index order.

constexpr int ERR_T = 256;
constexpr int ERR_BLOCKS = 1024;

template <int PASS>
__global__ void __launch_bounds__(ERR_T) k_est_err(int64_t m, const double* __restrict__ pred,
                                                   const int64_t* __restrict__ row_ptr, const double* __restrict__ mean,
                                                   double* __restrict__ part) {
  __shared__ double sh[ERR_T / 32][2];
  double s = 0.0, c = 0.0;
  const double mu = PASS == 1 ? *mean : 0.0;
  for (int64_t r = (int64_t)blockIdx.x * ERR_T + threadIdx.x; r < m; r += (int64_t)gridDim.x * ERR_T) {
    const int64_t t = row_ptr[r + 1] - row_ptr[r];
    if (t > 0) {
      const double rel = fabs(pred[r] - (double)t) / (double)t;
      if (PASS == 0) {
        s += rel;
        c += 1.0;
      } else {
        s += (rel - mu) * (rel - mu);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(SG_FULL, s, o);
    c += __shfl_xor_sync(SG_FULL, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[threadIdx.x >> 5][0] = s;
    sh[threadIdx.x >> 5][1] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ss = 0.0, cc = 0.0;
    for (int w = 0; w < ERR_T / 32; ++w) {
      ss += sh[w][0];
      cc += sh[w][1];
    }
    part[2 * blockIdx.x] = ss;
    part[2 * blockIdx.x + 1] = cc;
  }
}

// out[0] = live rows, out[1] = mean (PASS 0) / out[2] = std (PASS 1)
template <int PASS>
__global__ void __launch_bounds__(32) k_est_err_fold(int nb, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double s = 0.0, c = 0.0;
  for (int b = 0; b < nb; ++b) {
    s += part[2 * b];
    c += part[2 * b + 1];
  }
  if (PASS == 0) {
    out[0] = c;
    out[1] = c > 0 ? s / c : 0.0;
  } else {
    out[2] = out[0] > 0 ? sqrt(s / out[0]) : 0.0;
  }
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_abi_version(void) { return 1; }
unsigned long long sg_launch_count(void) { return g_launches.load(); }

int sg_kernel_timer(int enable) {
  ktimer_clear();
  g_kt_on.store(enable != 0);
  return SG_OK;
}

int sg_kernel_time(const char* name, double* total_ms, int64_t* launches) {
  if (!name || !total_ms || !launches) {
    set_error("sg_kernel_time: bad arguments");
    return SG_ERR_ARG;
  }
  std::lock_guard<std::mutex> g(g_kt_mu);
  double ms = 0.0;
  int64_t n = 0;
  for (auto& t : g_kt) {
    if (t.name != name) continue;
    if (cudaEventSynchronize(t.b) != cudaSuccess) return check_cuda("sg_kernel_time", 0);
    float e = 0.f;
    if (cudaEventElapsedTime(&e, t.a, t.b) != cudaSuccess) return check_cuda("sg_kernel_time", 0);
    ms += e;
    ++n;
  }
  *total_ms = ms;
  *launches = n;
  return SG_OK;
}
const char* sg_last_error(void) { return g_err.c_str(); }
size_t sg_workspace_bytes(int64_t m) { return workspace_bytes(m < 0 ? 0 : m); }

int sg_row_stats(int64_t m, int64_t b_ncols, const int64_t* a_ptr, const int32_t* a_col,
                 const int64_t* b_ptr, const int32_t* b_col, int64_t* products, int64_t* span_lo,
                 int64_t* span_hi, int64_t* totals2, void* stream) {
  if (m < 0 || !totals2) {
    set_error("sg_row_stats: bad arguments");
    return SG_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(totals2, 0, 2 * sizeof(int64_t), s);
  if (m == 0) return check_cuda("sg_row_stats", 0);
  constexpr int G = 8;
  k_row_stats<G><<<grid_for(m * G, 256), 256, 0, s>>>(m, b_ncols, a_ptr, a_col, b_ptr, b_col, products,
                                                      span_lo, span_hi, (unsigned long long*)totals2);
  const int gl = (int)std::min<int64_t>((m + RS_NT - 1) / RS_NT, 148 * 8);  // 8 sweeping blocks per SM
  k_row_stats_long<<<gl, RS_NT, 0, s>>>(m, b_ncols, a_ptr, a_col, b_ptr, b_col, products, span_lo, span_hi,
                                         (unsigned long long*)totals2);
  return check_cuda("sg_row_stats", 2);
}

int sg_hll_build(int64_t k, const int64_t* b_ptr, const int32_t* b_col, int p, uint8_t* regs,
                 void* stream) {
  if (p < 5 || p > 7 || k < 0) {
    set_error("sg_hll_build: precision must be 5, 6 or 7");
    return SG_ERR_ARG;
  }
  if (k == 0) return SG_OK;
  k_hll_build<<<grid_for(k, HLL_WARPS), HLL_WARPS * 32, 0, (cudaStream_t)stream>>>(k, b_ptr, b_col, p, regs);
  return check_cuda("sg_hll_build");
}

int sg_hll_estimate(int64_t nsel, const int64_t* rows, const int64_t* a_ptr, const int32_t* a_col,
                    const uint8_t* regs, int p, const double* lin_table, double alpha_mm, double* est,
                    void* stream) {
  if (p < 5 || p > 7 || nsel < 0) {
    set_error("sg_hll_estimate: precision must be 5, 6 or 7");
    return SG_ERR_ARG;
  }
  if (nsel == 0) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(nsel * 32, 256);
  if (p == 5)
    k_hll_estimate<1><<<g, 256, 0, s>>>(nsel, rows, a_ptr, a_col, regs, lin_table, alpha_mm, est);
  else if (p == 6)
    k_hll_estimate<2><<<g, 256, 0, s>>>(nsel, rows, a_ptr, a_col, regs, lin_table, alpha_mm, est);
  else
    k_hll_estimate<4><<<g, 256, 0, s>>>(nsel, rows, a_ptr, a_col, regs, lin_table, alpha_mm, est);
  return check_cuda("sg_hll_estimate");
}

int sg_plan(int64_t m, int pred_kind, const void* pred, const int64_t* products, const int64_t* span_lo,
            const int64_t* span_hi, const sg_tiers_t* tiers, int8_t* kind, int64_t* cap, int64_t* alloc,
            void* stream) {
  if (!tiers || tiers->n_hash < 1 || tiers->n_hash > 8 || tiers->n_dense < 1 || tiers->n_dense > 8 ||
      pred_kind < 0 || pred_kind > 2 || m < 0) {
    set_error("sg_plan: bad arguments");
    return SG_ERR_ARG;
  }
  if (m == 0) return SG_OK;
  k_plan<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(m, pred_kind, pred, products, span_lo, span_hi,
                                                             *tiers, kind, cap, alloc);
  return check_cuda("sg_plan");
}

int sg_scan(int64_t n, const int64_t* in, int64_t* out, void* ws, size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, n, w)) return SG_ERR_WORKSPACE;
  return scan_i64(n, in, out, w.partials, (cudaStream_t)stream);
}

int sg_select_fallback(int64_t m, const int8_t* kind, const int64_t* products, const uint8_t* overflow,
                       const int32_t* exclude_nwin, int64_t* rows_out, int64_t* n_out_host, void* ws,
                       size_t ws_bytes, void* stream) {
  Workspace w;
  if (!carve(ws, ws_bytes, m, w)) return SG_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (m == 0) {
    *n_out_host = 0;
    return SG_OK;
  }
  int g = grid_for(m, 256);
  k_fb_flags<<<g, 256, 0, s>>>(m, kind, products, overflow, exclude_nwin, w.tmp);
  // in-place scan of the flags (k_scan_down reads its tile before writing it)
  int rc = scan_i64(m, w.tmp, w.tmp, w.partials, s);
  if (rc) return rc;
  k_fb_scatter<<<g, 256, 0, s>>>(m, kind, products, overflow, exclude_nwin, w.tmp, rows_out);
  count_launches(2);
  cudaMemcpyAsync(n_out_host, w.tmp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_select_fallback sync");
  return check_cuda("sg_select_fallback");
}

int sg_est_errors(int64_t m, const double* pred, const int64_t* row_ptr, double* out3, void* ws, size_t ws_bytes,
                  void* stream) {
  if (m < 0 || !out3) {
    set_error("sg_est_errors: bad arguments");
    return SG_ERR_ARG;
  }
  if (!ws || ws_bytes < (size_t)ERR_BLOCKS * 16 + 64) {
    set_error("sg_est_errors: workspace too small");
    return SG_ERR_WORKSPACE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double* part = static_cast<double*>(ws);
  double* dev_out = part + 2 * ERR_BLOCKS;
  const int nb = (int)std::min<int64_t>(ERR_BLOCKS, std::max<int64_t>(1, (m + ERR_T - 1) / ERR_T));
  k_est_err<0><<<nb, ERR_T, 0, s>>>(m, pred, row_ptr, nullptr, part);
  k_est_err_fold<0><<<1, 32, 0, s>>>(nb, part, dev_out);
  k_est_err<1><<<nb, ERR_T, 0, s>>>(m, pred, row_ptr, dev_out + 1, part);
  k_est_err_fold<1><<<1, 32, 0, s>>>(nb, part, dev_out);
  if (int rc = check_cuda("k_est_err", 4)) return rc;
  cudaMemcpyAsync(out3, dev_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_cuda("sg_est_errors sync", 0);
  return SG_OK;
}

int sg_compact(int64_t m, int dtype, const int64_t* counts, const uint8_t* skip, const int64_t* src_off,
               const int64_t* dst_off, const int32_t* src_col, const void* src_val, int32_t* dst_col,
               void* dst_val, void* stream) {
  if (m == 0) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int g = grid_for(m * 32, 256);
  if (dtype == SG_F64)
    k_compact<double><<<g, 256, 0, s>>>(m, counts, skip, src_off, dst_off, src_col, (const double*)src_val,
                                        dst_col, (double*)dst_val);
  else
    k_compact<float><<<g, 256, 0, s>>>(m, counts, skip, src_off, dst_off, src_col, (const float*)src_val,
                                       dst_col, (float*)dst_val);
  return check_cuda("sg_compact");
}

}  // extern "C"

// -------------------------------------------------------------------------
// Deterministic values (EngineConfig(deterministic=True)): given C's final
// structure, every value is recomputed as a sum in the reference's stream
// order -- A entries ascending, then each B row's entries -- with plain
// adds (no atomics).  One warp per row: the warp walks the row's A entries
// in order; the lanes of one entry touch distinct C columns (a B row has
// unique columns), so one entry's adds never collide and the entries are
// applied one after another.  Values are bit-identical run to run and to a
// sequential sum (the reference's dense / fallback bins and its oracle,
// engine.py:13-14, accumulate.py:412-415, oracle.py:28-39).
namespace sg {

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* __restrict__ a, int64_t n, int32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <typename V>
__global__ void k_det_values(int64_t m, const int64_t* __restrict__ a_ptr, const int32_t* __restrict__ a_col,
                             const V* __restrict__ a_val, const int64_t* __restrict__ b_ptr,
                             const int32_t* __restrict__ b_col, const V* __restrict__ b_val,
                             const int64_t* __restrict__ c_ptr, const int32_t* __restrict__ c_col,
                             double* __restrict__ acc, V* __restrict__ c_val) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += nwarps) {
    const int64_t rs = c_ptr[r], n = c_ptr[r + 1] - rs;
    if (n == 0) continue;
    double* ar = acc + rs;
    for (int64_t i = lane; i < n; i += 32) ar[i] = 0.0;
    __syncwarp();
    for (int64_t t = a_ptr[r]; t < a_ptr[r + 1]; ++t) {
      const int32_t k = a_col[t];
      const double av = (double)a_val[t];
      const int64_t bs = b_ptr[k], bl = b_ptr[k + 1] - bs;
      for (int64_t q = lane; q < bl; q += 32) {
        const int64_t pos = lower_bound_i32(c_col + rs, n, b_col[bs + q]);
        ar[pos] = __dadd_rn(ar[pos], __dmul_rn(av, (double)b_val[bs + q]));  // no FMA: the reference rounds the product
      }
      __syncwarp();
    }
    for (int64_t i = lane; i < n; i += 32) c_val[rs + i] = (V)ar[i];
    __syncwarp();
  }
}

}  // namespace sg

extern "C" int sg_det_values(int64_t m, int dtype, const int64_t* a_ptr, const int32_t* a_col, const void* a_val,
                             const int64_t* b_ptr, const int32_t* b_col, const void* b_val, const int64_t* c_ptr,
                             const int32_t* c_col, void* c_val, double* acc, void* stream) {
  using namespace sg;
  if (m == 0) return SG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = (int)std::min<int64_t>((m + 7) / 8, 148 * 64);
  if (dtype == SG_F64)
    k_det_values<double><<<g, 256, 0, s>>>(m, a_ptr, a_col, (const double*)a_val, b_ptr, b_col,
                                           (const double*)b_val, c_ptr, c_col, acc, (double*)c_val);
  else
    k_det_values<float><<<g, 256, 0, s>>>(m, a_ptr, a_col, (const float*)a_val, b_ptr, b_col, (const float*)b_val,
                                          c_ptr, c_col, acc, (float*)c_val);
  count_launches(1);
  return check_cuda("k_det_values");
}
