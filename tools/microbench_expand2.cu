// Isolated column expansion: R rows x W words (R-MAT-like density: a dense
// head, ~4.5% overall), saved bitmap + word ranks in global memory, block per
// row.  Variants: 0 = per-thread loop direct to global; 1 = staged + coalesced
// copy; 2 = read-only (loads, popc checksum).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void emit_bits(unsigned long long bits, int colbase, int* out) {
  unsigned lo = (unsigned)bits, hi = (unsigned)(bits >> 32); int k = 0;
  while (lo) { out[k++] = colbase + __ffs(lo) - 1; lo &= lo - 1; }
  while (hi) { out[k++] = colbase + 31 + __ffs(hi); hi &= hi - 1; }
}
template <int V>
__global__ void __launch_bounds__(512) k(int R, int W, const unsigned long long* bm, const int* pre,
                                         const long long* off, int* out, unsigned long long* sink) {
  __shared__ int buf[11000];
  unsigned long long acc = 0;
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    const unsigned long long* b = bm + (size_t)r * W;
    const int* p = pre + (size_t)r * W;
    int* o = out + off[r];
    if (V == 0) {
      for (int i = threadIdx.x; i < W; i += 512) emit_bits(b[i], 64 * i, o + p[i]);
    } else if (V == 1) {
      for (int c = 0; c < W; c += 2048) {
        int rb = p[c], re = (c + 2048 < W) ? p[c + 2048] : (int)(off[r + 1] - off[r]);
        for (int i = c + threadIdx.x; i < c + 2048; i += 512) emit_bits(b[i], 64 * i, buf + (p[i] - rb));
        __syncthreads();
        for (int i = threadIdx.x; i < re - rb; i += 512) o[rb + i] = buf[i];
        __syncthreads();
      }
    } else if (V == 3) {
      const int lane = threadIdx.x & 31;
      unsigned lt; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      for (int i0 = 0; i0 < W; i0 += 512) {
        const int i = i0 + threadIdx.x;
        const unsigned long long bits = b[i];
        const int pos = p[i];
        const bool dense = __popcll(bits) > 8;
        if (!dense) emit_bits(bits, 64 * i, o + pos);
        unsigned dm = __ballot_sync(0xffffffffu, dense);
        while (dm) {
          const int src = __ffs(dm) - 1; dm &= dm - 1;
          const unsigned long long wb = __shfl_sync(0xffffffffu, bits, src);
          const int wp = __shfl_sync(0xffffffffu, pos, src);
          const int wc = 64 * (i0 + (threadIdx.x & ~31) + src);
          const unsigned l32 = (unsigned)wb, h32 = (unsigned)(wb >> 32);
          if ((l32 >> lane) & 1u) o[wp + __popc(l32 & lt)] = wc + lane;
          if ((h32 >> lane) & 1u) o[wp + __popc(l32) + __popc(h32 & lt)] = wc + 32 + lane;
        }
      }
    } else {
      for (int i = threadIdx.x; i < W; i += 512) acc += __popcll(b[i]) + p[i];
    }
  }
  if (acc == 12345) sink[0] = acc;
}
int main() {
  const int R = 20000, W = 16384;
  size_t nw = (size_t)R * W;
  unsigned long long* hb = (unsigned long long*)malloc(nw * 8);
  int* hp = (int*)malloc(nw * 4);
  long long* ho = (long long*)malloc((R + 1) * 8);
  unsigned s = 1; long long tot = 0; ho[0] = 0;
  for (int r = 0; r < R; ++r) {
    int run = 0;
    for (int w = 0; w < W; ++w) {
      unsigned long long x = 0;
      int dens = w < 200 ? 600 : 30;  // per-mille bit density: dense head (hub columns), sparse tail
      for (int b = 0; b < 64; ++b) { s = s * 1664525u + 1013904223u; if ((s >> 8) % 1000 < (unsigned)dens) x |= 1ull << b; }
      hb[(size_t)r * W + w] = x; hp[(size_t)r * W + w] = run; run += __builtin_popcountll(x);
    }
    tot += run; ho[r + 1] = tot;
  }
  printf("rows %d words %d outputs %lld (%.1f per row)\n", R, W, tot, (double)tot / R);
  unsigned long long *db, *sink; int *dp, *dout; long long* doff;
  cudaMalloc(&db, nw * 8); cudaMalloc(&dp, nw * 4); cudaMalloc(&doff, (R + 1) * 8); cudaMalloc(&dout, tot * 4); cudaMalloc(&sink, 8);
  cudaMemcpy(db, hb, nw * 8, cudaMemcpyHostToDevice); cudaMemcpy(dp, hp, nw * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(doff, ho, (R + 1) * 8, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int v : {0, 3, 2}) for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (v == 0) k<0><<<sms * 4, 512>>>(R, W, db, dp, doff, dout, sink);
    if (v == 1) k<1><<<sms * 3, 512>>>(R, W, db, dp, doff, dout, sink);
    if (v == 2) k<2><<<sms * 4, 512>>>(R, W, db, dp, doff, dout, sink);
    if (v == 3) k<3><<<sms * 4, 512>>>(R, W, db, dp, doff, dout, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = nw * 12.0 + (v != 2 ? tot * 4.0 : 0);
    printf("variant %d: %.2f ms  %.0f GB/s  %.2f ns/output\n", v, ms, bytes / ms / 1e6, ms * 1e6 / tot);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
