// Bitmap -> sorted column list expansion cost, in isolation (design check).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void emit_bits_smem(unsigned long long bits, int colbase, int* out) {
  unsigned lo = (unsigned)bits, hi = (unsigned)(bits >> 32);
  int k = 0;
  while (lo) { out[k++] = colbase + __ffs(lo) - 1; lo &= lo - 1; }
  while (hi) { out[k++] = colbase + 31 + __ffs(hi); hi &= hi - 1; }
}
__global__ void __launch_bounds__(1024, 1) k(const unsigned long long* gbm, int nwords, int* out, int reps, long long* cyc) {
  __shared__ unsigned long long bm[2048];
  __shared__ int pre[2048];
  __shared__ int colbuf[5120];
  for (int i = threadIdx.x; i < nwords; i += 1024) bm[i] = gbm[(size_t)blockIdx.x * nwords + i];
  __syncthreads();
  if (threadIdx.x == 0) { int r = 0; for (int i = 0; i < nwords; ++i) { pre[i] = r; r += __popcll(bm[i]); } }
  __syncthreads();
  long long t0 = clock64();
  int cnt = pre[nwords - 1] + __popcll(bm[nwords - 1]);
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < nwords; i += 1024) emit_bits_smem(bm[i], 64 * i, colbuf + pre[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += 1024) out[(size_t)blockIdx.x * 16384 + i] = colbuf[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = (clock64() - t0) / reps;
}
int main() {
  const int nw = 1000, blocks = 148;
  unsigned long long* h = new unsigned long long[(size_t)blocks * nw];
  unsigned s = 12345;
  for (size_t i = 0; i < (size_t)blocks * nw; ++i) {
    unsigned long long w = 0;
    for (int b = 0; b < 64; ++b) { s = s * 1664525u + 1013904223u; if ((s >> 8) % 1000 < 66) w |= 1ull << b; }
    h[i] = w;
  }
  unsigned long long* d; int* out; long long* cyc;
  cudaMalloc(&d, (size_t)blocks * nw * 8); cudaMalloc(&out, (size_t)blocks * 16384 * 4); cudaMalloc(&cyc, blocks * 8);
  cudaMemcpy(d, h, (size_t)blocks * nw * 8, cudaMemcpyHostToDevice);
  k<<<blocks, 1024>>>(d, nw, out, 50, cyc);
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  long long sum = 0; for (int i = 0; i < blocks; ++i) sum += c[i];
  printf("expand %d words (~%.0f bits): %lld cycles per window\n", nw, nw * 64 * 0.066, sum / blocks);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
