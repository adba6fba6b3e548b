// Store-path check: CTAs of 1024 threads write 10.8k-entry (int32 + fp64)
// slices of a large C array, like the window kernel's emission.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(1024, 1) k(int32_t* col, double* val, long long nitems, int per,
                                             unsigned long long* ticket, int sync_each, int order) {
  __shared__ long long it;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) it = atomicAdd(ticket, 1ull);
    __syncthreads();
    long long b = it;
    if (b >= nitems) return;
    long long slot = order ? (b * 2654435761ll) % nitems : b;
    long long base = slot * per + 3;  // unaligned like real windows
    for (int i = threadIdx.x; i < per; i += 1024) {
      col[base + i] = (int)(base + i);
      val[base + i] = (double)i;
    }
    if (sync_each) __syncthreads();
  }
}
int main() {
  long long n = 1277000000ll;  // entries (rmat18-size C)
  int per = 10852;
  long long items = n / per - 1;
  int32_t* col; double* val; unsigned long long* t;
  cudaMalloc(&col, n * 4); cudaMalloc(&val, n * 8); cudaMalloc(&t, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int order = 0; order < 2; ++order)
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(t, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 1024>>>(col, val, items, per, t, 1, order);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)items * per * 12;
    printf("order=%s rep %d: %.2f ms  %.0f GB/s  %.0f cycles/item/SM @1.9GHz\n", order ? "scattered" : "sequential",
           rep, ms, bytes / ms / 1e6, ms * 1e-3 * 1.9e9 * sms / items);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
