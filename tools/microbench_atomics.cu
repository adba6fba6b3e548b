// Throughput of the accumulator primitives on B200 (design evidence for
// DESIGN.md): shared-memory ATOMS.OR / ATOMS.CAS / fp64 add (CAS loop),
// plain STS.U8, and global RED.ADD.F64 into an L2-resident per-CTA window.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

template <int OP>
__global__ void k(int iters, double* gout, unsigned long long* sink) {
  extern __shared__ unsigned long long sm[];  // 128 KB
  const int W = 16384;  // 64-bit words
  for (int i = threadIdx.x; i < W; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  double* gw = gout + (size_t)blockIdx.x * 32768;  // 256 KB window per CTA
  for (int it = 0; it < iters; ++it) {
    s = rnd(s);
    uint32_t a = s & (W - 1);
    if (OP == 0) atomicOr(&sm[a], 1ull << (s >> 26));
    if (OP == 1) atomicCAS((int*)sm + (s & (2 * W - 1)), 0, (int)s);
    if (OP == 2) atomicAdd((double*)sm + a, 1.0);
    if (OP == 3) ((volatile unsigned char*)sm)[s & (8 * W - 1)] = 1;
    if (OP == 4) atomicAdd(gw + (s & 32767), 1.0);
    if (OP == 5) { unsigned long long w = sm[a]; sink[0] += (w >> 63); }
    if (OP == 6) atomicOr((unsigned*)sm + (s & (2 * W - 1)), 1u << (s >> 27));
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[1 + blockIdx.x % 7] += sm[0];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* g; cudaMalloc(&g, (size_t)sms * 4 * 32768 * 8);
  unsigned long long* sink; cudaMalloc(&sink, 64);
  const char* names[] = {"smem atomicOr u64 (ATOMS.OR)", "smem atomicCAS i32 (ATOMS.CAS)",
                         "smem atomicAdd f64 (CAS loop)", "smem st.u8 plain", "global RED.ADD.F64 L2-window",
                         "smem ld.u64 (LDS)", "smem atomicOr u32 (ATOMS.OR)"};
  for (int op = 0; op < 7; ++op) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (1024 / tpb > 1 ? 1 : 1);
      int iters = 4096;
      void (*kern)(int, double*, unsigned long long*) =
          op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : k<6>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
      kern<<<blocks, tpb, 131072>>>(16, g, sink);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<blocks, tpb, 131072>>>(iters, g, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * tpb * iters;
      printf("%-36s tpb=%4d  %8.1f Gop/s  (%.3f ops/clk/SM @1.9GHz)\n", names[op], tpb, ops / ms / 1e6,
             ops / (ms * 1e-3) / sms / 1.9e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
