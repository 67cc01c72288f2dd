// FP64 pipe throughput microbenchmark (DFMA / DADD / DMUL lane-ops per second).
// Used once per pool to pin the roofline denominator stated in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void kern(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) {
        x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
      } else if (OP == 1) {
        x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
        x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
      } else {
        x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, a); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, a);
        x4 = __dmul_rn(x4, a); x5 = __dmul_rn(x5, a); x6 = __dmul_rn(x6, a); x7 = __dmul_rn(x7, a);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <int OP>
void run(const char* name, int sms) {
  double* out; int threads = 256, blocks = sms * 8, iters = 4096;
  cudaMalloc(&out, sizeof(double) * threads * blocks);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<OP><<<blocks, threads>>>(out, iters, 1.0000001, 1e-300);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(out, iters, 1.0000001, 1e-300);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)threads * blocks * iters * 64;
  printf("%s: %.3f ms, %.2f T lane-ops/s, per SM per clk @1965MHz: %.1f\n", name, ms, ops / ms / 1e9,
         ops / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(out);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz l2=%d MB smem/blk optin=%zu regs/SM=%d\n", p.name, p.multiProcessorCount, p.clockRate,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  run<0>("DFMA", p.multiProcessorCount);
  run<1>("DADD", p.multiProcessorCount);
  run<2>("DMUL", p.multiProcessorCount);
  run<0>("DFMA", p.multiProcessorCount);
  return 0;
}
