// Latency microbenchmarks for the panel chain (one warp, clock64 around dependent chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --fmad=false tools/lat_bench.cu -o tools/lat_bench
#include <cstdio>

#include "../paper_2110_08375_b200/csrc/md.cuh"

using namespace mdls;

constexpr int N = 256;

__global__ void k_lat(double* out, long long* cyc, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 + 1e-12, c = 1e-20;
  long long t0, t1;
  int slot = 0;
  auto rec = [&](long long dt) {
    if (threadIdx.x == 0) cyc[slot] = dt;
    ++slot;
  };
  // DADD chain
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, c);
  t1 = clock64();
  rec(t1 - t0);
  // DFMA chain
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) a = __fma_rn(a, b, c);
  t1 = clock64();
  rec(t1 - t0);
  // dd_add chain
  md<2> x{{a, 1e-17}}, y{{1e-3, 1e-20}};
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) x = dd_add(x, y);
  t1 = clock64();
  rec(t1 - t0);
  // dd_mul chain
  md<2> z{{1.0000001, 1e-18}};
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) x = dd_mul(x, z);
  t1 = clock64();
  rec(t1 - t0);
  // shfl of a double + dadd
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
  t1 = clock64();
  rec(t1 - t0);
  // dsqrt chain
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) a = __dsqrt_rn(a + 2.0);
  t1 = clock64();
  rec(t1 - t0);
  // ddiv chain
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) a = __ddiv_rn(b, a + 2.0);
  t1 = clock64();
  rec(t1 - t0);
  // drcp chain
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) a = __drcp_rn(a + 2.0);
  t1 = clock64();
  rec(t1 - t0);
  // syncthreads
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  rec(t1 - t0);
  // fp32 rsqrt approx chain (MUFU)
  float f = (float)a + 2.0f;
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) f = rsqrtf(f) + 2.0f;
  t1 = clock64();
  rec(t1 - t0);
  // md<4> add chain
  md<4> q4{{a, 1e-17, 1e-34, 1e-51}}, r4{{1e-3, 1e-20, 1e-37, 1e-54}};
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) q4 = gen_add<4>(q4, r4);
  t1 = clock64();
  rec(t1 - t0);
  // int add chain (baseline for loop overhead)
  int ii = threadIdx.x;
  t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < N; ++i) ii = ii * 3 + 1;
  t1 = clock64();
  rec(t1 - t0);
  out[threadIdx.x] = a + x.v[0] + x.v[1] + f + q4.v[0] + ii;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  const char* names[] = {"DADD", "DFMA", "dd_add", "dd_mul", "shfl+DADD", "dsqrt_rn", "ddiv_rn", "drcp_rn",
                         "syncthreads(1 warp)", "rsqrtf+fadd", "qd add", "IMAD(int chain)"};
  for (int rep = 0; rep < 2; ++rep) {
    k_lat<<<1, 32>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
  }
  for (int i = 0; i < 12; ++i) printf("%-22s %8.1f cycles/op\n", names[i], (double)cyc[i] / N);
  return 0;
}
