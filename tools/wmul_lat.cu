// Latency of dependent md operations by one warp: per-thread mul/add vs the warp-cooperative wmul.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --fmad=false -o tools/wmul_lat tools/wmul_lat.cu
#include <cstdio>

#include "../paper_2110_08375_b200/csrc/md_warp.cuh"

using namespace mdls;

template <int M, int OP>
__global__ void lat(const double* in, double* out, long long* cyc, int reps) {
  md<M> a, b;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    a.v[k] = in[k];
    b.v[k] = in[M + k];
  }
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (OP == 0) a = mul<M>(a, b);
    else if (OP == 1) a = wmul<M>(a, b);
    else if (OP == 2) a = add<M>(a, b);
    else if (OP == 3) a = w_recip_fast<M>(a);
    else if (OP == 4) a = recip_fast<M>(a);
    else a = w_sqrt_fast<M>(a);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    for (int k = 0; k < M; ++k) out[k] = a.v[k];
    *cyc = (t1 - t0) / reps;
  }
}

template <int M>
void run() {
  double h[16];
  for (int k = 0; k < 2 * M; ++k) h[k] = 0.0;
  h[0] = 1.0000001;
  h[1] = 1e-17;
  h[M] = 0.9999999;
  h[M + 1] = -3e-18;
  double *in, *out;
  long long* cyc;
  cudaMalloc(&in, 16 * 8);
  cudaMalloc(&out, 16 * 8);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(in, h, 16 * 8, cudaMemcpyHostToDevice);
  const char* names[] = {"mul (1 thread)", "wmul (warp)", "add (1 thread)", "w_recip_fast", "recip_fast", "w_sqrt_fast"};
  for (int op = 0; op < 6; ++op) {
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: lat<M, 0><<<1, 32>>>(in, out, cyc, 20); break;
        case 1: lat<M, 1><<<1, 32>>>(in, out, cyc, 20); break;
        case 2: lat<M, 2><<<1, 32>>>(in, out, cyc, 20); break;
        case 3: lat<M, 3><<<1, 32>>>(in, out, cyc, 20); break;
        case 4: lat<M, 4><<<1, 32>>>(in, out, cyc, 20); break;
        default: lat<M, 5><<<1, 32>>>(in, out, cyc, 20); break;
      }
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("M=%d %-16s %8lld cycles\n", M, names[op], c);
  }
}

int main() {
  run<4>();
  run<8>();
  return 0;
}
