// Phase timing of one leaf factorisation (clock64 marks in CTA 0, thread 0).
// nvcc -DMDLS_LEAF_PROF -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --fmad=false tools/leaf_prof.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#define MDLS_LEAF_SMEM_TU
#include "../paper_2110_08375_b200/csrc/kern_leaf.cuh"

namespace mdls {
void set_stage(int) {}
int max_cluster_size() { return 16; }
void trace_begin(cudaStream_t, int) {}
void trace_end(cudaStream_t, int) {}
}  // namespace mdls

template <int M>
void run(int Mrows, int bmax) {
  using namespace mdls;
  const int K = 16;
  std::vector<double> h((size_t)M * Mrows * K);
  srand(1);
  for (size_t i = 0; i < (size_t)Mrows * K; ++i) h[i] = 2.0 * rand() / RAND_MAX - 1.0;
  double *A, *Y, *beta, *T;
  int* info;
  cudaMalloc(&A, h.size() * 8);
  cudaMalloc(&Y, h.size() * 8);
  cudaMalloc(&beta, M * K * 8);
  cudaMalloc(&T, M * 1024 * 8);
  cudaMalloc(&info, 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    int bw = 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = launch_leaf<M>(0, Mrows, 0, bmax, Mat{A, Mrows, (int64_t)Mrows * K}, Mat{Y, Mrows, (int64_t)Mrows * K},
                                   beta, K, Mat{T, 32, 1024}, info, &bw);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long p[64 * 12];
    cudaMemcpyFromSymbol(p, g_leaf_prof, sizeof(p));
    printf("M=%d rows=%d B=%d err=%s %.1f us\n", M, Mrows, bw, cudaGetErrorString(e), ms * 1e3);
    if (rep == 2) {
      double avg[9] = {0};
      for (int l = 0; l < bw; ++l)
        for (int ph = 1; ph <= 8; ++ph) avg[ph] += (double)(p[l * 12 + ph] - p[l * 12 + ph - 1]) / bw;
      const char* names[] = {"", "products", "warp+cta reduce", "cluster.sync", "dsmem sum", "scalars1", "scalars2",
                             "w/v", "update"};
      double tot = 0;
      for (int ph = 1; ph <= 8; ++ph) {
        printf("  %-16s %8.0f cycles\n", names[ph], avg[ph]);
        tot += avg[ph];
      }
      printf("  total/column %8.0f cycles; column 0 start->column %d end: %lld\n", tot, bw - 1,
             p[(bw - 1) * 12 + 8] - p[0]);
    }
  }
}

template <int M>
void run_chain(int Mrows) {
  using namespace mdls;
  const int K = 32;
  std::vector<double> h((size_t)M * Mrows * K);
  srand(2);
  for (size_t i = 0; i < (size_t)Mrows * K; ++i) h[i] = 2.0 * rand() / RAND_MAX - 1.0;
  double *A, *Y, *beta, *T;
  int* info;
  cudaMalloc(&A, h.size() * 8);
  cudaMalloc(&Y, h.size() * 8);
  cudaMemset(Y, 0, h.size() * 8);
  cudaMalloc(&beta, M * K * 8);
  cudaMalloc(&T, M * 32 * K * 8);
  cudaMalloc(&info, 4);
  const int B = chain_leaf_width<M>(Mrows, 0, 16);
  Mat Am{A, Mrows, (int64_t)Mrows * K}, Ym{Y, Mrows, (int64_t)Mrows * K};
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaError_t e0 = launch_leaf_chain<M>(0, Mrows, 0, B, Am, Ym, beta, K, Mat{T, 32, 32 * K}, info, Mat{nullptr, 0, 0}, -1);
    cudaEvent_t a0, a1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    cudaEventRecord(a0);
    cudaError_t e1 = launch_leaf_chain<M>(0, Mrows, B, B, Am, Ym, beta, K, Mat{T + 32 * B, 32, 32 * K}, info,
                                          Mat{T, 32, 32 * K}, 0);
    cudaEventRecord(a1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a0, a1);
    long long p[64 * 12];
    cudaMemcpyFromSymbol(p, g_leaf_prof, sizeof(p));
    printf("chain M=%d rows=%d B=%d %s/%s second leaf (with prologue) %.1f us\n", M, Mrows, B, cudaGetErrorString(e0),
           cudaGetErrorString(e1), ms * 1e3);
    if (rep == 2) {
      const char* names[] = {"stage", "cluster.sync", "Z partial+push", "wait Z + sum", "Z' + push", "wait Z'", "update"};
      for (int k = 1; k <= 6; ++k) printf("  prologue %-16s %8lld cycles\n", names[k], p[63 * 12 + k] - p[63 * 12 + k - 1]);
      printf("  prologue -> column 0 start %lld cycles\n", p[0] - p[63 * 12 + 6]);
    }
  }
}

int main() {
#ifdef PROF_OD
  run_chain<8>(1024);
  run<8>(1024, 8);
  run_chain<4>(1024);
  run<4>(1024, 8);
  return 0;
#endif
  run_chain<2>(1024);
  run_chain<2>(512);
  run<2>(1024, 16);
  run<2>(1024, 8);
  run<2>(512, 16);
  run<2>(256, 16);
#ifdef PROF_QD
  run<4>(1024, 8);
#endif
  // run<8>(1024, 8);  (od: long compile)
  return 0;
}
