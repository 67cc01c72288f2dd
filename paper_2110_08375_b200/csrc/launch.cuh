// launch.cuh -- host launchers of the heavy kernels, defined (and explicitly
// instantiated per precision) in separate translation units so the three
// precisions and the kernel families compile in parallel.
#pragma once
#include "types.cuh"

namespace mdls {

template <int M, bool TA, bool TB>
void gemm(cudaStream_t st, int64_t m, int64_t n, int64_t k, CMat A, CMat B, Mat C, int mode, double* part,
          int64_t part_cap_elems);

template <int M>
cudaError_t launch_leaf(cudaStream_t st, int64_t Mrows, int64_t js, int64_t bmax, Mat A, Mat Y, double* beta,
                        int64_t bps, Mat T, int* info, int* bw);

template <int M>
void launch_invert(cudaStream_t st, int64_t ntiles, int64_t nb, CMat U, Mat Vt, double diag_scale, const double* dbeta,
                   int* info);

template <int M>
void launch_bs_mulinv(cudaStream_t st, int64_t nb, int64_t tile, CMat Vt, const double* b, int64_t psb, double* x,
                      int64_t psx);

template <int M>
void launch_bs_update(cudaStream_t st, int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U, const double* x,
                      int64_t psx, double* b, int64_t psb);

}  // namespace mdls
