// launch.cuh -- host launchers of the heavy kernels, defined (and explicitly
// instantiated per precision) in separate translation units so the three
// precisions and the kernel families compile in parallel.
#pragma once
#include <cstdlib>

#include "types.cuh"

namespace mdls {

template <int M, bool TA, bool TB>
void gemm(cudaStream_t st, int64_t m, int64_t n, int64_t k, CMat A, CMat B, Mat C, int mode, double* part,
          int64_t part_cap_elems);

template <int M>
void leaf_t_product(cudaStream_t st, int B, int64_t n, int64_t r, CMat Y, CMat T, CMat C, Mat X, double* part,
                    int64_t part_cap_elems);

template <int M>
cudaError_t launch_leaf(cudaStream_t st, int64_t Mrows, int64_t js, int64_t bmax, Mat A, Mat Y, double* beta,
                        int64_t bps, Mat T, int* info, int* bw);

// chained leaves (register leaf with the previous-leaf prologue, kern_leaf.cuh)
inline int leaf_cluster_size() {
  static const int force8 = [] {
    const char* v = getenv("MDLS_LEAF_C");
    return (v && v[0] == '8') ? 1 : 0;
  }();
  return force8 ? 8 : max_cluster_size();
}
template <int M>
inline int chain_leaf_width(int64_t Mrows, int64_t js, int64_t bmax) {
  int B = 1;
  while (B * 2 <= bmax && B * 2 <= (M <= 2 ? 16 : 8)) B *= 2;
  if (B < 8) return 0;
  const int64_t rows = Mrows - js;
  const int C = (int)std::max<int64_t>(1, std::min<int64_t>(leaf_cluster_size(), rows));
  const int64_t R = cdiv(rows, C);
  if (2 * C < B) return 0;
  if (R <= 64 || (M <= 4 && R <= 128)) return B;
  return 0;
}
template <int M>
cudaError_t launch_leaf_chain(cudaStream_t st, int64_t Mrows, int64_t js, int B, Mat A, Mat Y, double* beta,
                              int64_t bps, Mat T, int* info, Mat Tp, int64_t jsp);

// the dataflow back substitution needs every row block of both update-kernel shapes inside one tile
template <int M>
inline bool bs_flow_ok(int64_t n, int64_t nb) {
  static const bool on = [] {
    const char* v = getenv("MDLS_BS_FLOW");
    return !(v && v[0] == '0');
  }();
  return on && nb % 32 == 0 && n % nb == 0;
}
template <int M>
void launch_invert(cudaStream_t st, int64_t ntiles, int64_t nb, CMat U, Mat Vt, Mat Us, int* info, int64_t info_off);

template <int M>
void launch_bs_mulinv(cudaStream_t st, int64_t nb, int64_t tile, CMat Vt, const double* b, int64_t psb, double* x,
                      int64_t psx, BsFlow fl, bool first);

template <int M>
void launch_bs_update(cudaStream_t st, int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U, const double* x,
                      int64_t psx, double* b, int64_t psb, BsFlow fl);

}  // namespace mdls
