// types.cuh -- operand descriptors shared by the kernels and the host drivers.
//
// All operands are limb-planar ("staggered"): limb l of element
// (i, j) of an (ptr, ld, ps) operand is ptr[l*ps + j*ld + i].  Kernels are
// templated on the limb count M (2 dd, 4 qd, 8 od) and run on the FP64 pipe;
// no tensor cores (multiple-double arithmetic is error-free transformations,
// not a plain contraction).  Every reduction has a fixed tree, so results are
// bitwise reproducible run to run.
#pragma once
#include <cooperative_groups.h>

#include <climits>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "md.cuh"

namespace mdls {
namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// launch accounting / per-stage tracing (defined in ledger.cu).  Every kernel
// launch of the library goes through MDLS_LAUNCH: it is counted, and when
// tracing is on it is bracketed by CUDA events on its own stream and charged to
// the current stage (the paper's per-stage tables) and kernel family.
// ---------------------------------------------------------------------------
enum Family { F_GEMM = 0, F_PANEL = 1, F_INVERT = 2, F_BS = 3, F_MISC = 4, F_NFAM = 5 };
void trace_begin(cudaStream_t st, int family);
void trace_end(cudaStream_t st, int family);
void set_stage(int stage);
#define MDLS_LAUNCH(FAM, ST, ...)          \
  do {                                     \
    ::mdls::trace_begin((ST), (FAM));      \
    __VA_ARGS__;                           \
    ::mdls::trace_end((ST), (FAM));        \
  } while (0)

struct Mat {
  double* p;
  int64_t ld, ps;
};
struct CMat {
  const double* p;
  int64_t ld, ps;
};

constexpr int kNumSMs = 148;
constexpr int64_t kMaxSplit = 8;

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int grid_for(int64_t n, int threads) {
  int64_t g = cdiv(n, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 8 * kNumSMs));
}


inline CMat cm(const Mat& a) { return CMat{a.p, a.ld, a.ps}; }
inline Mat sub(const Mat& a, int64_t i, int64_t j) { return Mat{a.p + i + j * a.ld, a.ld, a.ps}; }
inline CMat sub(const CMat& a, int64_t i, int64_t j) { return CMat{a.p + i + j * a.ld, a.ld, a.ps}; }

template <int M>
struct GemmCfg;
template <>
struct GemmCfg<2> {
  static constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
};
template <>
struct GemmCfg<4> {
  static constexpr int BM = 32, BN = 32, BK = 16, TM = 2, TN = 2;
};
template <>
struct GemmCfg<8> {
  static constexpr int BM = 16, BN = 16, BK = 16, TM = 1, TN = 1;
};

struct GemmArgs {
  int64_t m, n, k;
  const double* A;
  int64_t lda, psa;
  const double* B;
  int64_t ldb, psb;
  double* C;
  int64_t ldc, psc;
  int mode;
  int64_t kc;     // k chunk per split
  double* part;   // split partials (nullptr: no split)
  int64_t S;      // number of splits
};

template <int M>
struct PanelArgs {
  int64_t Mrows, j0, w;
  Mat A;
  Mat Y;          // explicit Y (same row/column indexing as A)
  double* beta;   // beta of global column j at beta[l*bps + j]
  int64_t bps;
  int* info;      // min-slot: 1-based first zero/non-finite R_jj
};

}  // namespace mdls
