// kern_misc.cuh -- elementwise md arithmetic and utility kernels.
#pragma once
#include "md_warp.cuh"
#include "types.cuh"

namespace mdls {

// ============================================================================
// A0: elementwise md arithmetic
// ============================================================================
template <int M>
__global__ void md_op_kernel(int op, int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                             double* __restrict__ c, int64_t ps) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    md<M> x = ld<M>(a, ps, e), r;
    md<M> y = (op >= 4) ? md_zero<M>() : ld<M>(b, ps, e);
    switch (op) {
      case 0: r = add<M>(x, y); break;
      case 1: r = sub<M>(x, y); break;
      case 2: r = mul<M>(x, y); break;
      case 3: r = div<M>(x, y); break;
      case 4: r = sqrt<M>(x); break;
      case 5: r = sqrt_fast<M>(x); break;
      default: r = recip_fast<M>(x); break;
    }
    st<M>(c, ps, e, r);
  }
}

// ops 7, 8, 9: the warp-cooperative product / square root / reciprocal (md_warp.cuh), one warp per entry
template <int M>
__global__ void md_op_warp_kernel(int op, int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                  double* __restrict__ c, int64_t ps) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = w0; e < n; e += nw) {  // warp-uniform loop
    const md<M> x = ld<M>(a, ps, e);
    const md<M> y = (op == 7) ? ld<M>(b, ps, e) : md_zero<M>();
    md<M> r;
    if constexpr (M <= 2) {
      r = (op == 7) ? mul<M>(x, y) : (op == 8 ? sqrt_fast<M>(x) : recip_fast<M>(x));
    } else {
      r = (op == 7) ? wmul<M>(x, y) : (op == 8 ? w_sqrt_fast<M>(x) : w_recip_fast<M>(x));
    }
    if ((threadIdx.x & 31) == 0) st<M>(c, ps, e, r);
  }
}

// ============================================================================
// utility kernels
// ============================================================================
// dst(i, j) = src(i, j) for i < rows, j < cols (all limbs); optional zero of the
// strictly-lower part (i > j) -- used for R_out.
template <int M>
__global__ void copy_kernel(int64_t rows, int64_t cols, CMat src, Mat dst, int zero_lower) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double v = src.p[k * src.ps + j * src.ld + i];
      dst.p[k * dst.ps + j * dst.ld + i] = (zero_lower && i > j) ? 0.0 : v;
    }
  }
}

// real embedding of a complex M x K matrix: E = [[Re, -Im], [Im, Re]] (2M x 2K, ld 2M) and of b: [Re b; Im b]
template <int M>
__global__ void embed_complex_kernel(int64_t rows, int64_t cols, CMat Ar, CMat Ai, const double* br,
                                     const double* bi, int64_t psb, Mat E, double* eb, int64_t pse) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double re = Ar.p[k * Ar.ps + j * Ar.ld + i], im = Ai.p[k * Ai.ps + j * Ai.ld + i];
      double* p = E.p + k * E.ps;
      p[j * E.ld + i] = re;
      p[j * E.ld + rows + i] = im;
      p[(cols + j) * E.ld + i] = -im;
      p[(cols + j) * E.ld + rows + i] = re;
      if (j == 0) {
        eb[k * pse + i] = br[k * psb + i];
        eb[k * pse + rows + i] = bi[k * psb + i];
      }
    }
  }
}

// explicit Y (unit lower trapezoidal) from a factored A: 0 above, 1 on, v below the diagonal
template <int M>
__global__ void extract_y_kernel(int64_t rows, int64_t cols, CMat a, Mat y) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double v = (i > j) ? a.p[k * a.ps + j * a.ld + i] : ((i == j && k == 0) ? 1.0 : 0.0);
      y.p[k * y.ps + j * y.ld + i] = v;
    }
  }
}

// Q = I on rows x cols
template <int M>
__global__ void set_identity_kernel(int64_t rows, int64_t cols, Mat q) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
#pragma unroll
    for (int k = 0; k < M; ++k) q.p[k * q.ps + j * q.ld + i] = (k == 0 && i == j) ? 1.0 : 0.0;
  }
}

// C = 0 on rows x cols
template <int M>
__global__ void set_zero_kernel(int64_t rows, int64_t cols, Mat q) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
#pragma unroll
    for (int k = 0; k < M; ++k) q.p[k * q.ps + j * q.ld + i] = 0.0;
  }
}

// info <- -1 if any limb of the rows x cols operand is not finite
template <int M>
__global__ void finite_check_kernel(int64_t rows, int64_t cols, CMat a, int* info) {
  const int64_t total = rows * cols;
  bool bad = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
#pragma unroll
    for (int k = 0; k < M; ++k) bad |= !isfinite(a.p[k * a.ps + j * a.ld + i]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(info, -1);
}

static __global__ void info_init_kernel(int* slot) { *slot = INT_MAX; }
// dev_info = min-slot (1-based first failure) or 0; a -1 (non-finite input) wins
static __global__ void info_finish_kernel(const int* slot, const int* pre, int* dev_info) {
  int v = *slot;
  int r = (v == INT_MAX) ? 0 : v;
  if (pre && *pre == -1) r = -1;
  *dev_info = r;
}
static __global__ void int_set_kernel(int* p, int v) { *p = v; }


// ||y||_2 of an md vector of length n in md (f1: the least-squares residual norm from the trailing
// entries of Q^T b): one CTA, per-thread accumulators over a fixed stride, a fixed-order
// shared-memory tree of exact accumulator merges, one normalisation, md sqrt (QDlib-style, A0).
template <int M>
__global__ void __launch_bounds__(256) norm2_kernel(int64_t n, const double* __restrict__ y, int64_t psy,
                                                    double* out, int64_t pso) {
  __shared__ Acc<M> part[256];
  Acc<M> acc;
  acc.init();
  int cnt = 0;
  for (int64_t i = threadIdx.x; i < n; i += 256) {
    const md<M> v = ld<M>(y, psy, i);
    acc.add_prod(v, v);
    if (++cnt == 8) {  // keep the lower bins small (md.cuh Acc)
      acc.renorm_bins();
      cnt = 0;
    }
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s >= 1; s >>= 1) {
    if ((int)threadIdx.x < s) {
      Acc<M> a = part[threadIdx.x];
      a.merge(part[threadIdx.x + s]);
      part[threadIdx.x] = a;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) st<M>(out, pso, 0, sqrt<M>(part[0].get()));
}

}  // namespace mdls
