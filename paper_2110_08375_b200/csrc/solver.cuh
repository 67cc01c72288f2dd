// solver.cuh -- host drivers (launch sequences) behind the C-ABI of include/mdls.h.
//
// Algorithm 2 (blocked Householder QR) and Algorithm 1 (tiled back
// substitution) as stream-ordered kernel sequences: no host
// synchronisation, no allocation (the caller's workspace is carved up here), so
// a whole least-squares solve can be captured in one CUDA graph.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/mdls.h"
#include "launch.cuh"
#include "kern_misc.cuh"

namespace mdls {

// ---------------------------------------------------------------------------
// workspace plan (bytes, 256-aligned segments)
// ---------------------------------------------------------------------------
struct Plan {
  size_t af = 0, q = 0, y = 0, w = 0, beta = 0, s = 0, t = 0, x = 0, part = 0, v0 = 0, v1 = 0, v2 = 0, vt = 0,
         info = 0, total = 0;
};

template <int M>
Plan make_plan(int op, int64_t Mr, int64_t K, int64_t nb) {
  Plan p;
  const size_t md = sizeof(double) * M;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  const int64_t mx = std::max(Mr, K);
  const bool qr_like = (op == MDLS_OP_QR || op == MDLS_OP_LSTSQ || op == MDLS_OP_LSTSQ_NOQ);
  if (op == MDLS_OP_LSTSQ || op == MDLS_OP_LSTSQ_NOQ) p.af = take(md * Mr * K);
  if (op == MDLS_OP_LSTSQ) p.q = take(md * Mr * Mr);
  if (qr_like) {
    p.y = take(md * Mr * K);
    p.w = take(md * Mr * K);
    p.beta = take(md * K);
    p.s = take(md * nb * nb);
    p.t = take(md * std::max<int64_t>(nb * nb, 256));
  }
  if (op == MDLS_OP_APPLY_QT) p.y = take(md * Mr * K);
  if (qr_like || op == MDLS_OP_APPLY_QT) {
    p.x = take(md * nb * mx);
    p.part = take(md * kMaxSplit * nb * mx);
  }
  p.v0 = take(md * mx);
  p.v1 = take(md * mx);
  p.v2 = take(md * mx);
  if (op == MDLS_OP_BACKSUB || op == MDLS_OP_LSTSQ || op == MDLS_OP_LSTSQ_NOQ) p.vt = take(md * nb * K);
  p.info = take(4 * sizeof(int));
  p.total = off;
  return p;
}


// ---------------------------------------------------------------------------
// Algorithm 2 on A (M x K), panels of width nb; fills Y (explicit), W, beta.
// ---------------------------------------------------------------------------
template <int M>
struct QrBufs {
  Mat Y, W;
  double* beta;
  Mat S, T, X;
  double* part;
  int64_t part_cap;
  int* info_slot;
};

// Panel k of Algorithm 2: factor columns [j0, j0+nb) in leaves of
// B <= 16 columns (launch_leaf: v, beta, R, leaf T); after each leaf
//   W_s = -Y_s T_s                              (the leaf's P_WY = I + W_s Y_s^T)
//   C_s += Y_s (W_s^T C_s)  on the panel columns right of the leaf ("beta R^T v",
//                                                 "update R" as two md GEMMs)
//   W_s += W_<s (Y_<s^T W_s) (block form of z = -beta (v + W Y^T v))
// so the panel's W (P_WY = I + W Y^T) is built column block by block.
template <int M>
cudaError_t qr_panel(cudaStream_t st, int64_t Mr, int64_t nb, int64_t k, Mat A, Mat Y, Mat W, double* beta,
                     int64_t bps, const QrBufs<M>& b) {
  const int64_t j0 = k * nb, r = Mr - j0;
  int64_t js = j0;
  while (js < j0 + nb) {
    int bw = 1;
    set_stage(MDLS_ST_PANEL);
    Mat Tl{b.T.p, 16, 256};
    cudaError_t e = launch_leaf<M>(st, Mr, js, j0 + nb - js, A, Y, beta, bps, Tl, b.info_slot, &bw);
    if (e != cudaSuccess) return e;
    const int64_t rs = Mr - js;
    const CMat Ys = sub(cm(Y), js, js);
    Mat Ws = sub(W, js, js);
    set_stage(MDLS_ST_WY);
    gemm<M, false, false>(st, rs, bw, bw, Ys, cm(Tl), Ws, 3, nullptr, 0);  // W_s = -Y_s T_s
    const int64_t rem = j0 + nb - (js + bw);
    if (rem > 0) {
      set_stage(MDLS_ST_PANEL);
      Mat Cs = sub(A, js, js + bw);
      gemm<M, true, false>(st, bw, rem, rs, cm(Ws), cm(Cs), b.X, 0, b.part, b.part_cap);
      gemm<M, false, false>(st, rs, rem, bw, Ys, cm(b.X), Cs, 1, nullptr, 0);
    }
    if (js > j0) {
      set_stage(MDLS_ST_WY);
      const int64_t np = js - j0;
      gemm<M, true, false>(st, np, bw, rs, sub(cm(Y), js, j0), cm(Ws), b.X, 0, b.part, b.part_cap);
      gemm<M, false, false>(st, r, bw, np, sub(cm(W), j0, j0), cm(b.X), sub(W, j0, js), 1, nullptr, 0);
    }
    js += bw;
  }
  (void)r;
  return cudaGetLastError();
}

// apply panel k to the columns [c0, c1) of A: C += Y_k (W_k^T C) ("YWT * C", "R + YWTC")
template <int M>
void qr_apply_panel(cudaStream_t st, int64_t Mr, int64_t nb, int64_t k, CMat Yk, CMat Wk, Mat A, int64_t c0,
                    int64_t c1, const QrBufs<M>& b) {
  if (c1 <= c0) return;
  const int64_t j0 = k * nb, r = Mr - j0;
  set_stage(MDLS_ST_TRAILING);
  Mat Cm = sub(A, j0, c0);
  gemm<M, true, false>(st, nb, c1 - c0, r, Wk, cm(Cm), b.X, 0, b.part, b.part_cap);
  gemm<M, false, false>(st, r, c1 - c0, nb, Yk, cm(b.X), Cm, 1, nullptr, 0);
}

template <int M>
cudaError_t qr_factor(cudaStream_t st, int64_t Mr, int64_t K, int64_t nb, Mat A, const QrBufs<M>& b, int64_t kbeg,
                      int64_t kend, bool trailing) {
  for (int64_t k = kbeg; k < kend; ++k) {
    const int64_t j0 = k * nb;
    cudaError_t e = qr_panel<M>(st, Mr, nb, k, A, b.Y, b.W, b.beta, K, b);
    if (e != cudaSuccess) return e;
    if (trailing) qr_apply_panel<M>(st, Mr, nb, k, sub(cm(b.Y), j0, j0), sub(cm(b.W), j0, j0), A, j0 + nb, K, b);
  }
  return cudaGetLastError();
}

// backward Q accumulation: Q = I; for k = N..1: Q_tr += W_k (Y_k^T Q_tr)
template <int M>
void form_q_backward(cudaStream_t st, int64_t Mr, int64_t K, int64_t nb, Mat Q, const QrBufs<M>& b) {
  set_stage(MDLS_ST_FORM_Q);
  MDLS_LAUNCH(F_MISC, st, set_identity_kernel<M><<<grid_for(Mr * Mr, 256), 256, 0, st>>>(Mr, Mr, Q));
  const int64_t N = K / nb;
  for (int64_t k = N - 1; k >= 0; --k) {
    const int64_t j0 = k * nb, r = Mr - j0;
    const CMat Yp = sub(cm(b.Y), j0, j0), Wp = sub(cm(b.W), j0, j0);
    Mat Qs = sub(Q, j0, j0);
    gemm<M, true, false>(st, nb, r, r, Yp, cm(Qs), b.X, 0, b.part, b.part_cap);
    gemm<M, false, false>(st, r, r, nb, Wp, cm(b.X), Qs, 1, nullptr, 0);
  }
}

// y = Q^T b by panels: y = b; for k = 1..N: y_k += Y_k (W_k^T y_k)
template <int M>
void apply_qt_panels(cudaStream_t st, int64_t Mr, int64_t K, int64_t nb, CMat Y, CMat W, Mat y, Mat X, double* part,
                     int64_t part_cap) {
  set_stage(MDLS_ST_QTB);
  const int64_t N = K / nb;
  for (int64_t k = 0; k < N; ++k) {
    const int64_t j0 = k * nb, r = Mr - j0;
    const CMat Yp = sub(Y, j0, j0), Wp = sub(W, j0, j0);
    Mat ys = sub(y, j0, 0);
    gemm<M, true, false>(st, nb, 1, r, Wp, cm(ys), X, 0, part, part_cap);
    gemm<M, false, false>(st, r, 1, nb, Yp, cm(X), ys, 1, nullptr, 0);
  }
}

// Algorithm 1: U x = y (leading n x n of U), tiles of nb
template <int M>
void backsub(cudaStream_t st, int64_t n, int64_t nb, CMat U, const double* y, int64_t psy, double* x, int64_t psx,
             Mat Vt, double* bwork, int* info_slot) {
  const int64_t N = n / nb;
  set_stage(MDLS_ST_INVERT);
  launch_invert<M>(st, N, nb, U, Vt, 1.0, nullptr, info_slot);
  // bwork = y (n entries)
  MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(n, 256), 256, 0, st>>>(n, 1, CMat{y, n, psy}, Mat{bwork, n, n}, 0));
  for (int64_t i = N - 1; i >= 0; --i) {
    set_stage(MDLS_ST_MULINV);
    launch_bs_mulinv<M>(st, nb, i, cm(Vt), bwork, n, x, psx);
    set_stage(MDLS_ST_BSUPDATE);
    if (i > 0) launch_bs_update<M>(st, nb, i, U, x, psx, bwork, n);
  }
}

}  // namespace mdls
