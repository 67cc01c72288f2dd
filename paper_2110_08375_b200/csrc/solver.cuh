// solver.cuh -- host drivers (launch sequences) behind the C-ABI of include/mdls.h.
//
// Algorithm 2 (blocked Householder QR) and Algorithm 1 (tiled back
// substitution) as stream-ordered kernel sequences: no host
// synchronisation, no allocation (the caller's workspace is carved up here), so
// a whole least-squares solve can be captured in one CUDA graph.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/mdls.h"
#include "launch.cuh"
#include "kern_misc.cuh"

namespace mdls {

// ---------------------------------------------------------------------------
// workspace plan (bytes, 256-aligned segments)
// ---------------------------------------------------------------------------
struct Plan {
  size_t af = 0, q = 0, y = 0, w = 0, beta = 0, s = 0, t = 0, x = 0, part = 0, v0 = 0, v1 = 0, v2 = 0, vt = 0, us = 0,
         flags = 0, hx = 0, info = 0, total = 0;
};

// md elements of one lane's split-K / stream-K partial buffer: kMaxSplit nb x max(M, K) partials, or the
// stream-K partials of two CTAs per SM (<= 64 x 64 dd / 32 x 32 qd / 32 x 16 od tiles: 8192 doubles) + flags
template <int M>
int64_t lane_part_elems(int64_t nb, int64_t mx) {
  return std::max<int64_t>(kMaxSplit * nb * mx, (int64_t)(2 * num_sms() + 8) * 8192 / M + 4096);
}

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
  if (op == MDLS_OP_LSTSQ || op == MDLS_OP_LSTSQ_NOQ) {
    p.af = take(md * Mr * K);
    p.hx = take(md * K);  // device x of a host-input solve (mdls_lstsq_host)
  }
  if (op == MDLS_OP_LSTSQ) p.q = take(md * Mr * Mr);
  if (qr_like) {
    p.y = take(md * Mr * K);
    p.w = take(md * Mr * K);
    p.beta = take(md * K);
    p.s = take(md * nb * nb);
    p.t = take(md * std::max<int64_t>(std::max<int64_t>(nb * nb, 1024), 32 * K));  // leaf T's (ld 32, column js)
  }
  if (op == MDLS_OP_APPLY_QT) p.y = take(md * Mr * K);
  if (qr_like || op == MDLS_OP_APPLY_QT) {
    p.x = take(5 * md * nb * mx);  // one GEMM-intermediate buffer per stream lane
    p.part = take(5 * md * lane_part_elems<M>(nb, mx));
  }
  p.v0 = take(md * mx);
  p.v1 = take(md * mx);
  p.v2 = take(md * mx);
  if (op == MDLS_OP_BACKSUB || op == MDLS_OP_LSTSQ || op == MDLS_OP_LSTSQ_NOQ) {
    p.vt = take(md * nb * K);
    p.us = take(md * nb * K);  // row-scaled diagonal tiles (tile inversion)
    p.flags = take(2 * sizeof(int) * (size_t)K);  // back-substitution dataflow counters (rows updated / x rows)
  }
  p.info = take(4 * sizeof(int));
  p.total = off;
  return p;
}


// ---------------------------------------------------------------------------
// Algorithm 2 on A (M x K), panels of width nb; fills Y (explicit), W, beta.
// ---------------------------------------------------------------------------
// per-stream GEMM scratch: intermediate X and split-K partials
struct Lane {
  cudaStream_t st;
  Mat X;          // nb x max(M, K) (also used as an M x nb operand)
  double* part;
  int64_t cap;
};

template <int M>
struct QrBufs {
  Mat Y, W;
  double* beta;
  Mat S, T, X;
  double* part;
  int64_t part_cap;
  int* info_slot;
  double* xbase;  // 5 lanes of X / part
  double* pbase;
  int64_t xcap;
  Lane lane(int i, cudaStream_t st) const {
    return Lane{st, Mat{xbase + (int64_t)i * xcap * M, X.ld, X.ps}, pbase + (int64_t)i * part_cap * M, part_cap};
  }
};

// Panel k of Algorithm 2: factor columns [j0, j0+nb) in leaves of
// B <= 16 columns (launch_leaf: v, beta, R, leaf T); after each leaf
//   W_s = -Y_s T_s                              (the leaf's P_WY = I + W_s Y_s^T)
//   C_s += Y_s (W_s^T C_s)  on the panel columns right of the leaf ("beta R^T v",
//                                                 "update R" as two md GEMMs)
//   W_s += W_<s (Y_<s^T W_s) (block form of z = -beta (v + W Y^T v))
// so the panel's W (P_WY = I + W Y^T) is built column block by block.
// The chain (leaf, W_s, in-panel update) runs on lane L0; the W-block
// recurrence, which nothing in the chain waits for, on lane L2 (may be L0).
template <int M>
cudaError_t qr_panel(const Lane& L0, const Lane& L2, int64_t Mr, int64_t nb, int64_t k, Mat A, Mat Y, Mat W,
                     double* beta, int64_t bps, const QrBufs<M>& b) {
  const int64_t j0 = k * nb, r = Mr - j0;
  int64_t js = j0;
  while (js < j0 + nb) {
    int bw = 1;
    set_stage(MDLS_ST_PANEL);
    Mat Tl{b.T.p, 32, 1024};  // leaf T, B <= 32
    cudaError_t e = launch_leaf<M>(L0.st, Mr, js, j0 + nb - js, A, Y, beta, bps, Tl, b.info_slot, &bw);
    if (e != cudaSuccess) return e;
    const int64_t rs = Mr - js;
    const CMat Ys = sub(cm(Y), js, js);
    Mat Ws = sub(W, js, js);
    set_stage(MDLS_ST_WY);
    gemm<M, false, false>(L0.st, rs, bw, bw, Ys, cm(Tl), Ws, 3, nullptr, 0);  // W_s = -Y_s T_s
    const int64_t rem = j0 + nb - (js + bw);
    if (rem > 0) {
      set_stage(MDLS_ST_PANEL);
      Mat Cs = sub(A, js, js + bw);
      gemm<M, true, false>(L0.st, bw, rem, rs, cm(Ws), cm(Cs), L0.X, 0, L0.part, L0.cap);
      gemm<M, false, false>(L0.st, rs, rem, bw, Ys, cm(L0.X), Cs, 1, nullptr, 0);
    }
    // L2's recurrence below rewrites W(:, js:js+bw) (it adds W_< (Y_<^T W_s) into W_s), so it may only
    // start once L0's in-panel product above has finished reading the leaf-local W_s
    if (js > j0 && L2.st != L0.st) {
      cudaEvent_t ev = pool_event();
      cudaEventRecord(ev, L0.st);
      cudaStreamWaitEvent(L2.st, ev, 0);
    }
    if (js > j0) {
      set_stage(MDLS_ST_WY);
      const int64_t np = js - j0;
      gemm<M, true, false>(L2.st, np, bw, rs, sub(cm(Y), js, j0), cm(Ws), L2.X, 0, L2.part, L2.cap);
      gemm<M, false, false>(L2.st, r, bw, np, sub(cm(W), j0, j0), cm(L2.X), sub(W, j0, js), 1, nullptr, 0);
    }
    js += bw;
  }
  return cudaGetLastError();
}

// apply panel k to the columns [c0, c1) of A: C += Y_k (W_k^T C) ("YWT * C", "R + YWTC")
template <int M>
void qr_apply_panel(const Lane& L, int64_t Mr, int64_t nb, int64_t k, CMat Yk, CMat Wk, Mat A, int64_t c0,
                    int64_t c1) {
  if (c1 <= c0) return;
  const int64_t j0 = k * nb, r = Mr - j0;
  set_stage(MDLS_ST_TRAILING);
  Mat Cm = sub(A, j0, c0);
  gemm<M, true, false>(L.st, nb, c1 - c0, r, Wk, cm(Cm), L.X, 0, L.part, L.cap);
  gemm<M, false, false>(L.st, r, c1 - c0, nb, Yk, cm(L.X), Cm, 1, nullptr, 0);
}

// forward Q accumulation step (the paper's Q = Q + Q W Y^T):
// Q(:, j0:) += (Q(:, j0:) W_k) Y_k^T
template <int M>
void form_q_forward_step(const Lane& L, int64_t Mr, int64_t nb, int64_t k, Mat Q, CMat Yk, CMat Wk) {
  const int64_t j0 = k * nb, r = Mr - j0;
  set_stage(MDLS_ST_FORM_Q);
  Mat Xq{L.X.p, Mr, Mr * nb};
  Mat Qs = sub(Q, 0, j0);
  gemm<M, false, false>(L.st, Mr, nb, r, cm(Qs), Wk, Xq, 0, L.part, L.cap);        // "Q * WY^T"
  gemm<M, false, true>(L.st, Mr, r, nb, cm(Xq), Yk, Qs, 1, nullptr, 0);            // "Q + QWY"
}

// Algorithm 2 with look-ahead over three streams: L0 carries the critical chain
// (panel k+1 starts as soon as panel k is applied to its columns), L1 the rest
// of the trailing update and the forward Q accumulation, L2 the W-block
// recurrence.  Q (nullable) is formed forward on L1 when q_forward, else the
// caller forms it backward afterwards.  All streams are joined into L0.
template <int M>
cudaError_t qr_factor_overlap(const Lane& L0, const Lane& L1, const Lane& L2, int64_t Mr, int64_t K, int64_t nb,
                              Mat A, const QrBufs<M>& b, Mat* Qf) {
  auto fork = [](cudaStream_t from, cudaStream_t to) {
    if (from == to) return;
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, from);
    cudaStreamWaitEvent(to, ev, 0);
  };
  fork(L0.st, L1.st);
  fork(L0.st, L2.st);
  if (Qf) {
    set_stage(MDLS_ST_FORM_Q);
    MDLS_LAUNCH(F_MISC, L1.st, set_identity_kernel<M><<<grid_for(Mr * Mr, 256), 256, 0, L1.st>>>(Mr, Mr, *Qf));
  }
  const int64_t N = K / nb;
  cudaEvent_t trail_done = nullptr;  // L1: trailing update of the previous panel finished
  cudaError_t e = cudaSuccess;
  for (int64_t k = 0; k < N; ++k) {
    const int64_t j0 = k * nb;
    e = qr_panel<M>(L0, L2, Mr, nb, k, A, b.Y, b.W, b.beta, K, b);
    if (e != cudaSuccess) break;
    fork(L0.st, L2.st);  // W_k complete on L2 after this point
    cudaEvent_t wk = pool_event();
    cudaEventRecord(wk, L2.st);
    const CMat Yk = sub(cm(b.Y), j0, j0), Wk = sub(cm(b.W), j0, j0);
    if (k + 1 < N) {
      cudaStreamWaitEvent(L0.st, wk, 0);
      if (trail_done) cudaStreamWaitEvent(L0.st, trail_done, 0);  // panel k+1's columns had panel k-1 applied
      qr_apply_panel<M>(L0, Mr, nb, k, Yk, Wk, A, j0 + nb, j0 + 2 * nb);  // look-ahead
    }
    cudaStreamWaitEvent(L1.st, wk, 0);
    qr_apply_panel<M>(L1, Mr, nb, k, Yk, Wk, A, j0 + 2 * nb, K);
    trail_done = pool_event();
    cudaEventRecord(trail_done, L1.st);
    if (Qf) form_q_forward_step<M>(L1, Mr, nb, k, *Qf, Yk, Wk);
  }
  fork(L1.st, L0.st);  // joined even on an error (a caller's graph capture must not stay forked)
  fork(L2.st, L0.st);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Algorithm 2 as a chain of leaves (every leaf a register-leaf cluster kernel
// that first applies the previous leaf to its own columns), with the trailing
// update split by distance.  Streams (all forked from and joined into `st`):
//   Lc (high priority): the leaves -- the only serial path of the factorisation;
//   La (high): per leaf s of panel k, C += Y_s X, X = -T_s^T (Y_s^T C), on the
//       columns beyond leaf s+1 up to the end of panel k+1 (leaf s+2 waits on it);
//   Lf (high): the same leaf update on the columns of panel k+2, one panel behind
//       in its dependencies (it waits for panel k-1's product below);
//   Lw (high): the panel's W (the block recurrence W_s += W_<s (Y_<s^T W_s));
//   Lb (high): once W_k is complete, panel k's update of every column beyond
//       panel k+2 as one k = nb product C += Y_k (W_k^T C) ("YWT * C",
//       "R + YWTC"), the columns of panel k+3 first;
//   Lq (low): the forward Q accumulation Q(:, j0:) += (Q(:, j0:) W_k) Y_k^T per
//       completed panel when Qf is given, on a capped number of CTAs
//       (GemmCap) so that the chain's updates always find free CTA slots.
// Every (reflector, column) pair is applied exactly once and every column sees
// the reflectors in Algorithm 2's order: a column of panel k+3 gets panels <= k
// through Lb, then panel k+1's leaves through Lf, panel k+2's through La, then
// its own panel's leaves (in-leaf and the next leaf's prologue).
// ---------------------------------------------------------------------------
template <int M>
bool chain_supported(int64_t Mr, int64_t K, int64_t nb) {
  int prevB = 0;
  for (int64_t js = 0; js < K;) {
    const int64_t j0 = (js / nb) * nb;
    const int B = chain_leaf_width<M>(Mr, js, j0 + nb - js);
    if (B == 0 || (prevB && prevB != B)) return false;
    prevB = B;
    js += B;
  }
  return true;
}

template <int M>
cudaError_t qr_factor_chain(cudaStream_t st, int64_t Mr, int64_t K, int64_t nb, Mat A, const QrBufs<M>& b, Mat Tall,
                            Mat* Qf, const cudaEvent_t* panel_ready = nullptr) {
  auto fork = [](cudaStream_t from, cudaStream_t to) {
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, from);
    cudaStreamWaitEvent(to, ev, 0);
  };
  cudaStream_t Lc = side_stream(0), Las = side_stream(1), Lws = side_stream(2), Lqs = side_stream(3),
               Lbs = side_stream(4), Lfs = side_stream(5);
  const Lane La = b.lane(0, Las), Lw = b.lane(1, Lws), Lq = b.lane(2, Lqs), Lb = b.lane(3, Lbs), Lf = b.lane(4, Lfs);
  for (cudaStream_t q : {Lc, Las, Lws, Lqs, Lbs, Lfs}) fork(st, q);
  // host-input solves (mdls_lstsq_host): column panel p of A arrives by its own copy, recorded in panel_ready[p];
  // each lane waits for the panels it is about to touch, once (the leaf chain for its panel, the near window up
  // to its last column, the far window for panel k+2, the panel products for all of A)
  const int64_t NP = cdiv(K, nb);
  std::vector<int64_t> panels_seen(8, -1);
  auto need = [&](int lane_id, cudaStream_t q, int64_t last_col) {
    if (!panel_ready || last_col < 0) return;
    const int64_t pidx = std::min<int64_t>(NP - 1, last_col / nb);
    for (int64_t t = panels_seen[(size_t)lane_id] + 1; t <= pidx; ++t) cudaStreamWaitEvent(q, panel_ready[t], 0);
    panels_seen[(size_t)lane_id] = std::max(panels_seen[(size_t)lane_id], pidx);
  };
  if (Qf) {
    set_stage(MDLS_ST_FORM_Q);
    MDLS_LAUNCH(F_MISC, Lqs, set_identity_kernel<M><<<grid_for(Mr * Mr, 256), 256, 0, Lqs>>>(Mr, Mr, *Qf));
  }
  std::vector<int64_t> jss;
  std::vector<int> Bs;
  for (int64_t js = 0; js < K;) {
    const int64_t j0 = (js / nb) * nb;
    const int B = chain_leaf_width<M>(Mr, js, j0 + nb - js);
    jss.push_back(js);
    Bs.push_back(B);
    js += B;
  }
  const int ns = (int)jss.size();
  const int64_t N = K / nb;
  // MDLS_DEFER=0: every leaf updates all trailing columns itself (no panel-level product)
  static const bool defer = [] {
    const char* v = getenv("MDLS_DEFER");
    return !(v && v[0] == '0');
  }();
  // CTAs of the forward-Q products: by default one per SM outside the leaf's cluster (MDLS_QCAP)
  static const int64_t qcap_env = [] {
    const char* v = getenv("MDLS_QCAP");
    return (int64_t)(v ? atoll(v) : -1);
  }();
  const int64_t qcap = qcap_env >= 0 ? qcap_env : std::max<int64_t>(1, num_sms() - leaf_cluster_size());
  // CTAs of the panel products (Lb): MDLS_BCAP
  static const int64_t bcap_env = [] {
    const char* v = getenv("MDLS_BCAP");
    return (int64_t)(v ? atoll(v) : -1);
  }();
  const int64_t bcap = bcap_env >= 0 ? bcap_env : 0;
  std::vector<cudaEvent_t> ev_apply((size_t)ns, nullptr);
  std::vector<cudaEvent_t> ev_bulk_a((size_t)N, nullptr);  // Lb: panel k applied to the columns of panel k+3
  std::vector<cudaEvent_t> ev_far((size_t)N, nullptr);     // Lf: panel k applied to the columns of panel k+2
  // MDLS_TIMELINE=1 (debug, not graph-capturable): per-leaf start/end and apply-end times, printed
  static const bool timeline = getenv("MDLS_TIMELINE") != nullptr;
  std::vector<cudaEvent_t> tl_ls, tl_le, tl_ae;
  cudaEvent_t tl0 = nullptr;
  auto tl_ev = [](cudaStream_t q) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, q);
    return e;
  };
  if (timeline) tl0 = tl_ev(Lc);
  // leaf s's update C += Y_s X, X = -T_s^T (Y_s^T C), of the columns [c0, c1)
  auto leaf_update = [&](const Lane& L, int s, int64_t c0, int64_t c1) {
    if (c0 >= c1) return;
    const int64_t js = jss[(size_t)s];
    const int B = Bs[(size_t)s];
    set_stage(MDLS_ST_TRAILING);
    const Mat Cm = sub(A, js, c0);
    const Mat Xb{L.X.p, B, L.X.ps};
    const Mat Ts{Tall.p + js * 32, 32, Tall.ps};
    leaf_t_product<M>(L.st, B, c1 - c0, Mr - js, sub(cm(b.Y), js, js), cm(Ts), cm(Cm), Xb, L.part, L.cap);
    gemm<M, false, false>(L.st, Mr - js, c1 - c0, B, sub(cm(b.Y), js, js), cm(Xb), Cm, 1, nullptr, 0);
  };
  cudaError_t err = cudaSuccess;
  for (int s = 0; s < ns && err == cudaSuccess; ++s) {
    const int64_t js = jss[(size_t)s];
    const int B = Bs[(size_t)s];
    const int64_t k = js / nb, j0 = k * nb, r = Mr - js;
    const bool first_in_panel = js == j0, last_in_panel = js + B == j0 + nb;
    const Mat Ts{Tall.p + js * 32, 32, Tall.ps};
    cudaEvent_t ev_leaf = pool_event();
    // Lc: leaf s (its prologue applies leaf s-1 to its own columns); leaf s-2 must have been applied to
    // every column beyond leaf s-1 (La) first, and panel k-2 to this panel (Lf)
    if (s >= 2) cudaStreamWaitEvent(Lc, ev_apply[(size_t)s - 2], 0);
    if (defer && first_in_panel && k >= 2 && ev_far[(size_t)k - 2]) cudaStreamWaitEvent(Lc, ev_far[(size_t)k - 2], 0);
    if (timeline) tl_ls.push_back(tl_ev(Lc));
    set_stage(MDLS_ST_PANEL);
    const Mat Tp = s > 0 ? Mat{Tall.p + jss[(size_t)s - 1] * 32, 32, Tall.ps} : Mat{nullptr, 0, 0};
    need(0, Lc, js + B - 1);
    err = launch_leaf_chain<M>(Lc, Mr, js, B, A, b.Y, b.beta, K, Ts, b.info_slot, Tp, s > 0 ? jss[(size_t)s - 1] : -1);
    if (err != cudaSuccess) break;
    cudaEventRecord(ev_leaf, Lc);
    if (timeline) tl_le.push_back(tl_ev(Lc));
    const int64_t c0 = (s + 1 < ns) ? jss[(size_t)s + 1] + Bs[(size_t)s + 1] : K;
    // La: the near window, up to the end of panel k+1 (everything without deferral).  Panel k+1 has had
    // panel k-1 applied by Lf (the first leaf of the panel waits for it; La is in order after that)
    cudaStreamWaitEvent(Las, ev_leaf, 0);
    if (defer && first_in_panel && k >= 1 && ev_far[(size_t)k - 1]) cudaStreamWaitEvent(Las, ev_far[(size_t)k - 1], 0);
    const int64_t c1 = defer ? std::min<int64_t>(K, (k + 2) * nb) : K;
    if (c0 < c1) need(1, Las, c1 - 1);
    leaf_update(La, s, c0, c1);
    ev_apply[(size_t)s] = pool_event();
    cudaEventRecord(ev_apply[(size_t)s], Las);
    if (timeline) tl_ae.push_back(tl_ev(Las));
    // Lf: panel k+2's columns, after panel k-1's product reached them (Lb)
    if (defer && (k + 2) * nb < K) {
      cudaStreamWaitEvent(Lfs, ev_leaf, 0);
      if (first_in_panel && k >= 1 && ev_bulk_a[(size_t)k - 1]) cudaStreamWaitEvent(Lfs, ev_bulk_a[(size_t)k - 1], 0);
      need(5, Lfs, std::min<int64_t>(K, (k + 3) * nb) - 1);
      leaf_update(Lf, s, std::max<int64_t>(c0, (k + 2) * nb), std::min<int64_t>(K, (k + 3) * nb));
    }
    if (defer && last_in_panel) {
      ev_far[(size_t)k] = pool_event();
      cudaEventRecord(ev_far[(size_t)k], Lfs);
    }
    // Lw: the panel's W, column block js..js+B-1
    cudaStreamWaitEvent(Lws, ev_leaf, 0);
    set_stage(MDLS_ST_WY);
    gemm<M, false, false>(Lws, r, B, B, sub(cm(b.Y), js, js), cm(Ts), sub(b.W, js, js), 3, nullptr, 0);
    if (js > j0) {
      const int64_t np = js - j0;
      gemm<M, true, false>(Lws, np, B, r, sub(cm(b.Y), js, j0), sub(cm(b.W), js, js), Lw.X, 0, Lw.part, Lw.cap);
      gemm<M, false, false>(Lws, Mr - j0, B, np, sub(cm(b.W), j0, j0), cm(Lw.X), sub(b.W, j0, js), 1, nullptr, 0);
    }
    if (last_in_panel || s == ns - 1) {
      const CMat Yk = sub(cm(b.Y), j0, j0), Wk = sub(cm(b.W), j0, j0);
      // Lb: panel k applied to the columns beyond panel k+2 (W_k complete on Lw)
      const int64_t cb = (k + 3) * nb;
      if (defer && cb < K) {
        fork(Lws, Lbs);
        need(4, Lbs, K - 1);
        GemmCap cap(bcap);
        const int64_t cm1 = std::min<int64_t>(K, cb + nb);
        qr_apply_panel<M>(Lb, Mr, nb, k, Yk, Wk, A, cb, cm1);
        ev_bulk_a[(size_t)k] = pool_event();
        cudaEventRecord(ev_bulk_a[(size_t)k], Lbs);
        qr_apply_panel<M>(Lb, Mr, nb, k, Yk, Wk, A, cm1, K);
      }
      if (Qf) {
        fork(Lws, Lqs);
        GemmCap cap(qcap);
        form_q_forward_step<M>(Lq, Mr, nb, k, *Qf, Yk, Wk);
      }
    }
  }
  // join every side stream even on an error, so a caller's graph capture is never left forked
  for (cudaStream_t q : {Lc, Las, Lws, Lqs, Lbs, Lfs}) fork(q, st);
  if (err != cudaSuccess) return err;
  if (timeline) {
    cudaEvent_t tw = tl_ev(Lws), tq = tl_ev(Lqs), tb = tl_ev(Lbs), tf = tl_ev(Lfs);
    cudaDeviceSynchronize();
    float t;
    for (size_t s = 0; s < tl_ae.size(); ++s) {
      float a0 = 0, a1 = 0, a2 = 0;
      if (s < tl_ls.size()) cudaEventElapsedTime(&a0, tl0, tl_ls[s]);
      if (s < tl_le.size()) cudaEventElapsedTime(&a1, tl0, tl_le[s]);
      cudaEventElapsedTime(&a2, tl0, tl_ae[s]);
      printf("leaf %3zu start %8.1f end %8.1f (%6.1f us)  apply end %8.1f us\n", s, a0 * 1e3, a1 * 1e3,
             (a1 - a0) * 1e3, a2 * 1e3);
    }
    const char* names[4] = {"W", "Q", "panel-update", "far-window"};
    cudaEvent_t evs[4] = {tw, tq, tb, tf};
    for (int i = 0; i < 4; ++i) {
      cudaEventElapsedTime(&t, tl0, evs[i]);
      printf("%s stream end %8.1f us\n", names[i], t * 1e3);
    }
  }
  return cudaGetLastError();
}

template <int M>
cudaError_t qr_factor(cudaStream_t st, int64_t Mr, int64_t K, int64_t nb, Mat A, const QrBufs<M>& b, int64_t kbeg,
                      int64_t kend, bool trailing) {
  const Lane L = b.lane(0, st);
  for (int64_t k = kbeg; k < kend; ++k) {
    const int64_t j0 = k * nb;
    cudaError_t e = qr_panel<M>(L, L, Mr, nb, k, A, b.Y, b.W, b.beta, K, b);
    if (e != cudaSuccess) return e;
    if (trailing) qr_apply_panel<M>(L, Mr, nb, k, sub(cm(b.Y), j0, j0), sub(cm(b.W), j0, j0), A, j0 + nb, K);
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
    const Lane L = b.lane(0, st);
    gemm<M, true, false>(st, nb, r, r, Yp, cm(Qs), L.X, 0, L.part, L.cap);
    gemm<M, false, false>(st, r, r, nb, Wp, cm(L.X), Qs, 1, nullptr, 0);
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

// Algorithm 1: U x = y (leading n x n of U), N = n/nb tiles.
// The tile inverses are computed in chunks of tiles, bottom first, on a
// low-priority side stream; the chain i = N..1 (x_i = U_i^-1 b_i, then
// b_j -= A_ji x_i for all j < i in one launch: the paper's "simultaneously
// update") runs on a high-priority side stream and starts as soon
// as the bottom chunk is inverted.
template <int M>
void backsub(cudaStream_t st, int64_t n, int64_t nb, CMat U, const double* y, int64_t psy, double* x, int64_t psx,
             Mat Vt, Mat Us, double* bwork, int* info_slot, int* flags) {
  const int64_t N = n / nb;
  cudaStream_t sinv = side_stream(3), sch = side_stream(0);
  auto fork = [](cudaStream_t from, cudaStream_t to) {
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, from);
    cudaStreamWaitEvent(to, ev, 0);
  };
  fork(st, sinv);
  fork(st, sch);
  set_stage(MDLS_ST_INVERT);
  static const int64_t chunk_env = [] {
    const char* v = getenv("MDLS_INV_CHUNK");
    return (int64_t)(v ? atoi(v) : 16);  // tiles per inversion launch, bottom first (0: all in one launch)
  }();
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(N, chunk_env > 0 ? chunk_env : N));
  std::vector<cudaEvent_t> inv_ready((size_t)N, nullptr);
  // bottom-first chunks growing 2, 4, 8, ... up to `chunk` tiles: the chain's first step waits only for a
  // two-tile inversion, later chunks finish ahead of the chain
  int64_t step = std::min<int64_t>(chunk, 2);
  for (int64_t hi = N; hi > 0; hi -= step, step = std::min<int64_t>(chunk, 2 * step)) {
    const int64_t lo = std::max<int64_t>(0, hi - step);
    launch_invert<M>(sinv, hi - lo, nb, sub(U, lo * nb, lo * nb), sub(Vt, 0, lo * nb), sub(Us, 0, lo * nb), info_slot,
                     lo * nb);
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, sinv);
    for (int64_t t = lo; t < hi; ++t) inv_ready[(size_t)t] = ev;
  }
  // dataflow counters (bs_flow_ok): rows of tile j updated so far / entries of x_i written
  BsFlow fl{nullptr, nullptr, N};
  if (flags && bs_flow_ok<M>(n, nb)) {
    fl.rows = flags;
    fl.xrdy = flags + N;
    cudaMemsetAsync(flags, 0, sizeof(int) * 2 * (size_t)N, sch);
  }
  // bwork = y (n entries)
  MDLS_LAUNCH(F_MISC, sch, copy_kernel<M><<<grid_for(n, 256), 256, 0, sch>>>(n, 1, CMat{y, n, psy}, Mat{bwork, n, n}, 0));
  cudaEvent_t waited = nullptr;
  for (int64_t i = N - 1; i >= 0; --i) {
    if (inv_ready[(size_t)i] != waited) {
      cudaStreamWaitEvent(sch, inv_ready[(size_t)i], 0);
      waited = inv_ready[(size_t)i];
    }
    set_stage(MDLS_ST_MULINV);
    launch_bs_mulinv<M>(sch, nb, i, cm(Vt), bwork, n, x, psx, fl, i == N - 1);
    set_stage(MDLS_ST_BSUPDATE);
    if (i >= 1) launch_bs_update<M>(sch, nb, i, 0, i * nb, U, x, psx, bwork, n, fl);
  }
  fork(sinv, st);
  fork(sch, st);
}

}  // namespace mdls
