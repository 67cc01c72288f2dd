// api.cuh -- the extern "C" entry points of include/mdls.h for one precision.
// Included by api_dd.cu / api_qd.cu / api_od.cu with MDLS_P (dd|qd|od) and
// MDLS_M (2|4|8) defined; argument checking, workspace carving, launches.
#pragma once
#include <cstdlib>

#include "solver.cuh"

#define MDLS_CAT2(a, b) a##b
#define MDLS_CAT(a, b) MDLS_CAT2(a, b)
#define MDLS_FN(name) MDLS_CAT(name, MDLS_P)

namespace mdls {
namespace api_impl {

constexpr int M = MDLS_M;

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int launched() { return cudaGetLastError() == cudaSuccess ? 0 : MDLS_ERR_CUDA; }

template <typename T>
inline T* at(void* work, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(work) + off);
}

// plane strides must cover the operand
inline bool mat_ok(const void* p, int64_t rows, int64_t cols, int64_t ld, int64_t ps) {
  return p && ld >= std::max<int64_t>(1, rows) && ps >= ld * cols;
}

// Q formation order: forward (Q += (Q W_k) Y_k^T after each panel, overlapping the
// factorisation; 1.4x the md pairs of backward at M = K) for dd, where the panel
// chain bounds the solve; backward for qd/od, which are GEMM bound.  MDLS_QFORM =
// forward|backward overrides.
template <int MM>
inline bool q_forward() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MDLS_QFORM");
    if (e && e[0] == 'f') v = 1;
    else if (e && e[0] == 'b') v = 0;
    else v = (MM <= 2) ? 1 : 0;
  }
  return v == 1;
}

// chained-leaf factorisation (solver.cuh::qr_factor_chain) where every leaf fits the register
// leaf; MDLS_CHAIN=0 forces the GEMM-chained panel path
template <int MM>
inline bool use_chain(int64_t Mr, int64_t K, int64_t nb) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MDLS_CHAIN");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1 && chain_supported<MM>(Mr, K, nb);
}

inline int tile_ok(int64_t Mr, int64_t K, int64_t nb) {
  if (K < 1) return -2;
  if (Mr < K) return -1;
  if (nb < 1 || nb > 256 || K % nb != 0) return -3;
  return 0;
}

}  // namespace api_impl
}  // namespace mdls

using namespace mdls;
using namespace mdls::api_impl;

extern "C" {

// the complex problem's workspace: the real embedding (2M x 2K), its right-hand side and solution, then the
// plan of the embedded real least-squares problem
static size_t zplan_bytes(int64_t Mr, int64_t K, int64_t nb, int form_q, size_t* emb) {
  const size_t md = sizeof(double) * M;
  *emb = align256(md * 4 * Mr * K) + align256(md * 2 * Mr) + align256(md * 2 * K);
  return *emb + make_plan<M>(form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ, 2 * Mr, 2 * K, nb).total;
}

size_t MDLS_FN(mdls_workspace_)(int op, int64_t Mr, int64_t K, int64_t nb) {
  if (op == MDLS_OP_ZLSTSQ) {
    if (tile_ok(2 * Mr, 2 * K, nb) || Mr < K) return 0;
    size_t emb;
    return zplan_bytes(Mr, K, nb, 1, &emb);
  }
  if (op == MDLS_OP_BACKSUB) {
    if (K < 1 || nb < 1 || nb > 256 || K % nb) return 0;
    return make_plan<M>(op, K, K, nb).total;
  }
  if (tile_ok(Mr, K, nb)) return 0;
  return make_plan<M>(op, Mr, K, nb).total;
}

int MDLS_FN(mdls_md_op_)(int op, int64_t n, const double* a, const double* b, double* c, int64_t ps, void* stream) {
  if (op < 0 || op > 9) return -1;
  if (n < 0) return -2;
  if (n == 0) return 0;
  if (!a) return -3;
  if (!b && (op < 4 || op == 7)) return -4;
  if (!c) return -5;
  if (ps < n) return -6;
  if (op >= 7)
    MDLS_LAUNCH(F_MISC, S(stream), md_op_warp_kernel<M><<<grid_for(32 * n, 128), 128, 0, S(stream)>>>(op, n, a, b, c, ps));
  else
    MDLS_LAUNCH(F_MISC, S(stream), md_op_kernel<M><<<grid_for(n, 128), 128, 0, S(stream)>>>(op, n, a, b, c, ps));
  return launched();
}

int MDLS_FN(mdls_invert_tiles_)(int64_t n, int64_t nb, const double* U, int64_t ldu, int64_t psu, double* Vt,
                                int64_t ldv, int64_t psv, int* dev_info, void* stream) {
  if (n < 1) return -1;
  if (nb < 1 || nb > 256 || n % nb) return -2;
  if (!mat_ok(U, n, n, ldu, psu)) return -3;
  if (!mat_ok(Vt, nb, n, ldv, psv)) return -6;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  int* slot = nullptr;
  if (dev_info) {
    slot = dev_info;
    MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(slot));
  } else {
    return -9;
  }
  launch_invert<M>(st, n / nb, nb, CMat{U, ldu, psu}, Mat{Vt, ldv, psv}, Mat{nullptr, 0, 0}, slot, 0);
  MDLS_LAUNCH(F_MISC, st, info_finish_kernel<<<1, 1, 0, st>>>(slot, nullptr, dev_info));
  return launched();
}

int MDLS_FN(mdls_backsub_)(int64_t n, int64_t nb, const double* U, int64_t ldu, int64_t psu, const double* y,
                           int64_t psy, double* x, int64_t psx, void* work, size_t work_bytes, int* dev_info,
                           void* stream) {
  if (n < 1) return -1;
  if (nb < 1 || nb > 256 || n % nb) return -2;
  if (!mat_ok(U, n, n, ldu, psu)) return -3;
  if (!y || psy < n) return -6;
  if (!x || psx < n) return -8;
  const Plan p = make_plan<M>(MDLS_OP_BACKSUB, n, n, nb);
  if (!work || work_bytes < p.total) return -10;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  int* slot = at<int>(work, p.info);
  MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(slot));
  backsub<M>(st, n, nb, CMat{U, ldu, psu}, y, psy, x, psx, Mat{at<double>(work, p.vt), nb, nb * n},
             Mat{at<double>(work, p.us), nb, nb * n}, at<double>(work, p.v0), slot, at<int>(work, p.flags));
  if (dev_info) MDLS_LAUNCH(F_MISC, st, info_finish_kernel<<<1, 1, 0, st>>>(slot, nullptr, dev_info));
  return launched();
}

static QrBufs<M> qr_bufs(void* work, const Plan& p, int64_t Mr, int64_t K, int64_t nb, double* W, int64_t ldw,
                         int64_t psw) {
  QrBufs<M> b;
  b.Y = Mat{at<double>(work, p.y), Mr, Mr * K};
  b.W = W ? Mat{W, ldw, psw} : Mat{at<double>(work, p.w), Mr, Mr * K};
  b.beta = at<double>(work, p.beta);
  b.S = Mat{at<double>(work, p.s), nb, nb * nb};
  b.T = Mat{at<double>(work, p.t), nb, nb * nb};
  const int64_t mx = std::max(Mr, K);
  b.X = Mat{at<double>(work, p.x), nb, nb * mx};
  b.part = at<double>(work, p.part);
  b.part_cap = lane_part_elems<M>(nb, mx);
  b.xbase = b.X.p;
  b.pbase = b.part;
  b.xcap = nb * mx;
  b.info_slot = at<int>(work, p.info);
  return b;
}

// host-resident inputs / output of mdls_lstsq_host_<p> (pinned, limb-planar)
struct HostIO {
  const double* A;
  int64_t lda, psa;
  const double* b;
  int64_t psb;
  double* x;
  int64_t psx;
  const double* A_dev;  // A's device-visible address when its pinned pages are mapped (UVA), else NULL
};
// device-visible address of page-locked, mapped host memory (NULL for pageable memory)
static const double* mapped_ptr(const double* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (at.type == cudaMemoryTypeHost && at.devicePointer) ? static_cast<const double*>(at.devicePointer) : nullptr;
}

// the whole least-squares pipeline of one problem on stream st (arguments already checked).  With hio the
// inputs come from host memory: b first, then A column panel by column panel on a copy stream (one event
// per panel), so the leaf chain starts on panel 0 while the rest of A is still crossing PCIe, and x is copied
// back at the end -- the host<->device transfers overlap the factorisation instead of preceding it.
static int lstsq_run(cudaStream_t st, int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                     const double* b, int64_t psb, double* x, int64_t psx, int form_q, double* R_out, int64_t ldr,
                     int64_t psr, double* Q_out, int64_t ldq, int64_t psq, double* y_out, int64_t psy, void* work,
                     int* dev_info, const HostIO* hio = nullptr) {
  const int op = form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ;
  const Plan p = make_plan<M>(op, Mr, K, nb);
  set_stage(MDLS_NSTAGES);
  QrBufs<M> bb = qr_bufs(work, p, Mr, K, nb, nullptr, 0, 0);
  int* pre = bb.info_slot + 2;
  auto fork = [](cudaStream_t from, cudaStream_t to) {
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, from);
    cudaStreamWaitEvent(to, ev, 0);
  };
  MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(bb.info_slot));
  MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(bb.info_slot + 1));
  MDLS_LAUNCH(F_MISC, st, int_set_kernel<<<1, 1, 0, st>>>(pre, 0));
  // factor a copy of A
  Mat Af{at<double>(work, p.af), Mr, Mr * K};
  const int64_t NP = cdiv(K, nb);
  std::vector<cudaEvent_t> ready;
  cudaStream_t cs = nullptr;
  if (hio) {
    double* bdev = at<double>(work, p.v2);
    for (int l = 0; l < M; ++l)
      cudaMemcpyAsync(bdev + l * Mr, hio->b + l * hio->psb, sizeof(double) * Mr, cudaMemcpyHostToDevice, st);
    b = bdev;
    psb = Mr;
    x = at<double>(work, p.hx);
    psx = K;
    cs = side_stream(7);
    fork(st, cs);  // the previous call's use of Af is over
    ready.resize((size_t)NP);
    for (int64_t t = 0; t < NP; ++t) {
      const int64_t c0 = t * nb, nc = std::min<int64_t>(K, c0 + nb) - c0;
      if (hio->A_dev) {
        // zero-copy: a copy kernel on 64 CTAs reads the mapped pinned pages over PCIe (a kernel node overlaps the
        // factorisation's kernels inside a CUDA graph, where copy-engine nodes were measured not to)
        MDLS_LAUNCH(F_MISC, cs, copy_kernel<M><<<64, 256, 0, cs>>>(Mr, nc, CMat{hio->A_dev + c0 * hio->lda, hio->lda,
                                                                               hio->psa}, sub(Af, 0, c0), 0));
      } else {
        for (int l = 0; l < M; ++l) {
          if (hio->lda == Mr)  // the panel of one limb plane is contiguous on both sides: one linear copy
            cudaMemcpyAsync(Af.p + l * Af.ps + c0 * Mr, hio->A + l * hio->psa + c0 * Mr, sizeof(double) * Mr * nc,
                            cudaMemcpyHostToDevice, cs);
          else
            cudaMemcpy2DAsync(Af.p + l * Af.ps + c0 * Mr, sizeof(double) * Mr, hio->A + l * hio->psa + c0 * hio->lda,
                              sizeof(double) * hio->lda, sizeof(double) * Mr, nc, cudaMemcpyHostToDevice, cs);
        }
      }
      ready[(size_t)t] = pool_event();
      cudaEventRecord(ready[(size_t)t], cs);
    }
    MDLS_LAUNCH(F_MISC, cs, finite_check_kernel<M><<<grid_for(Mr * K, 256), 256, 0, cs>>>(Mr, K, cm(Af), pre));
  } else {
    MDLS_LAUNCH(F_MISC, st, finite_check_kernel<M><<<grid_for(Mr * K, 256), 256, 0, st>>>(Mr, K, CMat{A, lda, psa}, pre));
    MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(Mr * K, 256), 256, 0, st>>>(Mr, K, CMat{A, lda, psa}, Af, 0));
  }
  MDLS_LAUNCH(F_MISC, st, finite_check_kernel<M><<<grid_for(Mr, 256), 256, 0, st>>>(Mr, 1, CMat{b, Mr, psb}, pre));
  cudaMemsetAsync(bb.Y.p, 0, sizeof(double) * M * Mr * K, st);
  cudaMemsetAsync(bb.W.p, 0, sizeof(double) * M * Mr * K, st);
  Mat Q = (form_q && Q_out) ? Mat{Q_out, ldq, psq} : Mat{form_q ? at<double>(work, p.q) : nullptr, Mr, Mr * Mr};
  const bool fwd = form_q && q_forward<M>();
  if (use_chain<M>(Mr, K, nb)) {
    if (qr_factor_chain<M>(st, Mr, K, nb, Af, bb, Mat{at<double>(work, p.t), 32, 32 * std::max<int64_t>(K, 32)},
                           fwd ? &Q : nullptr, hio ? ready.data() : nullptr) != cudaSuccess) {
      if (cs) fork(cs, st);
      return MDLS_ERR_CUDA;
    }
  } else {
    if (cs) fork(cs, st);  // the GEMM-chained path takes A whole
    if (qr_factor_overlap<M>(bb.lane(0, st), bb.lane(1, side_stream(0)), bb.lane(2, side_stream(1)), Mr, K, nb, Af,
                             bb, fwd ? &Q : nullptr) != cudaSuccess)
      return MDLS_ERR_CUDA;
  }
  if (cs) fork(cs, st);  // the copies and A's finite check are done before the info is read
  double* yv = at<double>(work, p.v1);
  if (form_q) {
    if (!fwd) form_q_backward<M>(st, Mr, K, nb, Q, bb);
    set_stage(MDLS_ST_QTB);
    gemm<M, true, false>(st, Mr, 1, Mr, cm(Q), CMat{b, Mr, psb}, Mat{yv, Mr, Mr}, 0, bb.part, bb.part_cap);
  } else {
    MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(Mr, 256), 256, 0, st>>>(Mr, 1, CMat{b, Mr, psb}, Mat{yv, Mr, Mr}, 0));
    apply_qt_panels<M>(st, Mr, K, nb, cm(bb.Y), cm(bb.W), Mat{yv, Mr, Mr}, bb.X, bb.part, bb.part_cap);
  }
  backsub<M>(st, K, nb, cm(Af), yv, Mr, x, psx, Mat{at<double>(work, p.vt), nb, nb * K},
             Mat{at<double>(work, p.us), nb, nb * K}, at<double>(work, p.v0), bb.info_slot, at<int>(work, p.flags));
  set_stage(MDLS_NSTAGES);
  if (R_out) MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(Mr * K, 256), 256, 0, st>>>(Mr, K, cm(Af), Mat{R_out, ldr, psr}, 1));
  if (y_out) MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(Mr, 256), 256, 0, st>>>(Mr, 1, CMat{yv, Mr, Mr}, Mat{y_out, Mr, psy}, 0));
  if (dev_info) MDLS_LAUNCH(F_MISC, st, info_finish_kernel<<<1, 1, 0, st>>>(bb.info_slot, pre, dev_info));
  if (hio)
    for (int l = 0; l < M; ++l)
      cudaMemcpyAsync(hio->x + l * hio->psx, x + l * psx, sizeof(double) * K, cudaMemcpyDeviceToHost, st);
  return launched();
}

int MDLS_FN(mdls_qr_)(int64_t Mr, int64_t K, int64_t nb, double* A, int64_t lda, int64_t psa, double* Q, int64_t ldq,
                      int64_t psq, double* W, int64_t ldw, int64_t psw, void* work, size_t work_bytes, int* dev_info,
                      void* stream) {
  if (int e = tile_ok(Mr, K, nb)) return e;
  if (!mat_ok(A, Mr, K, lda, psa)) return -4;
  if (Q && !mat_ok(Q, Mr, Mr, ldq, psq)) return -7;
  if (W && !mat_ok(W, Mr, K, ldw, psw)) return -10;
  const Plan p = make_plan<M>(MDLS_OP_QR, Mr, K, nb);
  if (!work || work_bytes < p.total) return -14;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  QrBufs<M> b = qr_bufs(work, p, Mr, K, nb, W, ldw, psw);
  MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(b.info_slot));
  MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(b.info_slot + 1));
  cudaMemsetAsync(b.Y.p, 0, sizeof(double) * M * Mr * K, st);
  if (W) {
    for (int l = 0; l < M; ++l) cudaMemset2DAsync(W + l * psw, sizeof(double) * ldw, 0, sizeof(double) * Mr, K, st);
  } else {
    cudaMemsetAsync(b.W.p, 0, sizeof(double) * M * Mr * K, st);
  }
  Mat Am{A, lda, psa};
  Mat Qm{Q, ldq, psq};
  const bool fwd = Q && q_forward<M>();
  if (use_chain<M>(Mr, K, nb)) {
    if (qr_factor_chain<M>(st, Mr, K, nb, Am, b, Mat{at<double>(work, p.t), 32, 32 * std::max<int64_t>(K, 32)},
                           fwd ? &Qm : nullptr) != cudaSuccess)
      return MDLS_ERR_CUDA;
  } else if (qr_factor_overlap<M>(b.lane(0, st), b.lane(1, side_stream(0)), b.lane(2, side_stream(1)), Mr, K, nb, Am,
                                  b, fwd ? &Qm : nullptr) != cudaSuccess) {
    return MDLS_ERR_CUDA;
  }
  if (Q && !fwd) form_q_backward<M>(st, Mr, K, nb, Qm, b);
  if (dev_info) MDLS_LAUNCH(F_MISC, st, info_finish_kernel<<<1, 1, 0, st>>>(b.info_slot, nullptr, dev_info));
  return launched();
}

int MDLS_FN(mdls_apply_qt_)(int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                            const double* W, int64_t ldw, int64_t psw, const double* b, int64_t psb, double* y,
                            int64_t psy, void* work, size_t work_bytes, void* stream) {
  if (int e = tile_ok(Mr, K, nb)) return e;
  if (!mat_ok(A, Mr, K, lda, psa)) return -4;
  if (!mat_ok(W, Mr, K, ldw, psw)) return -7;
  if (!b || psb < Mr) return -10;
  if (!y || psy < Mr) return -12;
  const Plan p = make_plan<M>(MDLS_OP_APPLY_QT, Mr, K, nb);
  if (!work || work_bytes < p.total) return -15;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  Mat Y{at<double>(work, p.y), Mr, Mr * K};
  MDLS_LAUNCH(F_MISC, st, extract_y_kernel<M><<<grid_for(Mr * K, 256), 256, 0, st>>>(Mr, K, CMat{A, lda, psa}, Y));
  double* yv = y;
  if (y != b) MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(Mr, 256), 256, 0, st>>>(Mr, 1, CMat{b, Mr, psb}, Mat{y, Mr, psy}, 0));
  const int64_t mx = std::max(Mr, K);
  apply_qt_panels<M>(st, Mr, K, nb, cm(Y), CMat{W, ldw, psw}, Mat{yv, Mr, psy}, Mat{at<double>(work, p.x), nb, nb * mx},
                     at<double>(work, p.part), kMaxSplit * nb * mx);
  return launched();
}

int MDLS_FN(mdls_qt_b_)(int64_t Mr, int64_t Nc, const double* Q, int64_t ldq, int64_t psq, const double* b,
                        int64_t psb, double* y, int64_t psy, void* work, size_t work_bytes, void* stream) {
  if (Mr < 1) return -1;
  if (Nc < 0) return -2;
  if (Nc == 0) return 0;
  if (!mat_ok(Q, Mr, Nc, ldq, psq)) return -3;
  if (!b || psb < Mr) return -6;
  if (!y || psy < Nc || y == b) return -8;
  cudaStream_t st = S(stream);
  set_stage(MDLS_ST_QTB);
  // split-K partials go to the workspace when it is large enough
  const size_t need = sizeof(double) * M * kMaxSplit * Nc;
  double* part = (work && work_bytes >= need) ? static_cast<double*>(work) : nullptr;
  gemm<M, true, false>(st, Nc, 1, Mr, CMat{Q, ldq, psq}, CMat{b, Mr, psb}, Mat{y, Nc, psy}, 0, part,
                       part ? kMaxSplit * Nc : 0);
  return launched();
}

int MDLS_FN(mdls_zlstsq_)(int64_t Mr, int64_t K, int64_t nb, const double* Are, const double* Aim, int64_t lda,
                          int64_t psa, const double* bre, const double* bim, int64_t psb, double* xre, double* xim,
                          int64_t psx, int form_q, void* work, size_t work_bytes, int* dev_info, void* stream) {
  if (Mr < K) return -1;
  if (K < 1) return -2;
  if (nb < 1 || nb > 256 || (2 * K) % nb) return -3;
  if (!mat_ok(Are, Mr, K, lda, psa)) return -4;
  if (!mat_ok(Aim, Mr, K, lda, psa)) return -5;
  if (!bre || psb < Mr) return -8;
  if (!bim) return -9;
  if (!xre || psx < K) return -11;
  if (!xim) return -12;
  size_t emb;
  if (!work || work_bytes < zplan_bytes(Mr, K, nb, form_q, &emb)) return -16;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  const size_t md = sizeof(double) * M;
  double* E = static_cast<double*>(work);
  double* eb = at<double>(work, align256(md * 4 * Mr * K));
  double* ex = at<double>(work, align256(md * 4 * Mr * K) + align256(md * 2 * Mr));
  const int64_t M2 = 2 * Mr, K2 = 2 * K;
  MDLS_LAUNCH(F_MISC, st, embed_complex_kernel<M><<<grid_for(Mr * K, 256), 256, 0, st>>>(
                              Mr, K, CMat{Are, lda, psa}, CMat{Aim, lda, psa}, bre, bim, psb, Mat{E, M2, M2 * K2}, eb, M2));
  const int rc = lstsq_run(st, M2, K2, nb, E, M2, M2 * K2, eb, M2, ex, K2, form_q, nullptr, 0, 0, nullptr, 0, 0, nullptr,
                           0, static_cast<char*>(work) + emb, dev_info);
  if (rc) return rc;
  MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(K, 256), 256, 0, st>>>(K, 1, CMat{ex, K, K2}, Mat{xre, K, psx}, 0));
  MDLS_LAUNCH(F_MISC, st, copy_kernel<M><<<grid_for(K, 256), 256, 0, st>>>(K, 1, CMat{ex + K, K, K2}, Mat{xim, K, psx}, 0));
  return launched();
}

int MDLS_FN(mdls_norm2_)(int64_t n, const double* y, int64_t psy, double* out, int64_t pso, void* stream) {
  if (n < 0) return -1;
  if (!y || psy < n) return -2;
  if (!out || pso < 1) return -4;
  set_stage(MDLS_NSTAGES);
  cudaStream_t st = S(stream);
  MDLS_LAUNCH(F_MISC, st, norm2_kernel<M><<<1, 256, 0, st>>>(n, y, psy, out, pso));
  return launched();
}

int MDLS_FN(mdls_gemm_)(int64_t m, int64_t n, int64_t k, int trans_a, int trans_b, const double* A, int64_t lda,
                        int64_t psa, const double* B, int64_t ldb, int64_t psb, double* C, int64_t ldc, int64_t psc,
                        int mode, void* work, size_t work_bytes, void* stream) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (k < 0) return -3;
  if (trans_a < 0 || trans_a > 1) return -4;
  if (trans_b < 0 || trans_b > 1) return -5;
  if (m == 0 || n == 0) return 0;
  if (!mat_ok(A, trans_a ? k : m, trans_a ? m : k, lda, psa)) return -6;
  if (!mat_ok(B, trans_b ? n : k, trans_b ? k : n, ldb, psb)) return -9;
  if (!mat_ok(C, m, n, ldc, psc) || C == A || C == B) return -12;
  if (mode < 0 || mode > 3) return -15;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  const size_t need = sizeof(double) * M * kMaxSplit * m * n;
  double* part = (work && work_bytes >= need) ? static_cast<double*>(work) : nullptr;
  const int64_t cap = part ? kMaxSplit * m * n : 0;
  const CMat Am{A, lda, psa}, Bm{B, ldb, psb};
  const Mat Cm{C, ldc, psc};
  if (k == 0) {
    if (mode == 0 || mode == 3)
      MDLS_LAUNCH(F_MISC, st, set_zero_kernel<M><<<grid_for(m * n, 256), 256, 0, st>>>(m, n, Cm));
    return launched();
  }
  if (trans_a && trans_b) gemm<M, true, true>(st, m, n, k, Am, Bm, Cm, mode, part, cap);
  else if (trans_a) gemm<M, true, false>(st, m, n, k, Am, Bm, Cm, mode, part, cap);
  else if (trans_b) gemm<M, false, true>(st, m, n, k, Am, Bm, Cm, mode, part, cap);
  else gemm<M, false, false>(st, m, n, k, Am, Bm, Cm, mode, part, cap);
  return launched();
}

int MDLS_FN(mdls_lstsq_)(int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                         const double* b, int64_t psb, double* x, int64_t psx, int form_q, double* R_out, int64_t ldr,
                         int64_t psr, double* Q_out, int64_t ldq, int64_t psq, double* y_out, int64_t psy, void* work,
                         size_t work_bytes, int* dev_info, void* stream) {
  if (int e = tile_ok(Mr, K, nb)) return e;
  if (!mat_ok(A, Mr, K, lda, psa)) return -4;
  if (!b || psb < Mr) return -7;
  if (!x || psx < K) return -9;
  if (R_out && !mat_ok(R_out, Mr, K, ldr, psr)) return -12;
  if (Q_out && !form_q) return -11;
  if (Q_out && !mat_ok(Q_out, Mr, Mr, ldq, psq)) return -15;
  if (y_out && psy < Mr) return -19;
  const int op = form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ;
  if (!work || work_bytes < make_plan<M>(op, Mr, K, nb).total) return -21;
  return lstsq_run(S(stream), Mr, K, nb, A, lda, psa, b, psb, x, psx, form_q, R_out, ldr, psr, Q_out, ldq, psq, y_out,
                   psy, work, dev_info);
}

// host argument checks of mdls_lstsq_batched_<p> (-i = argument i)
static int batched_check(int64_t batch, int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                         int64_t strideA, const double* b, int64_t psb, int64_t strideB, const double* x, int64_t psx,
                         int64_t strideX, int form_q, int groups, const void* work, size_t work_bytes) {
  if (batch < 0) return -1;
  if (int e = tile_ok(Mr, K, nb)) return e - 1;
  if (!mat_ok(A, Mr, K, lda, psa)) return -5;
  if (strideA < (M - 1) * psa + lda * K) return -8;
  if (!b || psb < Mr) return -9;
  if (strideB < (M - 1) * psb + Mr) return -11;
  if (!x || psx < K) return -12;
  if (strideX < (M - 1) * psx + K) return -14;
  if (groups < 1 || groups > kMaxGroups) return -16;
  const int op = form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ;
  if (!work || work_bytes < align256(make_plan<M>(op, Mr, K, nb).total) * (size_t)groups) return -18;
  return 0;
}

// independent least-squares problems p = 0..batch-1 (A_p = A + p*strideA, b_p, x_p likewise):
// problem p runs on stream group p mod G with workspace slice p mod G, so G solves overlap on the device
int MDLS_FN(mdls_lstsq_batched_)(int64_t batch, int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda,
                                 int64_t psa, int64_t strideA, const double* b, int64_t psb, int64_t strideB,
                                 double* x, int64_t psx, int64_t strideX, int form_q, int groups, void* work,
                                 size_t work_bytes, int* dev_info, void* stream) {
  if (int e = batched_check(batch, Mr, K, nb, A, lda, psa, strideA, b, psb, strideB, x, psx, strideX, form_q, groups,
                            work, work_bytes))
    return e;
  const int op = form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ;
  const size_t slice = align256(make_plan<M>(op, Mr, K, nb).total);
  if (batch == 0) return 0;
  cudaStream_t st = S(stream);
  const int G = (int)std::min<int64_t>(groups, batch);
  std::vector<cudaStream_t> gst((size_t)G);
  for (int g = 0; g < G; ++g) {
    StreamGroup sg(g);
    gst[(size_t)g] = side_stream(6);
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(gst[(size_t)g], ev, 0);
  }
  int rc = 0;
  for (int64_t p = 0; p < batch && rc == 0; ++p) {
    const int g = (int)(p % G);
    StreamGroup sg(g);
    rc = lstsq_run(gst[(size_t)g], Mr, K, nb, A + p * strideA, lda, psa, b + p * strideB, psb, x + p * strideX, psx,
                   form_q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0, static_cast<char*>(work) + slice * (size_t)g,
                   dev_info ? dev_info + p : nullptr);
  }
  for (int g = 0; g < G; ++g) {  // joined even on an error (a caller's graph capture must not stay forked)
    cudaEvent_t ev = pool_event();
    cudaEventRecord(ev, gst[(size_t)g]);
    cudaStreamWaitEvent(st, ev, 0);
  }
  return rc;
}

// plans: the same calls captured once into a library-owned CUDA graph (buffers fixed at capture);
// mdls_plan_launch replays them with one host call
int MDLS_FN(mdls_lstsq_plan_)(int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                              const double* b, int64_t psb, double* x, int64_t psx, int form_q, void* work,
                              size_t work_bytes, int* dev_info, void** plan) {
  if (!plan) return -15;
  *plan = nullptr;
  if (int e = tile_ok(Mr, K, nb)) return e;
  if (!mat_ok(A, Mr, K, lda, psa)) return -4;
  if (!b || psb < Mr) return -7;
  if (!x || psx < K) return -9;
  const int op = form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ;
  if (!work || work_bytes < make_plan<M>(op, Mr, K, nb).total) return -13;
  cudaStream_t cs = capture_begin();
  if (!cs) return MDLS_ERR_CUDA;
  const int64_t n0 = mdls_launch_count();
  const int rc = lstsq_run(cs, Mr, K, nb, A, lda, psa, b, psb, x, psx, form_q, nullptr, 0, 0, nullptr, 0, 0, nullptr,
                           0, work, dev_info);
  const int rc2 = capture_end(cs, mdls_launch_count() - n0, plan);
  return rc ? rc : rc2;
}

// host-input least squares: A, b, x in pinned host memory (see include/mdls.h).  A's panels cross PCIe by
// copy-engine copies in stream order (direct call) and by the zero-copy panel kernel inside a plan's graph
// (measured, dd 1024: direct 4.70 vs 4.85 ms, plan 4.37 vs 4.65 ms); MDLS_HOST_ZC=0 / 1 forces one or the other
static bool host_zero_copy(bool in_plan) {
  static const int v = [] {
    const char* e = getenv("MDLS_HOST_ZC");
    return e ? atoi(e) : -1;
  }();
  return v < 0 ? in_plan : v != 0;
}
static int lstsq_host_check(int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                            const double* b, int64_t psb, const double* x, int64_t psx, int form_q, const void* work,
                            size_t work_bytes) {
  if (int e = tile_ok(Mr, K, nb)) return e;
  if (!mat_ok(A, Mr, K, lda, psa)) return -4;
  if (!b || psb < Mr) return -7;
  if (!x || psx < K) return -9;
  const int op = form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ;
  if (!work || work_bytes < make_plan<M>(op, Mr, K, nb).total) return -13;
  return 0;
}

int MDLS_FN(mdls_lstsq_host_)(int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                              const double* b, int64_t psb, double* x, int64_t psx, int form_q, void* work,
                              size_t work_bytes, int* dev_info, void* stream) {
  if (int e = lstsq_host_check(Mr, K, nb, A, lda, psa, b, psb, x, psx, form_q, work, work_bytes)) return e;
  const HostIO hio{A, lda, psa, b, psb, x, psx, host_zero_copy(false) ? mapped_ptr(A) : nullptr};
  return lstsq_run(S(stream), Mr, K, nb, nullptr, 0, 0, nullptr, 0, nullptr, 0, form_q, nullptr, 0, 0, nullptr, 0, 0,
                   nullptr, 0, work, dev_info, &hio);
}

int MDLS_FN(mdls_lstsq_host_plan_)(int64_t Mr, int64_t K, int64_t nb, const double* A, int64_t lda, int64_t psa,
                                   const double* b, int64_t psb, double* x, int64_t psx, int form_q, void* work,
                                   size_t work_bytes, int* dev_info, void** plan) {
  if (!plan) return -15;
  *plan = nullptr;
  if (int e = lstsq_host_check(Mr, K, nb, A, lda, psa, b, psb, x, psx, form_q, work, work_bytes)) return e;
  cudaStream_t cs = capture_begin();
  if (!cs) return MDLS_ERR_CUDA;
  const int64_t n0 = mdls_launch_count();
  const HostIO hio{A, lda, psa, b, psb, x, psx, host_zero_copy(true) ? mapped_ptr(A) : nullptr};
  const int rc = lstsq_run(cs, Mr, K, nb, nullptr, 0, 0, nullptr, 0, nullptr, 0, form_q, nullptr, 0, 0, nullptr, 0, 0,
                           nullptr, 0, work, dev_info, &hio);
  const int rc2 = capture_end(cs, mdls_launch_count() - n0, plan);
  return rc ? rc : rc2;
}

int MDLS_FN(mdls_lstsq_batched_plan_)(int64_t batch, int64_t Mr, int64_t K, int64_t nb, const double* A,
                                      int64_t lda, int64_t psa, int64_t strideA, const double* b, int64_t psb,
                                      int64_t strideB, double* x, int64_t psx, int64_t strideX, int form_q,
                                      int groups, void* work, size_t work_bytes, int* dev_info, void** plan) {
  if (!plan) return -20;
  *plan = nullptr;
  if (int e = batched_check(batch, Mr, K, nb, A, lda, psa, strideA, b, psb, strideB, x, psx, strideX, form_q, groups,
                            work, work_bytes))
    return e;
  cudaStream_t cs = capture_begin();
  if (!cs) return MDLS_ERR_CUDA;
  const int64_t n0 = mdls_launch_count();
  const int rc = MDLS_FN(mdls_lstsq_batched_)(batch, Mr, K, nb, A, lda, psa, strideA, b, psb, strideB, x, psx,
                                              strideX, form_q, groups, work, work_bytes, dev_info, cs);
  const int rc2 = capture_end(cs, mdls_launch_count() - n0, plan);
  if (rc && *plan) {
    mdls_plan_destroy(*plan);
    *plan = nullptr;
  }
  return rc ? rc : rc2;
}

size_t MDLS_FN(mdls_workspace_batched_)(int op, int64_t Mr, int64_t K, int64_t nb, int groups) {
  if (op != MDLS_OP_LSTSQ && op != MDLS_OP_LSTSQ_NOQ) return 0;
  if (groups < 1 || groups > kMaxGroups || tile_ok(Mr, K, nb)) return 0;
  return align256(make_plan<M>(op, Mr, K, nb).total) * (size_t)groups;
}

int MDLS_FN(mdls_qr_panel_)(int64_t Mr, int64_t nb, int64_t k, double* Ak, int64_t lda, int64_t psa, double* Wk,
                            int64_t ldw, int64_t psw, double* Yk, int64_t ldy, int64_t psy, void* work,
                            size_t work_bytes, int* dev_info, void* stream) {
  if (Mr < 1) return -1;
  if (nb < 1 || nb > 256) return -2;
  if (k < 0 || (k + 1) * nb > Mr) return -3;
  if (!mat_ok(Ak, Mr, nb, lda, psa)) return -4;
  // Wk, Yk are only touched on rows k*nb..M-1: a row-trimmed buffer may be passed (ld >= M - k*nb)
  if (!mat_ok(Wk, Mr - k * nb, nb, ldw, psw)) return -7;
  if (!mat_ok(Yk, Mr - k * nb, nb, ldy, psy)) return -10;
  const Plan p = make_plan<M>(MDLS_OP_QR, Mr, nb, nb);
  if (!work || work_bytes < p.total) return -14;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  const int64_t j0 = k * nb;
  // global-column views of the caller's M x nb panel buffers (column j -> j - j0)
  Mat Ag{Ak - j0 * lda, lda, psa}, Wg{Wk - j0 * ldw, ldw, psw}, Yg{Yk - j0 * ldy, ldy, psy};
  QrBufs<M> b = qr_bufs(work, p, Mr, nb, nb, nullptr, 0, 0);
  MDLS_LAUNCH(F_MISC, st, info_init_kernel<<<1, 1, 0, st>>>(b.info_slot));
  for (int l = 0; l < M; ++l) {
    cudaMemset2DAsync(Wk + l * psw + j0, sizeof(double) * ldw, 0, sizeof(double) * (Mr - j0), nb, st);
    cudaMemset2DAsync(Yk + l * psy + j0, sizeof(double) * ldy, 0, sizeof(double) * (Mr - j0), nb, st);
  }
  // beta: per panel, stored in the workspace (indexed by global column)
  const Lane L = b.lane(0, st);
  if (qr_panel<M>(L, L, Mr, nb, k, Ag, Yg, Wg, b.beta - j0, nb, b) != cudaSuccess) return MDLS_ERR_CUDA;
  if (dev_info) MDLS_LAUNCH(F_MISC, st, info_finish_kernel<<<1, 1, 0, st>>>(b.info_slot, nullptr, dev_info));
  return launched();
}

int MDLS_FN(mdls_qr_update_)(int64_t Mr, int64_t nb, int64_t k, const double* Wk, int64_t ldw, int64_t psw,
                             const double* Yk, int64_t ldy, int64_t psy, double* A, int64_t lda, int64_t psa,
                             int64_t c0, int64_t c1, void* work, size_t work_bytes, void* stream) {
  if (Mr < 1) return -1;
  if (nb < 1 || nb > 256) return -2;
  if (k < 0 || (k + 1) * nb > Mr) return -3;
  if (!mat_ok(Wk, Mr - k * nb, nb, ldw, psw)) return -4;  // rows k*nb..M-1 only (see mdls_qr_panel)
  if (!mat_ok(Yk, Mr - k * nb, nb, ldy, psy)) return -7;
  if (c0 < 0 || c1 < c0) return -13;
  if (!mat_ok(A, Mr, c1, lda, psa)) return -10;
  if (c1 > Mr) return -14;
  // scratch: one GEMM lane (X = W^T C, nb x (c1 - c0) <= nb x M, and split-K partials): the plan of a one-panel QR
  const Plan p = make_plan<M>(MDLS_OP_QR, Mr, nb, nb);
  if (!work || work_bytes < p.total) return -16;
  cudaStream_t st = S(stream);
  set_stage(MDLS_NSTAGES);
  QrBufs<M> b = qr_bufs(work, p, Mr, nb, nb, nullptr, 0, 0);
  const int64_t j0 = k * nb;
  qr_apply_panel<M>(b.lane(0, st), Mr, nb, k, CMat{Yk + j0, ldy, psy}, CMat{Wk + j0, ldw, psw}, Mat{A, lda, psa}, c0,
                    c1);
  return launched();
}

}  // extern "C"
