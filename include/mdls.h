/*
 * mdls.h -- C-ABI of libmdls.so: multiple-double least squares on B200 (sm_100a).
 *
 * Method: arXiv 2110.08375 (J. Verschelde, "Least Squares on GPUs in Multiple
 * Double Precision"), cited as P:<line> of PAPER.md.  The least squares solution
 * x of A x = b minimises ||b - A x||_2; A = Q R reduces A x = b to R x = Q^T b,
 * solved by back substitution.  Q, R come from the blocked Householder
 * QR of Algorithm 2, R x = y from the tiled accelerated back
 * substitution of Algorithm 1.
 *
 * PRECISIONS.  Every compute entry point exists four times, suffix _dd, _qd,
 * _od: double double, quad double, octo double = m = 2, 4, 8 limbs,
 * and _d: plain IEEE double (m = 1), the paper's "double precision version"
 * whose timings are listed beside the md runs.  _d runs the same
 * algorithms and kernels with one rounded operation per md operation (products
 * accumulated by FMA); its ledger prices every operation at one flop.
 *
 * LAYOUT ("staggered").  An md matrix is m plain double matrices,
 * most significant first.  Every matrix operand is described by
 *     (ptr, ld, ps):  limb l of element (i, j) is ptr[l*ps + j*ld + i]
 * i.e. each limb plane is column-major with leading dimension ld >= rows and
 * planes are ps >= ld*cols doubles apart.  A vector of length n is (ptr, ps)
 * with limb l of entry i at ptr[l*ps + i], ps >= n.
 *
 * MEMORY AND STREAMS.  All matrix/vector pointers are DEVICE pointers (CUDA
 * global memory of the current device) unless the name says host_.  The caller
 * owns every buffer; the library never allocates, frees or synchronises in a
 * compute call.  Scratch space is the caller's `work` buffer (device, 256-byte
 * aligned), of at least mdls_workspace_<p>() bytes.  `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream); every compute
 * call only enqueues work on it and returns.
 *
 * ERRORS.  Return 0 on success; -i when argument i (1-based) is invalid
 * (checked on the host before anything is enqueued; nothing is launched);
 * MDLS_ERR_CUDA when a launch failed (cudaGetLastError).  Numerical failures are
 * reported asynchronously through `dev_info` (a device int, may be NULL):
 *     0  success
 *     k > 0  the first (1-based, global row order) zero or non-finite diagonal
 *            entry of R met (QR) or of the triangular matrix (back substitution)
 *     -1  the input held a non-finite limb (lstsq only checks its inputs)
 * dev_info is written with plain stores/atomicMin on the stream; read it after
 * synchronising.
 */
#ifndef MDLS_H
#define MDLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDLS_ERR_CUDA (-100)
#define MDLS_ERR_UNSUPPORTED (-101)

/* operations for mdls_workspace_<p> and mdls_count_<p> */
enum {
  MDLS_OP_QR = 0,        /* mdls_qr_<p> (with Q formed when q_mode = 1)            */
  MDLS_OP_BACKSUB = 1,   /* mdls_backsub_<p>                                       */
  MDLS_OP_LSTSQ = 2,     /* mdls_lstsq_<p>: QR + Q + Q^T b (explicit Q) + backsub  */
  MDLS_OP_APPLY_QT = 3,  /* mdls_apply_qt_<p>                                      */
  MDLS_OP_LSTSQ_NOQ = 4, /* lstsq without forming Q (Q^T b applied from the panels) */
  MDLS_OP_ZLSTSQ = 5     /* mdls_zlstsq_<p>: complex least squares (M, K: the complex shape) */
};

/* stages of the flop ledger; the labels follow the paper's tables
 * (Algorithm 2 rows P:737-745, Algorithm 1 rows P:1118-1120) */
enum {
  MDLS_ST_HOUSE = 0,     /* "beta, v": Householder vectors (A1)              */
  MDLS_ST_PANEL = 1,     /* "beta R^T * v" + "update R" inside the panel (A2) */
  MDLS_ST_WY = 2,        /* "compute W" (A3)                                  */
  MDLS_ST_TRAILING = 3,  /* "YWT * C" + "R + YWTC": C += Y (W^T C) (A4)       */
  MDLS_ST_FORM_Q = 4,    /* "Q * WY^T" + "Q + QWY": Q formation (A5)          */
  MDLS_ST_QTB = 5,       /* Q^T b (A6; not in the paper's tables)             */
  MDLS_ST_INVERT = 6,    /* "invert diagonal tiles" (A7)                      */
  MDLS_ST_MULINV = 7,    /* "multiply with inverses" (A8)                     */
  MDLS_ST_BSUPDATE = 8,  /* "back substitution" update b_j -= A_ji x_i (A9)   */
  MDLS_NSTAGES = 9
};

/* canonical md operation counts of one call (host integers; A10 ledger).
 * flops = sum over stages of add*T1[add] + mul*T1[mul] + div*T1[div] +
 * sqrt*(T1[div] + 2*T1[mul]), with T1 = the paper's Table 1 sums:
 * dd 20/23/70, qd 89/336/893, od 269/1742/5126. */
typedef struct {
  int64_t add[MDLS_NSTAGES];  /* md additions and subtractions */
  int64_t mul[MDLS_NSTAGES];  /* md multiplications            */
  int64_t div[MDLS_NSTAGES];  /* md divisions                  */
  int64_t sqrt[MDLS_NSTAGES]; /* md square roots               */
  double flops[MDLS_NSTAGES]; /* Table-1-weighted double flops */
  double total_flops;
} mdls_counts;

const char *mdls_strerror(int code);
int mdls_version(void);
/* number of limbs of each precision */
int mdls_limbs(int prec_index /* 0 dd, 1 qd, 2 od, 3 d (plain double) */);

/* Instrumentation (host side, process wide).
 * mdls_launch_count: kernels launched by the library since it was loaded.
 * mdls_trace_enable(1): bracket every subsequent launch with CUDA events on its
 *   own stream (the paper's per-stage kernel times).  Must be off
 *   during CUDA-graph capture.
 * mdls_trace_collect: wait for the traced launches, add their event times per
 *   stage (stage_ms[MDLS_NSTAGES + 1]; the last slot is setup/copies) and per
 *   kernel family (family_ms[5], family_launches[5]: 0 md GEMM, 1 panel,
 *   2 tile inversion, 3 back substitution, 4 other), release the events.
 *   Returns the number of launches collected or MDLS_ERR_CUDA. Arrays may be NULL. */
int64_t mdls_launch_count(void);

/* Plans (library-owned CUDA graphs).  mdls_lstsq_plan_<p> / mdls_lstsq_batched_plan_<p> take the arguments of
 * the direct call (minus the stream) and capture its whole launch sequence once, on a library stream of the
 * current device, into an instantiated CUDA graph returned in *plan; the buffers (A, b, x, work, dev_info) are
 * fixed at capture and must stay allocated while the plan lives.  Nothing runs at creation.
 * mdls_plan_launch enqueues one replay on `stream` (one host call for the hundreds of kernels of a solve;
 * stream-ordered like the direct call).  Returns 0 or MDLS_ERR_CUDA; -1 for a NULL plan.
 * mdls_plan_launches: library kernels per replay.  mdls_plan_destroy releases the graph (NULL is a no-op). */
int mdls_plan_launch(void *plan, void *stream);
int64_t mdls_plan_launches(void *plan);
void mdls_plan_destroy(void *plan);
void mdls_trace_enable(int on);
int mdls_trace_collect(double *stage_ms, double *family_ms, int64_t *family_launches);

#define MDLS_DECLARE(P)                                                                                              \
  /* bytes of `work` needed by `op` for an M x K problem with tile size nb.  Returns 0 for invalid sizes. */        \
  size_t mdls_workspace_##P(int op, int64_t M, int64_t K, int64_t nb);                                             \
                                                                                                                   \
  /* canonical md-op counts of `op` (host only; A10).  Returns 0 or -i. */                                         \
  int mdls_count_##P(int op, int64_t M, int64_t K, int64_t nb, mdls_counts *out);                                  \
                                                                                                                   \
  /* A0: elementwise md arithmetic on device vectors (op: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt, 5 latency-lean sqrt, \
   * 6 latency-lean reciprocal 1/a -- the panel's Newton/Karp variants; 7 mul, 8 latency-lean sqrt, 9 latency-lean  \
   * reciprocal computed by one warp per entry (md_warp.cuh: the panel's warp-cooperative qd/od scalar chain; dd    \
   * falls back to ops 2/5/6); b unused for ops 4-6, 8, 9).                                                          \
   * c = a op b, n entries, planes ps apart (same ps for a, b, c).  The operations are the readings of              \
   * DESIGN.md. */                                                                                       \
  int mdls_md_op_##P(int op, int64_t n, const double *a, const double *b, double *c, int64_t ps, void *stream);     \
                                                                                                                   \
  /* Algorithm 2: blocked Householder QR of the M x K matrix A, K = N*nb, M >= K, nb | K,               \
   * 1 <= nb <= 256.  On return A holds R in its upper triangle (R_jj >= 0 unless a column was exactly zero         \
   * below its diagonal, GVL Alg. 5.1.1) and the Householder vectors v_j (v_j(1) = 1 implicit)           \
   * strictly below.  W (M x K, nullable): column j holds the W column of reflector j, rows >= panel start; the     \
   * panel's P_WY = I + W Y^T.  Q (M x M, nullable): Q = P_WY(1) ... P_WY(N), A = Q R.                 \
   * All three are (ptr, ld, ps) operands. */                                                                      \
  int mdls_qr_##P(int64_t M, int64_t K, int64_t nb, double *A, int64_t lda, int64_t psa, double *Q, int64_t ldq,   \
                  int64_t psq, double *W, int64_t ldw, int64_t psw, void *work, size_t work_bytes, int *dev_info,  \
                  void *stream);                                                                                   \
                                                                                                                   \
  /* y = Q^T b from a factored A (mdls_qr output) and its W: y = b; for k = 1..N: y += Y_k (W_k^T y).               \
   * b, y: vectors of length M (may alias). */                                                                     \
  int mdls_apply_qt_##P(int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda, int64_t psa,               \
                        const double *W, int64_t ldw, int64_t psw, const double *b, int64_t psb, double *y,        \
                        int64_t psy, void *work, size_t work_bytes, void *stream);                                 \
                                                                                                                   \
  /* y = Q^T b with an explicit Q of M rows and N columns (N = M: the full Q; N < M: a column block,     \
   * as in the column-sharded Q^T b).  b: length M, y: length N; b and y must not alias. */                        \
  int mdls_qt_b_##P(int64_t M, int64_t N, const double *Q, int64_t ldq, int64_t psq, const double *b, int64_t psb,  \
                    double *y, int64_t psy, void *work, size_t work_bytes, void *stream);                          \
                                                                                                                   \
  /* A3-A6 building block: the md tile product of the trailing update "YWT * C" / "R + YWTC" and    \
   * of Q formation, C (mode)= op(A) op(B) with op(X) = X or X^T (trans_a, trans_b), op(A) m x k, op(B) k x n,       \
   * C m x n.  mode: 0 C = P, 1 C += P, 2 C -= P, 3 C = -P.  Every product is one md mul, every sum an md add       \
   * (dd: unnormalised pair accumulation; qd/od: level-bin accumulation); long k is split      \
   * over CTAs and reduced in a fixed order when `work` holds >= 8*m*n*8*limbs bytes (else no split).              \
   * All operands device, limb-planar (ptr, ld, ps); C must not alias A or B. */                                   \
  int mdls_gemm_##P(int64_t m, int64_t n, int64_t k, int trans_a, int trans_b, const double *A, int64_t lda,       \
                    int64_t psa, const double *B, int64_t ldb, int64_t psb, double *C, int64_t ldc, int64_t psc,   \
                    int mode, void *work, size_t work_bytes, void *stream);                                        \
                                                                                                                   \
  /* A7: invert the N = n/nb diagonal nb x nb tiles of the upper-triangular U (leading n x n).          \
   * Vt receives the TRANSPOSED inverses: tile i of U^-1 at columns [i*nb, (i+1)*nb) of an nb x n operand,          \
   * Vt(c, i*nb + r) = (U_i^-1)(r, c).  dev_info: first zero diagonal (1-based). */                                \
  int mdls_invert_tiles_##P(int64_t n, int64_t nb, const double *U, int64_t ldu, int64_t psu, double *Vt,          \
                            int64_t ldv, int64_t psv, int *dev_info, void *stream);                                \
                                                                                                                   \
  /* Algorithm 1: solve U x = y for the leading n x n upper-triangular block of U, N = n/nb tiles:      \
   * invert the diagonal tiles, then for i = N..1: x_i = U_i^-1 y_i and y_j -= A_ji x_i (j < i).                   \
   * y is read only (copied into work); x: vector of length n. */                                                  \
  int mdls_backsub_##P(int64_t n, int64_t nb, const double *U, int64_t ldu, int64_t psu, const double *y,          \
                       int64_t psy, double *x, int64_t psx, void *work, size_t work_bytes, int *dev_info,          \
                       void *stream);                                                                              \
                                                                                                                   \
  /* least squares (Table 11 pipeline P:1459-1463): A = QR (A is not modified; factored in work),          \
   * y = Q^T b, R(1:K,1:K) x = y(1:K) by Algorithm 1.  With form_q = 1 Q is formed explicitly and y = Q^T b is a    \
   * product with Q (the paper's pipeline, Q_out receives Q if not NULL); with form_q = 0 Q^T b is applied from    \
   * the panels.  R_out (M x K, nullable) receives R (strictly lower part zero).  y_out (length M, nullable)        \
   * receives Q^T b; its entries K+1..M give the residual norm.  x: vector of length K. */                         \
  int mdls_lstsq_##P(int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda, int64_t psa, const double *b, \
                     int64_t psb, double *x, int64_t psx, int form_q, double *R_out, int64_t ldr, int64_t psr,     \
                     double *Q_out, int64_t ldq, int64_t psq, double *y_out, int64_t psy, void *work,              \
                     size_t work_bytes, int *dev_info, void *stream);                                              \
                                                                                                                   \
  /* a batch of independent least-squares problems (SURVEY 8e batch sharding; the paper's motivation is many     \
   * solves inside a path tracker): problem p = 0..batch-1 is mdls_lstsq on A + p*strideA,             \
   * b + p*strideB, x + p*strideX (strides in doubles, no overlap: strideA >= (m-1)*psa + lda*K etc.), all of     \
   * the same M x K shape and tile nb.  The problems run on `groups` (1..16) library stream groups -- problem p on \
   * group p mod groups with the workspace slice p mod groups -- so up to `groups` solves overlap on the device; \
   * every group is forked from and joined into `stream`.  work: mdls_workspace_batched_<p>(op, M, K, nb, groups)\
   * bytes.  dev_info (nullable): batch device ints, entry p as mdls_lstsq's dev_info of problem p. */           \
  int mdls_lstsq_batched_##P(int64_t batch, int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda,        \
                             int64_t psa, int64_t strideA, const double *b, int64_t psb, int64_t strideB,          \
                             double *x, int64_t psx, int64_t strideX, int form_q, int groups, void *work,          \
                             size_t work_bytes, int *dev_info, void *stream);                                      \
  /* least squares with HOST inputs and output (the end-to-end call): A (M x K, lda >= M, planes psa  \
   * apart), b (planes psb >= M apart) and x (planes psx >= K apart) are in page-locked host memory (cudaHostAlloc \
   * / torch pin_memory; pageable memory makes the copies synchronous).  b is copied first; A column panel by     \
   * column panel (nb columns, every limb plane) on a library copy stream (copy engines; inside a plan a        \
   * zero-copy kernel reading the mapped pinned pages), one event per panel, so the leaf                          \
   * chain starts on panel 0 while the rest of A is in flight and every lane waits only for the panels it        \
   * touches; x is copied back at the end.  Everything is stream-ordered on `stream` (x is valid after it        \
   * synchronises).  work: mdls_workspace_<p>(form_q ? MDLS_OP_LSTSQ : MDLS_OP_LSTSQ_NOQ, M, K, nb) bytes (device). \
   * Errors: -1..-3 sizes, -4 A, -7 b, -9 x, -13 workspace; dev_info as mdls_lstsq. */                          \
  int mdls_lstsq_host_##P(int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda, int64_t psa,            \
                          const double *b, int64_t psb, double *x, int64_t psx, int form_q, void *work,           \
                          size_t work_bytes, int *dev_info, void *stream);                                        \
  /* plan version of mdls_lstsq_host_<p>: the host buffers are fixed at capture (keep them pinned and alive). */ \
  int mdls_lstsq_host_plan_##P(int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda, int64_t psa,       \
                               const double *b, int64_t psb, double *x, int64_t psx, int form_q, void *work,      \
                               size_t work_bytes, int *dev_info, void **plan);                                    \
  /* plan versions of mdls_lstsq_<p> and mdls_lstsq_batched_<p> (see "Plans" above); *plan = NULL on error. */  \
  int mdls_lstsq_plan_##P(int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda, int64_t psa,            \
                          const double *b, int64_t psb, double *x, int64_t psx, int form_q, void *work,             \
                          size_t work_bytes, int *dev_info, void **plan);                                          \
  int mdls_lstsq_batched_plan_##P(int64_t batch, int64_t M, int64_t K, int64_t nb, const double *A, int64_t lda,  \
                                  int64_t psa, int64_t strideA, const double *b, int64_t psb, int64_t strideB,     \
                                  double *x, int64_t psx, int64_t strideX, int form_q, int groups, void *work,     \
                                  size_t work_bytes, int *dev_info, void **plan);                                  \
  /* bytes of `work` for mdls_lstsq_batched_<p> (op MDLS_OP_LSTSQ or MDLS_OP_LSTSQ_NOQ); 0 for invalid sizes. */ \
  size_t mdls_workspace_batched_##P(int op, int64_t M, int64_t K, int64_t nb, int groups);                        \
                                                                                                                   \
  /* complex least squares (row f2, re/im parts in separate limb-planar arrays):          \
   * x = argmin ||b - A x||_2 for complex A (M x K: Are + i Aim, both (ptr, lda, psa)), b (bre + i bim, planes psb)\
   * and x (xre + i xim, planes psx).  Solved through the real embedding [[Re A, -Im A], [Im A, Re A]] (2M x 2K)  \
   * [Re x; Im x] = [Re b; Im b] -- the same minimiser, since ||b - Ax||^2 = ||Re(b - Ax)||^2 + ||Im(b - Ax)||^2 -- \
   * by the real pipeline (mdls_lstsq, tile nb; 2K % nb == 0 required).  work: mdls_workspace_<p>(MDLS_OP_ZLSTSQ, \
   * M, K, nb) bytes (form_q = 1) -- the embedded problem, its plan and the real solution. */                   \
  int mdls_zlstsq_##P(int64_t M, int64_t K, int64_t nb, const double *Are, const double *Aim, int64_t lda,        \
                      int64_t psa, const double *bre, const double *bim, int64_t psb, double *xre, double *xim,    \
                      int64_t psx, int form_q, void *work, size_t work_bytes, int *dev_info, void *stream);         \
                                                                                                                   \
  /* ||y||_2 of the md vector y of length n (n >= 0), in md: one md number written to out (limb l at           \
   * out[l*pso]).  With y = (Q^T b)(K+1:M) from mdls_lstsq's y_out this is the least-squares residual norm        \
   * ||b - A x||_2 (orthogonality of Q).  Fixed-order reduction (bitwise reproducible). */  \
  int mdls_norm2_##P(int64_t n, const double *y, int64_t psy, double *out, int64_t pso, void *stream);             \
                                                                                                                   \
  /* multi-GPU building blocks (block-column sharded QR; host orchestration in sharded.py).           \
   * qr_panel: factor panel k, i.e. the columns [k*nb, (k+1)*nb) of A passed as the M x nb operand Ak (rows        \
   * 0..M-1, all earlier panels already applied), M >= (k+1)*nb; on return Ak holds R and v like mdls_qr, and     \
   * Wk, Yk (M x nb, rows < k*nb zero) hold the panel's W and explicit Y (unit diagonal): P_WY = I + Wk Yk^T.      \
   * dev_info as for mdls_qr (global 1-based row).  Wk and Yk are only accessed on rows k*nb..M-1, so a caller    \
   * may keep just those rows (the sharded driver broadcasts them): pass the buffer pointer minus k*nb, ld >=       \
   * M - k*nb (the same holds for qr_update's Wk, Yk). */                                                            \
  int mdls_qr_panel_##P(int64_t M, int64_t nb, int64_t k, double *Ak, int64_t lda, int64_t psa, double *Wk,        \
                        int64_t ldw, int64_t psw, double *Yk, int64_t ldy, int64_t psy, void *work,                 \
                        size_t work_bytes, int *dev_info, void *stream);                                           \
  /* qr_update: C += Yk (Wk^T C) for the columns [c0, c1) of A (c1 <= M), rows k*nb..M-1 ("YWT * C", "R + YWTC"); \
   * work: mdls_workspace_<p>(MDLS_OP_QR, M, nb, nb) bytes.                                                         \
   * With Wk and Yk exchanged it computes C += Wk (Yk^T C): the backward Q-formation step on a column block. */   \
  int mdls_qr_update_##P(int64_t M, int64_t nb, int64_t k, const double *Wk, int64_t ldw, int64_t psw,             \
                         const double *Yk, int64_t ldy, int64_t psy, double *A, int64_t lda, int64_t psa,          \
                         int64_t c0, int64_t c1, void *work, size_t work_bytes, void *stream);

MDLS_DECLARE(dd)
MDLS_DECLARE(qd)
MDLS_DECLARE(od)
MDLS_DECLARE(d)

#undef MDLS_DECLARE

#ifdef __cplusplus
}
#endif
#endif /* MDLS_H */
