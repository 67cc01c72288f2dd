/*
 * oracle/mdls_oracle.c -- CPU ORACLE FOR THE MULTIPLE-DOUBLE LEAST-SQUARES PATH.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and
 *   bench.py's cpu_baseline / --impl reference legs may load this library.  The
 *   product (paper_2110_08375_b200/, libmdls.so) never links, imports or calls it,
 *   and this file shares no code, header, table or constant with the CUDA path.
 *
 * What it computes (PAPER.md = arXiv 2110.08375, cited as P:<line>):
 *   - multiple double numbers: unevaluated sums of m doubles, m = 2 (dd), 4 (qd),
 *     8 (od); m = 1 is plain IEEE double arithmetic (one rounded
 *     +,-,*,/,sqrt per operation), the paper's "double precision version" whose
 *     timings are listed beside the md runs.  Arithmetic is the paper's named families: QDlib for dd
 *      and CAMPARY's generated qd/od code (P:152-156,
 *     P:615-625).  The paper prints no algorithm, only their Table 1 operation
 *     counts; the exact variants below are the readings of DESIGN.md
 *     ("md arithmetic readings"), which reproduce every octo double cell of
 *     Table 1 exactly (tests/test_oracle_counts.py pins that).
 *   - blocked Householder QR reaches the same (Q, R) as the textbook
 *     unblocked Householder QR in exact arithmetic; this oracle IS that textbook
 *     computation (Golub & Van Loan Alg. 5.1.1 house + Alg. 5.2.1 QR),
 *     carried out in md arithmetic, with Q accumulated backward.
 *   - tiled back substitution reaches the same x as plain back
 *     substitution; this oracle is plain row back substitution.
 *   - least squares: A = QR, R x = Q^T b.
 *
 * Storage: an md matrix is m plain double matrices, most significant
 * first.  Plane l of an R x C operand starts at ptr + l*ld*C, column-major with
 * leading dimension ld.  Vectors are m planes of length n (stride n).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (no FMA contraction: the
 * error-free transformations below depend on every +,-,* being rounded once).
 * With -DMDLS_ORACLE_COUNT every base-double +,-,*,/ is tallied (Table 1 pins).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXM 8
/* m = 1 is plain IEEE double ("1d", the paper's reference rows) */
#define BAD_M(m) ((m) != 1 && (m) != 2 && (m) != 4 && (m) != 8)

/* ------------------------------------------------------------------------- */
/* base double operations, optionally counted                                 */
/* ------------------------------------------------------------------------- */
#ifdef MDLS_ORACLE_COUNT
static uint64_t g_cnt[4]; /* additions, subtractions, multiplications, divisions */
static inline double ADD(double a, double b) { g_cnt[0]++; return a + b; }
static inline double SUB(double a, double b) { g_cnt[1]++; return a - b; }
static inline double MUL(double a, double b) { g_cnt[2]++; return a * b; }
static inline double DIV(double a, double b) { g_cnt[3]++; return a / b; }
/* negation of one limb: Table 1 tallies it as a subtraction (md readings) */
static inline double NEG(double a) { g_cnt[1]++; return -a; }
void oracle_count_reset(void) { memset(g_cnt, 0, sizeof(g_cnt)); }
void oracle_count_get(uint64_t *out) { memcpy(out, g_cnt, sizeof(g_cnt)); }
int oracle_is_counting(void) { return 1; }
#else
static inline double ADD(double a, double b) { return a + b; }
static inline double SUB(double a, double b) { return a - b; }
static inline double MUL(double a, double b) { return a * b; }
static inline double DIV(double a, double b) { return a / b; }
static inline double NEG(double a) { return -a; }
void oracle_count_reset(void) {}
void oracle_count_get(uint64_t *out) { memset(out, 0, 4 * sizeof(uint64_t)); }
int oracle_is_counting(void) { return 0; }
#endif

/* ------------------------------------------------------------------------- */
/* error-free transformations                                                 */
/* ------------------------------------------------------------------------- */

/* two_sum (Knuth): s = fl(a+b), e = a+b-s exactly.  2 additions, 4 subtractions. */
static void two_sum(double a, double b, double *s, double *e) {
  double ss = ADD(a, b);
  double bb = SUB(ss, a);
  *e = ADD(SUB(a, SUB(ss, bb)), SUB(b, bb));
  *s = ss;
}

/* quick_two_sum / Fast2Sum (Dekker), valid when |a| >= |b|: 1 addition, 2 subtractions. */
static void quick_two_sum(double a, double b, double *s, double *e) {
  double ss = ADD(a, b);
  *e = SUB(b, SUB(ss, a));
  *s = ss;
}

/* Veltkamp split as in QDlib: a = hi + lo, each half fits in 26 bits. */
static void split(double a, double *hi, double *lo) {
  const double SPLITTER = 134217729.0;               /* 2^27 + 1 */
  const double SPLIT_THRESH = 6.69692879491417e+299; /* 2^996 */
  if (a > SPLIT_THRESH || a < -SPLIT_THRESH) {
    double as = a * 3.7252902984619140625e-09; /* 2^-28 */
    double t = MUL(SPLITTER, as);
    double h = SUB(t, SUB(t, as));
    double l = SUB(as, h);
    *hi = h * 268435456.0; /* 2^28 */
    *lo = l * 268435456.0;
  } else {
    double t = MUL(SPLITTER, a);
    *hi = SUB(t, SUB(t, a));
    *lo = SUB(a, *hi);
  }
}

/* two_prod (Dekker, no FMA): p = fl(a*b), e = a*b-p exactly.
 * 7 multiplications, 3 additions, 7 subtractions (the tally Table 1 implies). */
static void two_prod(double a, double b, double *p, double *e) {
  double ah, al, bh, bl;
  double pp = MUL(a, b);
  split(a, &ah, &al);
  split(b, &bh, &bl);
  *e = ADD(ADD(ADD(SUB(MUL(ah, bh), pp), MUL(ah, bl)), MUL(al, bh)), MUL(al, bl));
  *p = pp;
}

/* exported for the EFT exactness pins */
void oracle_two_sum(double a, double b, double *out) { two_sum(a, b, &out[0], &out[1]); }
void oracle_quick_two_sum(double a, double b, double *out) { quick_two_sum(a, b, &out[0], &out[1]); }
void oracle_two_prod(double a, double b, double *out) { two_prod(a, b, &out[0], &out[1]); }
void oracle_split(double a, double *out) { split(a, &out[0], &out[1]); }

/* ------------------------------------------------------------------------- */
/* double double (QDlib)                                           */
/* ------------------------------------------------------------------------- */

/* QDlib dd_real::ieee_add. 8 additions, 12 subtractions (Table 1 dd add row). */
static void dd_add(const double *a, const double *b, double *c) {
  double s1, s2, t1, t2;
  two_sum(a[0], b[0], &s1, &s2);
  two_sum(a[1], b[1], &t1, &t2);
  s2 = ADD(s2, t1);
  quick_two_sum(s1, s2, &s1, &s2);
  s2 = ADD(s2, t2);
  quick_two_sum(s1, s2, &c[0], &c[1]);
}

/* QDlib dd * dd: two_prod of the leading limbs plus the two cross products. */
static void dd_mul(const double *a, const double *b, double *c) {
  double p1, p2;
  two_prod(a[0], b[0], &p1, &p2);
  p2 = ADD(p2, ADD(MUL(a[0], b[1]), MUL(a[1], b[0])));
  quick_two_sum(p1, p2, &c[0], &c[1]);
}

/* QDlib dd * double. */
static void dd_mul_d(const double *a, double b, double *c) {
  double p1, p2;
  two_prod(a[0], b, &p1, &p2);
  p2 = ADD(p2, MUL(a[1], b));
  quick_two_sum(p1, p2, &c[0], &c[1]);
}

/* QDlib dd + double. */
static void dd_add_d(const double *a, double b, double *c) {
  double s1, s2;
  two_sum(a[0], b, &s1, &s2);
  s2 = ADD(s2, a[1]);
  quick_two_sum(s1, s2, &c[0], &c[1]);
}

static void dd_sub(const double *a, const double *b, double *c) {
  double nb[2] = {NEG(b[0]), NEG(b[1])};
  dd_add(a, nb, c);
}

/* QDlib dd_real::accurate_div: three quotient digits q1, q2, q3. */
static void dd_div(const double *a, const double *b, double *c) {
  double q1, q2, q3, r[2], t[2];
  q1 = DIV(a[0], b[0]);
  dd_mul_d(b, q1, t);
  dd_sub(a, t, r); /* r = a - q1*b */
  q2 = DIV(r[0], b[0]);
  dd_mul_d(b, q2, t);
  dd_sub(r, t, r); /* r -= q2*b */
  q3 = DIV(r[0], b[0]);
  quick_two_sum(q1, q2, &q1, &q2);
  double q[2] = {q1, q2};
  dd_add_d(q, q3, c);
}

/* QDlib dd sqrt: one Newton correction of the double reciprocal square root
 * (P:633-635): x = 1/sqrt(a0); ax = a0*x; c = ax + (a - ax^2)_0 * (x/2). */
static void dd_sqrt(const double *a, double *c) {
  if (a[0] == 0.0) { c[0] = c[1] = 0.0; return; }
  double x = DIV(1.0, sqrt(a[0]));
  double ax = MUL(a[0], x);
  double sq[2], d[2];
  two_prod(ax, ax, &sq[0], &sq[1]);
  dd_sub(a, sq, d);
  two_sum(ax, MUL(d[0], MUL(x, 0.5)), &c[0], &c[1]);
}

/* ------------------------------------------------------------------------- */
/* quad double and octo double (CAMPARY "fast" family)             */
/* ------------------------------------------------------------------------- */

/* Renormalisation of m+1 terms to m limbs (CAMPARY fast_renorm2L<m+1,m>):
 * 2m-1 Fast2Sums.  Level 1 is a bottom-up Fast2Sum sweep over f[0..m]; level 2
 * is a top-down sweep over its first m outputs that emits a limb whenever the
 * Fast2Sum error is nonzero, then zero-pads.  (Reading: DESIGN.md.) */
static void renorm(int m, const double *f, double *r) {
  double g[MAXM + 1];
  double s = f[m];
  for (int i = m - 1; i >= 0; --i) quick_two_sum(f[i], s, &s, &g[i + 1]);
  g[0] = s;
  double eps = g[0];
  int j = 0;
  for (int i = 1; i <= m - 1; ++i) {
    double rr, e;
    quick_two_sum(eps, g[i], &rr, &e);
    if (e != 0.0) {
      r[j++] = rr;
      eps = e;
    } else {
      eps = rr;
    }
  }
  r[j++] = eps;
  for (; j < m; ++j) r[j] = 0.0;
}

/* CAMPARY baileyAdd_fast<m,m,m>: position sums from the least significant
 * upward; each error is carried by two_sums through the less significant
 * positions and its remainder added into the tail term f[m]. */
static void mdg_add(int m, const double *a, const double *b, double *c) {
  double f[MAXM + 1], e;
  f[m] = 0.0;
  for (int i = m - 1; i >= 0; --i) {
    two_sum(a[i], b[i], &f[i], &e);
    for (int j = i + 1; j < m; ++j) two_sum(f[j], e, &f[j], &e);
    f[m] = ADD(f[m], e);
  }
  renorm(m, f, c);
}

/* carry an error term x through f[n+1..m-1] and into the tail f[m] */
static void carry(int m, int n, double *f, double x) {
  for (int j = n + 1; j < m; ++j) two_sum(f[j], x, &f[j], &x);
  f[m] = ADD(f[m], x);
}

/* CAMPARY baileyMul_fast<m,la,lb> for la, lb in {1, m}, m output limbs:
 *   f[m] = sum of the plain products a_i*b_j with i+j = m;
 *   for levels n = m-1 .. 0: every two_prod a_i*b_{n-i} (i ascending) is summed
 *   into f[n] by two_sum (the first is assigned), its product error and then
 *   the sum error are carried through f[n+1..m-1] into f[m];
 *   then renorm(f[0..m]). */
static void mdg_mul_gen(int m, int la, const double *a, int lb, const double *b, double *c) {
  double f[MAXM + 1];
  int first = 1;
  f[m] = 0.0;
  for (int i = 0; i < la; ++i) {
    int j = m - i;
    if (j < 0 || j >= lb) continue;
    double p = MUL(a[i], b[j]);
    if (first) { f[m] = p; first = 0; } else f[m] = ADD(f[m], p);
  }
  for (int n = m - 1; n >= 0; --n) {
    int have = 0;
    for (int i = 0; i <= n; ++i) {
      int j = n - i;
      if (i >= la || j >= lb) continue;
      double p, pe, e;
      two_prod(a[i], b[j], &p, &pe);
      if (!have) {
        f[n] = p;
        have = 1;
        carry(m, n, f, pe);
      } else {
        two_sum(f[n], p, &f[n], &e);
        carry(m, n, f, pe);
        carry(m, n, f, e);
      }
    }
    if (!have) f[n] = 0.0;
  }
  renorm(m, f, c);
}

static void mdg_mul(int m, const double *a, const double *b, double *c) { mdg_mul_gen(m, m, a, m, b, c); }

/* long division: q0 = a0/b0; for i = 1..m: r -= q_{i-1}*b (md x double, the
 * subtraction an addition of the negated limbs); q_i = r0/b0; renorm(q0..qm). */
static void mdg_div(int m, const double *a, const double *b, double *c) {
  double q[MAXM + 1], r[MAXM], t[MAXM], qb[1];
  memcpy(r, a, sizeof(double) * m);
  q[0] = DIV(a[0], b[0]);
  for (int i = 1; i <= m; ++i) {
    qb[0] = q[i - 1];
    mdg_mul_gen(m, m, b, 1, qb, t);
    for (int k = 0; k < m; ++k) t[k] = NEG(t[k]);
    mdg_add(m, r, t, r);
    q[i] = DIV(r[0], b[0]);
  }
  renorm(m, q, c);
}

/* QDlib-style square root extended to m limbs: Newton on the
 * reciprocal square root, y <- y + (1/2 - (a/2) y^2) y, from y0 = 1/sqrt(a0),
 * ceil(log2 m)+1 times; result a*y. */
static void mdg_sqrt(int m, const double *a, double *c) {
  if (a[0] == 0.0) { memset(c, 0, sizeof(double) * m); return; }
  int iters = (m == 4) ? 3 : 4;
  double y[MAXM] = {0}, h[MAXM], t[MAXM], half[MAXM] = {0};
  y[0] = DIV(1.0, sqrt(a[0]));
  half[0] = 0.5;
  for (int k = 0; k < m; ++k) h[k] = a[k] * 0.5; /* exact scaling by a power of two */
  for (int it = 0; it < iters; ++it) {
    mdg_mul(m, y, y, t);
    mdg_mul(m, h, t, t);
    for (int k = 0; k < m; ++k) t[k] = NEG(t[k]);
    mdg_add(m, half, t, t);
    mdg_mul(m, t, y, t);
    mdg_add(m, y, t, y);
  }
  mdg_mul(m, a, y, c);
}

/* ------------------------------------------------------------------------- */
/* precision dispatch                                                         */
/* ------------------------------------------------------------------------- */
static void md_add(int m, const double *a, const double *b, double *c) {
  if (m == 1) c[0] = ADD(a[0], b[0]);
  else if (m == 2) dd_add(a, b, c); else mdg_add(m, a, b, c);
}
static void md_mul(int m, const double *a, const double *b, double *c) {
  if (m == 1) c[0] = MUL(a[0], b[0]);
  else if (m == 2) dd_mul(a, b, c); else mdg_mul(m, a, b, c);
}
static void md_div(int m, const double *a, const double *b, double *c) {
  if (m == 1) c[0] = DIV(a[0], b[0]);
  else if (m == 2) dd_div(a, b, c); else mdg_div(m, a, b, c);
}
static void md_sqrt(int m, const double *a, double *c) {
  if (m == 1) c[0] = sqrt(a[0]); /* correctly rounded (IEEE 754) */
  else if (m == 2) dd_sqrt(a, c); else mdg_sqrt(m, a, c);
}
static void md_neg(int m, const double *a, double *c) {
  for (int k = 0; k < m; ++k) c[k] = NEG(a[k]);
}
static void md_sub(int m, const double *a, const double *b, double *c) {
  double nb[MAXM];
  md_neg(m, b, nb);
  md_add(m, a, nb, c);
}
static void md_zero(int m, double *c) { memset(c, 0, sizeof(double) * m); }
static void md_set_d(int m, double d, double *c) { md_zero(m, c); c[0] = d; }
static void md_copy(int m, const double *a, double *c) { memcpy(c, a, sizeof(double) * m); }
/* sign of a renormalised expansion is the sign of its leading limb */
static double md_lead(const double *a) { return a[0]; }
static void md_abs(int m, const double *a, double *c) {
  if (a[0] < 0.0) md_neg(m, a, c); else md_copy(m, a, c);
}
/* a < b  <=>  lead(a - b) < 0 */
static int md_lt(int m, const double *a, const double *b) {
  double d[MAXM];
  md_sub(m, a, b, d);
  return d[0] < 0.0;
}

/* vectorised single-operation entry point (op: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt) */
int oracle_md_op(int op, int m, int64_t n, const double *a, const double *b, double *c) {
  if (BAD_M(m)) return -2;
  for (int64_t i = 0; i < n; ++i) {
    double x[MAXM], y[MAXM], z[MAXM];
    for (int k = 0; k < m; ++k) {
      x[k] = a[k * n + i];
      y[k] = b ? b[k * n + i] : 0.0;
    }
    switch (op) {
      case 0: md_add(m, x, y, z); break;
      case 1: md_sub(m, x, y, z); break;
      case 2: md_mul(m, x, y, z); break;
      case 3: md_div(m, x, y, z); break;
      case 4: md_sqrt(m, x, z); break;
      default: return -1;
    }
    for (int k = 0; k < m; ++k) c[k * n + i] = z[k];
  }
  return 0;
}
/* renormalisation of an (m+1)-term array, for the renorm pins */
int oracle_renorm(int m, const double *f, double *r) {
  if (BAD_M(m)) return -2;
  renorm(m, f, r);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* limb-planar element access                                                 */
/* ------------------------------------------------------------------------- */
typedef struct {
  double *p;
  int64_t ld, cols;
  int m;
} mat_t;

static inline void get(const mat_t *A, int64_t i, int64_t j, double *x) {
  for (int k = 0; k < A->m; ++k) x[k] = A->p[k * A->ld * A->cols + j * A->ld + i];
}
static inline void put(const mat_t *A, int64_t i, int64_t j, const double *x) {
  for (int k = 0; k < A->m; ++k) A->p[k * A->ld * A->cols + j * A->ld + i] = x[k];
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

/* ------------------------------------------------------------------------- */
/* Householder vector: Golub & Van Loan (3rd ed.) Algorithm 5.1.1  */
/* x = x[0..n-1] (md, contiguous m-limb records).  On return v[0] = 1, beta,  */
/* and mu = the first entry of P x (= ||x||_2 when sigma != 0, else x1).      */
/* ------------------------------------------------------------------------- */
static void house(int m, int64_t n, const double *x, double *v, double *beta, double *mu) {
  double sigma[MAXM], t[MAXM], x1[MAXM];
  md_zero(m, sigma);
  for (int64_t i = 1; i < n; ++i) { /* sigma = x(2:n)^T x(2:n), ascending */
    md_mul(m, &x[i * m], &x[i * m], t);
    md_add(m, sigma, t, sigma);
  }
  md_copy(m, &x[0], x1);
  md_set_d(m, 1.0, &v[0]);
  for (int64_t i = 1; i < n; ++i) md_copy(m, &x[i * m], &v[i * m]);
  if (md_lead(sigma) == 0.0) {
    md_zero(m, beta);
    md_copy(m, x1, mu);
    return;
  }
  double x1sq[MAXM], mu_[MAXM], v1[MAXM], v1sq[MAXM], num[MAXM], den[MAXM];
  md_mul(m, x1, x1, x1sq);
  md_add(m, x1sq, sigma, t);
  md_sqrt(m, t, mu_); /* mu = sqrt(x1^2 + sigma) */
  if (md_lead(x1) <= 0.0) {
    md_sub(m, x1, mu_, v1); /* v1 = x1 - mu */
  } else {
    double ns[MAXM];
    md_neg(m, sigma, ns);
    md_add(m, x1, mu_, t);
    md_div(m, ns, t, v1); /* v1 = -sigma / (x1 + mu) */
  }
  md_mul(m, v1, v1, v1sq);
  double two[MAXM];
  md_set_d(m, 2.0, two);
  md_mul(m, two, v1sq, num);
  md_add(m, sigma, v1sq, den);
  md_div(m, num, den, beta); /* beta = 2 v1^2 / (sigma + v1^2) */
  for (int64_t i = 1; i < n; ++i) md_div(m, &v[i * m], v1, &v[i * m]); /* v = v / v1 */
  md_copy(m, mu_, mu);
}

int oracle_house(int m, int64_t n, const double *x_planes, double *v_planes, double *beta, double *mu) {
  if (BAD_M(m)) return -2;
  double *x = malloc(sizeof(double) * m * n), *v = malloc(sizeof(double) * m * n);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) x[i * m + k] = x_planes[k * n + i];
  house(m, n, x, v, beta, mu);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) v_planes[k * n + i] = v[i * m + k];
  free(x);
  free(v);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* unblocked Householder QR (GVL Alg. 5.2.1)                                  */
/* A (M x K, ld >= M): on exit R in the upper triangle (R_jj = mu, the        */
/* sub-diagonal part of column j holds v_j(2:), v_j(1) = 1 implicit);          */
/* beta: m planes of K.  Every dot product accumulates from 0 ascending.       */
/* ------------------------------------------------------------------------- */
int oracle_qr(int m, int64_t M, int64_t K, double *Ap, int64_t lda, double *beta_p, int nthreads) {
  if (BAD_M(m)) return -2;
  if (M < K || K < 0 || lda < M) return -1;
  set_threads(nthreads);
  mat_t A = {Ap, lda, K, m};
  double *x = malloc(sizeof(double) * m * (M + 1));
  double *v = malloc(sizeof(double) * m * (M + 1));
  for (int64_t j = 0; j < K; ++j) {
    int64_t n = M - j;
    for (int64_t i = 0; i < n; ++i) get(&A, j + i, j, &x[i * m]);
    double beta[MAXM], mu[MAXM];
    house(m, n, x, v, beta, mu);
    /* apply P = I - beta v v^T to the columns c > j (independent: threaded) */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = j + 1; c < K; ++c) {
      double s[MAXM], t[MAXM], a[MAXM], w[MAXM];
      md_zero(m, s);
      for (int64_t i = 0; i < n; ++i) { /* s = v . A(j:M, c) */
        get(&A, j + i, c, a);
        md_mul(m, &v[i * m], a, t);
        md_add(m, s, t, s);
      }
      md_mul(m, beta, s, w); /* w = beta * s */
      for (int64_t i = 0; i < n; ++i) { /* A(j:M, c) -= w v */
        get(&A, j + i, c, a);
        md_mul(m, w, &v[i * m], t);
        md_sub(m, a, t, a);
        put(&A, j + i, c, a);
      }
    }
    put(&A, j, j, mu);
    for (int64_t i = 1; i < n; ++i) put(&A, j + i, j, &v[i * m]);
    for (int k = 0; k < m; ++k) beta_p[k * K + j] = beta[k];
  }
  free(x);
  free(v);
  return 0;
}

/* load v_j (full length M-j, v_j(1) = 1) from the factored A */
static void load_v(const mat_t *A, int64_t M, int64_t j, double *v) {
  int m = A->m;
  md_set_d(m, 1.0, &v[0]);
  for (int64_t i = 1; i < M - j; ++i) get(A, j + i, j, &v[i * m]);
}

/* Q = H_1 H_2 ... H_K, accumulated backward: Q = I; for j = K..1:
 * Q(j:M, c) -= beta_j (v_j . Q(j:M, c)) v_j for the columns c >= j. */
int oracle_form_q(int m, int64_t M, int64_t K, const double *Ap, int64_t lda, const double *beta_p, double *Qp,
                  int64_t ldq, int nthreads) {
  if (BAD_M(m)) return -2;
  if (M < K || ldq < M || lda < M) return -1;
  set_threads(nthreads);
  mat_t A = {(double *)Ap, lda, K, m};
  mat_t Q = {Qp, ldq, M, m};
  for (int k = 0; k < m; ++k) memset(Qp + (int64_t)k * ldq * M, 0, sizeof(double) * ldq * M);
  for (int64_t i = 0; i < M; ++i) Qp[i * ldq + i] = 1.0;
  double *v = malloc(sizeof(double) * m * (M + 1));
  for (int64_t j = K - 1; j >= 0; --j) {
    int64_t n = M - j;
    load_v(&A, M, j, v);
    double beta[MAXM];
    for (int k = 0; k < m; ++k) beta[k] = beta_p[k * K + j];
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t c = j; c < M; ++c) {
      double s[MAXM], t[MAXM], a[MAXM], w[MAXM];
      md_zero(m, s);
      for (int64_t i = 0; i < n; ++i) {
        get(&Q, j + i, c, a);
        md_mul(m, &v[i * m], a, t);
        md_add(m, s, t, s);
      }
      md_mul(m, beta, s, w);
      for (int64_t i = 0; i < n; ++i) {
        get(&Q, j + i, c, a);
        md_mul(m, w, &v[i * m], t);
        md_sub(m, a, t, a);
        put(&Q, j + i, c, a);
      }
    }
  }
  free(v);
  return 0;
}

/* y = Q^T b by applying the reflectors: y = b; for j = 1..K:
 * y(j:M) -= beta_j (v_j . y(j:M)) v_j. */
int oracle_apply_qt(int m, int64_t M, int64_t K, const double *Ap, int64_t lda, const double *beta_p,
                    const double *b, double *y) {
  if (BAD_M(m)) return -2;
  mat_t A = {(double *)Ap, lda, K, m};
  mat_t Y = {y, M, 1, m};
  if (y != b) memcpy(y, b, sizeof(double) * m * M);
  double *v = malloc(sizeof(double) * m * (M + 1));
  for (int64_t j = 0; j < K; ++j) {
    int64_t n = M - j;
    load_v(&A, M, j, v);
    double beta[MAXM], s[MAXM], t[MAXM], a[MAXM], w[MAXM];
    for (int k = 0; k < m; ++k) beta[k] = beta_p[k * K + j];
    md_zero(m, s);
    for (int64_t i = 0; i < n; ++i) {
      get(&Y, j + i, 0, a);
      md_mul(m, &v[i * m], a, t);
      md_add(m, s, t, s);
    }
    md_mul(m, beta, s, w);
    for (int64_t i = 0; i < n; ++i) {
      get(&Y, j + i, 0, a);
      md_mul(m, w, &v[i * m], t);
      md_sub(m, a, t, a);
      put(&Y, j + i, 0, a);
    }
  }
  free(v);
  return 0;
}

/* y = Q^T b with an explicit Q (y_c = sum_i Q(i,c) b_i, ascending i). */
int oracle_qt_b_explicit(int m, int64_t M, const double *Qp, int64_t ldq, const double *b, double *y,
                         int nthreads) {
  if (BAD_M(m)) return -2;
  set_threads(nthreads);
  mat_t Q = {(double *)Qp, ldq, M, m};
  mat_t B = {(double *)b, M, 1, m};
  double *out = malloc(sizeof(double) * m * M);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < M; ++c) {
    double s[MAXM], t[MAXM], q[MAXM], bb[MAXM];
    md_zero(m, s);
    for (int64_t i = 0; i < M; ++i) {
      get(&Q, i, c, q);
      get(&B, i, 0, bb);
      md_mul(m, q, bb, t);
      md_add(m, s, t, s);
    }
    for (int k = 0; k < m; ++k) out[k * M + c] = s[k];
  }
  memcpy(y, out, sizeof(double) * m * M);
  free(out);
  return 0;
}

/* plain back substitution on the leading n x n of R: for i = n..1:
 * s = y_i; for l = i+1..n: s -= R_il x_l; x_i = s / R_ii.
 * Returns 0, or i+1 (1-based) for the first zero diagonal met. */
int oracle_backsub(int m, int64_t n, const double *Rp, int64_t ldr, int64_t rcols, const double *y, int64_t ylen,
                   double *x) {
  if (BAD_M(m)) return -2;
  mat_t R = {(double *)Rp, ldr, rcols, m};
  double *xx = malloc(sizeof(double) * m * (n + 1));
  int info = 0;
  for (int64_t i = n - 1; i >= 0; --i) {
    double s[MAXM], t[MAXM], r[MAXM];
    for (int k = 0; k < m; ++k) s[k] = y[k * ylen + i];
    for (int64_t l = i + 1; l < n; ++l) {
      get(&R, i, l, r);
      md_mul(m, r, &xx[l * m], t);
      md_sub(m, s, t, s);
    }
    get(&R, i, i, r);
    if (r[0] == 0.0 && !info) info = (int)(i + 1);
    md_div(m, s, r, &xx[i * m]);
  }
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) x[k * n + i] = xx[i * m + k];
  free(xx);
  return info;
}

/* md dot product s = sum_i a_i b_i accumulated from 0 in ascending i (n entries,
 * planes pa / pb apart, strides sa / sb between entries) */
int oracle_dot(int m, int64_t n, const double *a, int64_t pa, int64_t sa, const double *b, int64_t pb, int64_t sb,
               double *out) {
  if (BAD_M(m)) return -2;
  double s[MAXM], t[MAXM], x[MAXM], y[MAXM];
  md_zero(m, s);
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < m; ++k) {
      x[k] = a[k * pa + i * sa];
      y[k] = b[k * pb + i * sb];
    }
    md_mul(m, x, y, t);
    md_add(m, s, t, s);
  }
  md_copy(m, s, out);
  return 0;
}

/* ||y||_2 in md: s = sum_i y_i^2 ascending from 0, then md sqrt (the residual norm of SPEC S:448 when
 * y = (Q^T b)(K+1:M)) */
int oracle_norm2(int m, int64_t n, const double *y, int64_t psy, double *out) {
  if (BAD_M(m)) return -2;
  double s[MAXM], t[MAXM], v[MAXM];
  md_zero(m, s);
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < m; ++k) v[k] = y[k * psy + i];
    md_mul(m, v, v, t);
    md_add(m, s, t, s);
  }
  md_sqrt(m, s, out);
  return 0;
}

/* ||b - A x||_2 in md, evaluated directly: r_i = b_i - sum_j A_ij x_j (ascending j), then oracle_norm2 */
int oracle_residual_direct(int m, int64_t M, int64_t K, const double *Ap, int64_t lda, const double *x,
                           const double *b, double *out) {
  if (BAD_M(m)) return -2;
  mat_t A = {(double *)Ap, lda, K, m};
  double *r = malloc(sizeof(double) * m * M);
  for (int64_t i = 0; i < M; ++i) {
    double s[MAXM], t[MAXM], a[MAXM], xx[MAXM];
    for (int k = 0; k < m; ++k) s[k] = b[k * M + i];
    for (int64_t j = 0; j < K; ++j) {
      get(&A, i, j, a);
      for (int k = 0; k < m; ++k) xx[k] = x[k * K + j];
      md_mul(m, a, xx, t);
      md_sub(m, s, t, s);
    }
    for (int k = 0; k < m; ++k) r[k * M + i] = s[k];
  }
  int rc = oracle_norm2(m, M, r, M, out);
  free(r);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* least squares: A = QR (A copied), y = Q^T b (reflectors), R x = y(1:K)      */
/* ------------------------------------------------------------------------- */
int oracle_lstsq(int m, int64_t M, int64_t K, const double *Ap, int64_t lda, const double *b, double *x,
                 double *R_out, double *y_out, int nthreads) {
  if (BAD_M(m)) return -2;
  double *F = malloc(sizeof(double) * m * M * K);
  for (int k = 0; k < m; ++k)
    for (int64_t j = 0; j < K; ++j)
      memcpy(F + (int64_t)k * M * K + j * M, Ap + (int64_t)k * lda * K + j * lda, sizeof(double) * M);
  double *beta = malloc(sizeof(double) * m * K);
  double *y = malloc(sizeof(double) * m * M);
  int rc = oracle_qr(m, M, K, F, M, beta, nthreads);
  if (!rc) rc = oracle_apply_qt(m, M, K, F, M, beta, b, y);
  if (!rc) rc = oracle_backsub(m, K, F, M, K, y, M, x);
  if (R_out) {
    for (int k = 0; k < m; ++k)
      for (int64_t j = 0; j < K; ++j)
        for (int64_t i = 0; i < M; ++i)
          R_out[(int64_t)k * M * K + j * M + i] = (i <= j) ? F[(int64_t)k * M * K + j * M + i] : 0.0;
  }
  if (y_out) memcpy(y_out, y, sizeof(double) * m * M);
  free(F);
  free(beta);
  free(y);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* invariants (computed in md, returned as the leading limb)                  */
/* ------------------------------------------------------------------------- */

/* E1 = max |Q^T Q - I| over the columns listed (all when cols == NULL). */
double oracle_inv_orth(int m, int64_t M, const double *Qp, int64_t ldq, const int64_t *cols, int64_t ncols,
                       int nthreads) {
  set_threads(nthreads);
  mat_t Q = {(double *)Qp, ldq, M, m};
  int64_t nc = cols ? ncols : M;
  double worst = 0.0;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : worst)
  for (int64_t cc = 0; cc < nc; ++cc) {
    int64_t c = cols ? cols[cc] : cc;
    for (int64_t r = 0; r < M; ++r) {
      double s[MAXM], t[MAXM], a[MAXM], b[MAXM], one[MAXM];
      md_zero(m, s);
      for (int64_t i = 0; i < M; ++i) {
        get(&Q, i, r, a);
        get(&Q, i, c, b);
        md_mul(m, a, b, t);
        md_add(m, s, t, s);
      }
      if (r == c) {
        md_set_d(m, 1.0, one);
        md_sub(m, s, one, s);
      }
      double e = fabs(s[0]);
      if (e > worst) worst = e;
    }
  }
  return worst;
}

/* E2 = max |A - Q R| / max |A| over the listed columns (R upper K x K block in an M x K array). */
double oracle_inv_recon(int m, int64_t M, int64_t K, const double *Ap, int64_t lda, const double *Qp, int64_t ldq,
                        const double *Rp, int64_t ldr, const int64_t *cols, int64_t ncols, int nthreads) {
  set_threads(nthreads);
  mat_t A = {(double *)Ap, lda, K, m}, Q = {(double *)Qp, ldq, M, m}, R = {(double *)Rp, ldr, K, m};
  int64_t nc = cols ? ncols : K;
  double worst = 0.0, amax = 0.0;
  for (int64_t j = 0; j < K; ++j)
    for (int64_t i = 0; i < M; ++i) {
      double a = fabs(Ap[j * lda + i]);
      if (a > amax) amax = a;
    }
#pragma omp parallel for schedule(dynamic, 1) reduction(max : worst)
  for (int64_t cc = 0; cc < nc; ++cc) {
    int64_t c = cols ? cols[cc] : cc;
    for (int64_t i = 0; i < M; ++i) {
      double s[MAXM], t[MAXM], q[MAXM], r[MAXM], a[MAXM];
      md_zero(m, s);
      for (int64_t l = 0; l <= c; ++l) {
        get(&Q, i, l, q);
        get(&R, l, c, r);
        md_mul(m, q, r, t);
        md_add(m, s, t, s);
      }
      get(&A, i, c, a);
      md_sub(m, a, s, s);
      double e = fabs(s[0]);
      if (e > worst) worst = e;
    }
  }
  return amax > 0 ? worst / amax : worst;
}

/* E3 = ||A^T (b - A x)||_inf / (||A||_inf (||A||_inf ||x||_inf + ||b||_inf)). */
double oracle_inv_normal(int m, int64_t M, int64_t K, const double *Ap, int64_t lda, const double *x,
                         const double *b, int nthreads) {
  set_threads(nthreads);
  mat_t A = {(double *)Ap, lda, K, m};
  double *r = malloc(sizeof(double) * m * M);
  double anorm = 0.0, xnorm = 0.0, bnorm = 0.0;
#pragma omp parallel for schedule(static) reduction(max : anorm)
  for (int64_t i = 0; i < M; ++i) { /* r = b - A x, and the row sums of |A| */
    double s[MAXM], t[MAXM], a[MAXM], xx[MAXM];
    for (int k = 0; k < m; ++k) s[k] = b[k * M + i];
    double rowsum = 0.0;
    for (int64_t j = 0; j < K; ++j) {
      get(&A, i, j, a);
      for (int k = 0; k < m; ++k) xx[k] = x[k * K + j];
      md_mul(m, a, xx, t);
      md_sub(m, s, t, s);
      rowsum += fabs(a[0]);
    }
    for (int k = 0; k < m; ++k) r[k * M + i] = s[k];
    if (rowsum > anorm) anorm = rowsum;
  }
  for (int64_t j = 0; j < K; ++j) xnorm = fmax(xnorm, fabs(x[j]));
  for (int64_t i = 0; i < M; ++i) bnorm = fmax(bnorm, fabs(b[i]));
  double worst = 0.0;
#pragma omp parallel for schedule(static) reduction(max : worst)
  for (int64_t j = 0; j < K; ++j) { /* A^T r */
    double s[MAXM], t[MAXM], a[MAXM], rr[MAXM];
    md_zero(m, s);
    for (int64_t i = 0; i < M; ++i) {
      get(&A, i, j, a);
      for (int k = 0; k < m; ++k) rr[k] = r[k * M + i];
      md_mul(m, a, rr, t);
      md_add(m, s, t, s);
    }
    double e = fabs(s[0]);
    if (e > worst) worst = e;
  }
  free(r);
  double den = anorm * (anorm * xnorm + bnorm);
  return den > 0 ? worst / den : worst;
}

/* ------------------------------------------------------------------------- */
/* BLOCKED algorithms with per-stage md-operation counters (the A10 ledger     */
/* pin).  The paper accumulates, per kernel, the md operations it executes and */
/* prices them with Table 1.  These functions carry out Algorithm 2 */
/* (blocked Householder QR) and Algorithm 1 (tiled back             */
/* substitution) step by step in the paper's order and count every  */
/* md add/sub, mul, div and sqrt per stage.  They are single threaded (the     */
/* counters are plain globals) and slow; they serve the ledger pin and the     */
/* blocked == unblocked check (same result in exact        */
/* arithmetic).  Readings: Householder vector scaled by one        */
/* reciprocal 1/v1 then multiplications (Z5, the GPU's choice); every sum      */
/* accumulates from 0 unless it updates an existing entry; the trailing update */
/* is Y (W^T C), never forming Y W^T; Q backward; tile inverses exploit zeros. */
/* ------------------------------------------------------------------------- */
enum { ST_HOUSE, ST_PANEL, ST_WY, ST_TRAILING, ST_FORM_Q, ST_QTB, ST_INVERT, ST_MULINV, ST_BSUPDATE, N_ST };
static int64_t g_mdc[N_ST][4]; /* add (incl. sub), mul, div, sqrt per stage */
static int g_st;
static void c_add(int m, const double *a, const double *b, double *c) { g_mdc[g_st][0]++; md_add(m, a, b, c); }
static void c_sub(int m, const double *a, const double *b, double *c) { g_mdc[g_st][0]++; md_sub(m, a, b, c); }
static void c_mul(int m, const double *a, const double *b, double *c) { g_mdc[g_st][1]++; md_mul(m, a, b, c); }
static void c_div(int m, const double *a, const double *b, double *c) { g_mdc[g_st][2]++; md_div(m, a, b, c); }
static void c_sqrt(int m, const double *a, double *c) { g_mdc[g_st][3]++; md_sqrt(m, a, c); }

/* dense md matrix of r x c, contiguous m-limb records, column-major (scratch) */
#define EL(P, ld, i, j) (&(P)[(((int64_t)(j)) * (ld) + (i)) * m])

/* GVL Alg. 5.1.1 with the reciprocal reading (Z5): v = x * (1/v1).  Counts in
 * the current stage.  Returns 1 when the x1 <= 0 branch was taken (no division
 * for v1) and sigma != 0, else 0. */
static int bhouse(int m, int64_t n, const double *x, double *v, double *beta, double *mu) {
  double sigma[MAXM], t[MAXM];
  md_zero(m, sigma);
  for (int64_t i = 1; i < n; ++i) {
    c_mul(m, &x[i * m], &x[i * m], t);
    c_add(m, sigma, t, sigma);
  }
  md_set_d(m, 1.0, &v[0]);
  if (md_lead(sigma) == 0.0) { /* P = I (GVL: beta = 0) */
    for (int64_t i = 1; i < n; ++i) md_copy(m, &x[i * m], &v[i * m]);
    md_zero(m, beta);
    md_copy(m, &x[0], mu);
    return 0;
  }
  double x1sq[MAXM], v1[MAXM], v1sq[MAXM], num[MAXM], den[MAXM], two[MAXM], one[MAXM], rv1[MAXM];
  int nonpos = 0;
  c_mul(m, &x[0], &x[0], x1sq);
  c_add(m, x1sq, sigma, t);
  c_sqrt(m, t, mu);
  if (md_lead(&x[0]) <= 0.0) {
    c_sub(m, &x[0], mu, v1);
    nonpos = 1;
  } else {
    double ns[MAXM];
    md_neg(m, sigma, ns);
    c_add(m, &x[0], mu, t);
    c_div(m, ns, t, v1);
  }
  c_mul(m, v1, v1, v1sq);
  md_set_d(m, 2.0, two);
  c_mul(m, two, v1sq, num);
  c_add(m, sigma, v1sq, den);
  c_div(m, num, den, beta);
  md_set_d(m, 1.0, one);
  c_div(m, one, v1, rv1);
  for (int64_t i = 1; i < n; ++i) c_mul(m, &x[i * m], rv1, &v[i * m]);
  return nonpos;
}

/* Algorithm 2 on F (M x K, limb-planar, ld M): R over F (v below the diagonal),
 * Y and W of every panel kept in Yall / Wall (M x K dense records, panel k in
 * rows j0.., columns j0..j0+nb-1), beta (K records).  *nonpos += columns that
 * took the x1 <= 0 branch. */
static void blocked_qr(int m, int64_t M, int64_t K, int64_t nb, mat_t *F, double *Yall, double *Wall, double *betas,
                       int64_t *nonpos) {
  const int64_t N = K / nb;
  double *x = malloc(sizeof(double) * m * (M + 1)), *v = malloc(sizeof(double) * m * (M + 1));
  double *tv = malloc(sizeof(double) * m * (nb + 1));
  double *T = malloc(sizeof(double) * m * nb * (K + 1));
  for (int64_t k = 0; k < N; ++k) {
    const int64_t j0 = k * nb, r = M - j0, ct = K - j0 - nb;
    /* step 1: for l = 1..n: v, beta; update R_kk */
    for (int64_t l = 0; l < nb; ++l) {
      const int64_t j = j0 + l, n = M - j;
      for (int64_t i = 0; i < n; ++i) get(F, j + i, j, &x[i * m]);
      double beta[MAXM], mu[MAXM];
      g_st = ST_HOUSE;
      *nonpos += bhouse(m, n, x, v, beta, mu);
      g_st = ST_PANEL;
      for (int64_t c = j + 1; c < j0 + nb; ++c) { /* beta R^T v, then R -= v w^T on the panel */
        double s[MAXM], t[MAXM], a[MAXM], w[MAXM];
        md_zero(m, s);
        for (int64_t i = 0; i < n; ++i) {
          get(F, j + i, c, a);
          c_mul(m, &v[i * m], a, t);
          c_add(m, s, t, s);
        }
        c_mul(m, beta, s, w);
        for (int64_t i = 0; i < n; ++i) {
          get(F, j + i, c, a);
          c_mul(m, w, &v[i * m], t);
          c_sub(m, a, t, a);
          put(F, j + i, c, a);
        }
      }
      put(F, j, j, mu);
      for (int64_t i = 1; i < n; ++i) put(F, j + i, j, &v[i * m]);
      md_copy(m, beta, &betas[j * m]);
      /* Y(:, l) = v (rows j0.., zeros above row j) */
      for (int64_t i = 0; i < r; ++i) {
        if (i < l) md_zero(m, EL(Yall, M, j0 + i, j));
        else md_copy(m, &v[(i - l) * m], EL(Yall, M, j0 + i, j));
      }
    }
    /* step 2: W by z = -beta (v + W Y^T v), column by column */
    g_st = ST_WY;
    for (int64_t l = 0; l < nb; ++l) {
      const int64_t j = j0 + l;
      double nbeta[MAXM];
      md_neg(m, &betas[j * m], nbeta);
      for (int64_t p = 0; p < l; ++p) { /* t_p = Y_p^T v_l over the rows where v_l is nonzero */
        double s[MAXM], t[MAXM];
        md_zero(m, s);
        for (int64_t i = l; i < r; ++i) {
          c_mul(m, EL(Yall, M, j0 + i, j0 + p), EL(Yall, M, j0 + i, j), t);
          c_add(m, s, t, s);
        }
        md_copy(m, s, &tv[p * m]);
      }
      for (int64_t i = 0; i < r; ++i) {
        double u[MAXM], t[MAXM], z[MAXM];
        md_zero(m, u);
        for (int64_t p = 0; p < l; ++p) { /* u_i = (W t)_i */
          c_mul(m, EL(Wall, M, j0 + i, j0 + p), &tv[p * m], t);
          c_add(m, u, t, u);
        }
        c_add(m, EL(Yall, M, j0 + i, j), u, z); /* v + W Y^T v */
        c_mul(m, nbeta, z, EL(Wall, M, j0 + i, j));
      }
    }
    /* step 4: if k < N, R := R + Y (W^T C) on the trailing columns */
    if (ct > 0) {
      g_st = ST_TRAILING;
      for (int64_t c = 0; c < ct; ++c) {
        for (int64_t p = 0; p < nb; ++p) { /* T = W^T C */
          double s[MAXM], t[MAXM], a[MAXM];
          md_zero(m, s);
          for (int64_t i = 0; i < r; ++i) {
            get(F, j0 + i, j0 + nb + c, a);
            c_mul(m, EL(Wall, M, j0 + i, j0 + p), a, t);
            c_add(m, s, t, s);
          }
          md_copy(m, s, EL(T, nb, p, c));
        }
      }
      for (int64_t c = 0; c < ct; ++c)
        for (int64_t i = 0; i < r; ++i) { /* C += Y T */
          double s[MAXM], t[MAXM];
          get(F, j0 + i, j0 + nb + c, s);
          for (int64_t p = 0; p < nb; ++p) {
            c_mul(m, EL(Yall, M, j0 + i, j0 + p), EL(T, nb, p, c), t);
            c_add(m, s, t, s);
          }
          put(F, j0 + i, j0 + nb + c, s);
        }
    }
  }
  free(x);
  free(v);
  free(tv);
  free(T);
}

/* Q = P_WY(1) ... P_WY(N) backward: Q = I; for k = N..1: Q_tr += W_k (Y_k^T Q_tr),
 * Q_tr = Q(j0:M, j0:M) (the paper forms Q forward; equal in exact arithmetic) */
static void blocked_form_q(int m, int64_t M, int64_t K, int64_t nb, const double *Yall, const double *Wall, mat_t *Q) {
  const int64_t N = K / nb;
  for (int k = 0; k < m; ++k) memset(Q->p + (int64_t)k * Q->ld * Q->cols, 0, sizeof(double) * Q->ld * Q->cols);
  for (int64_t i = 0; i < M; ++i) Q->p[i * Q->ld + i] = 1.0;
  double *X = malloc(sizeof(double) * m * nb * (M + 1));
  g_st = ST_FORM_Q;
  for (int64_t k = N - 1; k >= 0; --k) {
    const int64_t j0 = k * nb, r = M - j0;
    for (int64_t c = 0; c < r; ++c)
      for (int64_t p = 0; p < nb; ++p) { /* X = Y_k^T Q_tr */
        double s[MAXM], t[MAXM], q[MAXM];
        md_zero(m, s);
        for (int64_t i = 0; i < r; ++i) {
          get(Q, j0 + i, j0 + c, q);
          c_mul(m, EL(Yall, M, j0 + i, j0 + p), q, t);
          c_add(m, s, t, s);
        }
        md_copy(m, s, EL(X, nb, p, c));
      }
    for (int64_t c = 0; c < r; ++c)
      for (int64_t i = 0; i < r; ++i) { /* Q_tr += W_k X */
        double s[MAXM], t[MAXM];
        get(Q, j0 + i, j0 + c, s);
        for (int64_t p = 0; p < nb; ++p) {
          c_mul(m, EL(Wall, M, j0 + i, j0 + p), EL(X, nb, p, c), t);
          c_add(m, s, t, s);
        }
        put(Q, j0 + i, j0 + c, s);
      }
  }
  free(X);
}

/* Algorithm 1 on the leading n x n of U (limb-planar, ld ldu,
 * ucols columns): invert the N diagonal tiles (zeros exploited: column k of
 * U_i^-1 solves U_i v = e_k, v_k = 1/u_kk, v_r = -(sum_{l=r+1..k} u_rl v_l) / u_rr
 * with the reciprocals 1/u_rr formed once per tile), then for
 * i = N..1: x_i = U_i^-1 b_i, b_j -= A_ji x_i (j < i).  Returns 0 or the 1-based
 * first zero diagonal. */
static int blocked_backsub(int m, int64_t n, int64_t nb, const mat_t *U, const double *y, double *x) {
  const int64_t N = n / nb;
  double *V = malloc(sizeof(double) * m * nb * nb * (N + 1)); /* tile i at V + i nb^2 m, nb x nb */
  double *d = malloc(sizeof(double) * m * (nb + 1));
  double *b = malloc(sizeof(double) * m * (n + 1));
  int info = 0;
  g_st = ST_INVERT;
  for (int64_t ti = 0; ti < N; ++ti) {
    const int64_t o = ti * nb;
    double *Vi = V + ti * nb * nb * m;
    double one[MAXM], u[MAXM];
    md_set_d(m, 1.0, one);
    for (int64_t rr = 0; rr < nb; ++rr) {
      get(U, o + rr, o + rr, u);
      if (u[0] == 0.0 && !info) info = (int)(o + rr + 1);
      c_div(m, one, u, &d[rr * m]);
    }
    for (int64_t k = 0; k < nb; ++k) {
      for (int64_t rr = k + 1; rr < nb; ++rr) md_zero(m, EL(Vi, nb, rr, k));
      md_copy(m, &d[k * m], EL(Vi, nb, k, k));
      for (int64_t rr = k - 1; rr >= 0; --rr) {
        double s[MAXM], t[MAXM], ns[MAXM];
        md_zero(m, s);
        for (int64_t l = rr + 1; l <= k; ++l) {
          get(U, o + rr, o + l, u);
          c_mul(m, u, EL(Vi, nb, l, k), t);
          c_add(m, s, t, s);
        }
        md_neg(m, s, ns);
        c_mul(m, ns, &d[rr * m], EL(Vi, nb, rr, k));
      }
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) b[i * m + k] = y[(int64_t)k * n + i];
  for (int64_t ti = N - 1; ti >= 0; --ti) {
    const int64_t o = ti * nb;
    const double *Vi = V + ti * nb * nb * m;
    g_st = ST_MULINV;
    for (int64_t rr = 0; rr < nb; ++rr) { /* x_i = U_i^-1 b_i */
      double s[MAXM], t[MAXM];
      md_zero(m, s);
      for (int64_t c = rr; c < nb; ++c) {
        c_mul(m, EL(Vi, nb, rr, c), &b[(o + c) * m], t);
        c_add(m, s, t, s);
      }
      for (int k = 0; k < m; ++k) x[(int64_t)k * n + o + rr] = s[k];
    }
    g_st = ST_BSUPDATE;
    for (int64_t tj = 0; tj < ti; ++tj) /* b_j -= A_ji x_i */
      for (int64_t rr = 0; rr < nb; ++rr) {
        double *s = &b[(tj * nb + rr) * m], t[MAXM], a[MAXM], xx[MAXM];
        for (int64_t c = 0; c < nb; ++c) {
          get(U, tj * nb + rr, o + c, a);
          for (int k = 0; k < m; ++k) xx[k] = x[(int64_t)k * n + o + c];
          c_mul(m, a, xx, t);
          c_sub(m, s, t, s);
        }
      }
  }
  free(V);
  free(d);
  free(b);
  return info;
}

/* The blocked pipelines the ledger prices (op codes as MDLS_OP_* of include/mdls.h:
 * 0 QR with Q formed, 1 BACKSUB, 2 LSTSQ = QR + Q + explicit Q^T b + BS, 3 APPLY_QT
 * (Q^T b from the panels, after a QR whose counts are discarded), 4 LSTSQ_NOQ = QR +
 * Q^T b from the panels + BS).  A: M x K (ld M) or, for BACKSUB, the upper
 * triangular K x K; b: M (or K).  Outputs (nullable): x (K), R (M x K, strictly
 * lower part zero), Q (M x M), y = Q^T b (M).  counts: int64[9][4] (add, mul, div,
 * sqrt per stage, MDLS_ST_* order); nonpos: columns with x1 <= 0 and sigma != 0.
 * Returns 0, a 1-based zero-diagonal row, or -1 for invalid arguments. */
int oracle_blocked(int op, int m, int64_t M, int64_t K, int64_t nb, const double *A, const double *b, double *x,
                   double *R_out, double *Q_out, double *y_out, int64_t *counts, int64_t *nonpos) {
  if (BAD_M(m)) return -1;
  if (nb < 1 || K < 1 || K % nb || (op != 1 && M < K) || op < 0 || op > 4) return -1;
  memset(g_mdc, 0, sizeof(g_mdc));
  int64_t np = 0;
  int info = 0;
  if (op == 1) {
    mat_t U = {(double *)A, K, K, m};
    double *xx = x ? x : malloc(sizeof(double) * m * K);
    info = blocked_backsub(m, K, nb, &U, b, xx);
    if (!x) free(xx);
  } else {
    double *F = malloc(sizeof(double) * m * M * K);
    memcpy(F, A, sizeof(double) * m * M * K);
    mat_t Fm = {F, M, K, m};
    double *Yall = calloc((size_t)m * M * K, sizeof(double)), *Wall = calloc((size_t)m * M * K, sizeof(double));
    double *betas = malloc(sizeof(double) * m * K);
    blocked_qr(m, M, K, nb, &Fm, Yall, Wall, betas, &np);
    double *Q = NULL;
    if (op == 0 || op == 2) {
      Q = Q_out ? Q_out : malloc(sizeof(double) * m * M * M);
      mat_t Qm = {Q, M, M, m};
      blocked_form_q(m, M, K, nb, Yall, Wall, &Qm);
    }
    if (op == 3) memset(g_mdc, 0, sizeof(g_mdc)); /* APPLY_QT prices only the application */
    double *y = malloc(sizeof(double) * m * M);
    if (op >= 2) {
      g_st = ST_QTB;
      if (op == 2) { /* explicit: y_c = sum_i Q_ic b_i */
        mat_t Qm = {Q, M, M, m};
        for (int64_t c = 0; c < M; ++c) {
          double s[MAXM], t[MAXM], q[MAXM], bb[MAXM];
          md_zero(m, s);
          for (int64_t i = 0; i < M; ++i) {
            get(&Qm, i, c, q);
            for (int k = 0; k < m; ++k) bb[k] = b[(int64_t)k * M + i];
            c_mul(m, q, bb, t);
            c_add(m, s, t, s);
          }
          for (int k = 0; k < m; ++k) y[(int64_t)k * M + c] = s[k];
        }
      } else { /* by panels: y(j0:) += Y_k (W_k^T y(j0:)) */
        memcpy(y, b, sizeof(double) * m * M);
        mat_t Ym = {y, M, 1, m};
        double *tv = malloc(sizeof(double) * m * (nb + 1));
        for (int64_t k = 0; k < K / nb; ++k) {
          const int64_t j0 = k * nb, r = M - j0;
          for (int64_t p = 0; p < nb; ++p) {
            double s[MAXM], t[MAXM], a[MAXM];
            md_zero(m, s);
            for (int64_t i = 0; i < r; ++i) {
              get(&Ym, j0 + i, 0, a);
              c_mul(m, EL(Wall, M, j0 + i, j0 + p), a, t);
              c_add(m, s, t, s);
            }
            md_copy(m, s, &tv[p * m]);
          }
          for (int64_t i = 0; i < r; ++i) {
            double s[MAXM], t[MAXM];
            get(&Ym, j0 + i, 0, s);
            for (int64_t p = 0; p < nb; ++p) {
              c_mul(m, EL(Yall, M, j0 + i, j0 + p), &tv[p * m], t);
              c_add(m, s, t, s);
            }
            put(&Ym, j0 + i, 0, s);
          }
        }
        free(tv);
      }
      if (y_out) memcpy(y_out, y, sizeof(double) * m * M);
    }
    if (op == 2 || op == 4) { /* R(1:K, 1:K) x = y(1:K) by Algorithm 1 */
      double *yk = malloc(sizeof(double) * m * K);
      for (int k = 0; k < m; ++k) memcpy(yk + (int64_t)k * K, y + (int64_t)k * M, sizeof(double) * K);
      double *Rk = malloc(sizeof(double) * m * K * K);
      for (int k = 0; k < m; ++k)
        for (int64_t j = 0; j < K; ++j)
          for (int64_t i = 0; i < K; ++i)
            Rk[(int64_t)k * K * K + j * K + i] = (i <= j) ? F[(int64_t)k * M * K + j * M + i] : 0.0;
      mat_t U = {Rk, K, K, m};
      double *xx = x ? x : malloc(sizeof(double) * m * K);
      info = blocked_backsub(m, K, nb, &U, yk, xx);
      if (!x) free(xx);
      free(yk);
      free(Rk);
    }
    if (R_out)
      for (int k = 0; k < m; ++k)
        for (int64_t j = 0; j < K; ++j)
          for (int64_t i = 0; i < M; ++i)
            R_out[(int64_t)k * M * K + j * M + i] = (i <= j) ? F[(int64_t)k * M * K + j * M + i] : 0.0;
    if (Q && Q != Q_out) free(Q);
    free(y);
    free(F);
    free(Yall);
    free(Wall);
    free(betas);
  }
  if (counts) memcpy(counts, g_mdc, sizeof(g_mdc));
  if (nonpos) *nonpos = np;
  return info;
}

/* ------------------------------------------------------------------------- */
/* complex least squares (row f2; "real and complex matrices",      */
/* P:384-385 real and imaginary parts kept separately, P:515-516 the          */
/* transpose replaced by the Hermitian transpose).  A complex md number is    */
/* the pair (re, im) of md numbers; arithmetic is the schoolbook definition:  */
/*   (a + bi)(c + di) = (ac - bd) + (ad + bc) i,   conj(a + bi) = a - bi,      */
/*   |z|^2 = a^2 + b^2,  1/z = conj(z) / |z|^2.                                */
/* Unblocked complex Householder QR: for column j, x = A(j:M, j),             */
/*   mu = ||x||_2 = sqrt(|x_1|^2 + sigma), sigma = sum_{i>1} |x_i|^2,         */
/*   phase = x_1 / |x_1| (1 when x_1 = 0), alpha = -phase mu,                 */
/*   v = x - alpha e_1 (v_1 = phase (|x_1| + mu), no cancellation),           */
/*   v <- v / v_1, beta = 2 / (v^H v),  H = I - beta v v^H (Hermitian,        */
/*   unitary), H x = alpha e_1, R_jj = alpha; sigma = 0 and Im x_1 = 0:        */
/*   H = I, R_jj = x_1.  Columns c > j: w = v^H a_c, a_c -= beta v w.         */
/* Q^H b by the reflectors in order, then complex back substitution.          */
/* Storage: re and im parts in separate limb-planar arrays.       */
/* ------------------------------------------------------------------------- */
static void z_mul(int m, const double *ar, const double *ai, const double *br, const double *bi, double *cr,
                  double *ci) {
  double t1[MAXM], t2[MAXM], t3[MAXM], t4[MAXM];
  md_mul(m, ar, br, t1);
  md_mul(m, ai, bi, t2);
  md_mul(m, ar, bi, t3);
  md_mul(m, ai, br, t4);
  md_sub(m, t1, t2, cr);
  md_add(m, t3, t4, ci);
}
/* conj(a) b */
static void z_cmul(int m, const double *ar, const double *ai, const double *br, const double *bi, double *cr,
                   double *ci) {
  double nai[MAXM];
  md_neg(m, ai, nai);
  z_mul(m, ar, nai, br, bi, cr, ci);
}
static void z_abs2(int m, const double *ar, const double *ai, double *c) {
  double t1[MAXM], t2[MAXM];
  md_mul(m, ar, ar, t1);
  md_mul(m, ai, ai, t2);
  md_add(m, t1, t2, c);
}
/* a / b = a conj(b) / |b|^2 */
static void z_div(int m, const double *ar, const double *ai, const double *br, const double *bi, double *cr,
                  double *ci) {
  double nbi[MAXM], tr[MAXM], ti[MAXM], d[MAXM];
  md_neg(m, bi, nbi);
  z_mul(m, ar, ai, br, nbi, tr, ti);
  z_abs2(m, br, bi, d);
  md_div(m, tr, d, cr);
  md_div(m, ti, d, ci);
}

int oracle_zlstsq(int m, int64_t M, int64_t K, const double *Are, const double *Aim, int64_t lda, const double *bre,
                  const double *bim, double *xre, double *xim, double *Rre, double *Rim) {
  if (BAD_M(m)) return -2;
  if (M < K || K < 1) return -3;
  /* working copies, element-major (m limbs contiguous): F(i, j) at ((j * M + i) * m) */
  double *Fr = malloc(sizeof(double) * m * M * K), *Fi = malloc(sizeof(double) * m * M * K);
  double *yr = malloc(sizeof(double) * m * M), *yi = malloc(sizeof(double) * m * M);
  double *vr = malloc(sizeof(double) * m * M), *vi = malloc(sizeof(double) * m * M);
  double *xr_ = malloc(sizeof(double) * m * K), *xi_ = malloc(sizeof(double) * m * K);
  for (int64_t j = 0; j < K; ++j)
    for (int64_t i = 0; i < M; ++i)
      for (int k = 0; k < m; ++k) {
        Fr[(j * M + i) * m + k] = Are[(int64_t)k * lda * K + j * lda + i];
        Fi[(j * M + i) * m + k] = Aim[(int64_t)k * lda * K + j * lda + i];
      }
  for (int64_t i = 0; i < M; ++i)
    for (int k = 0; k < m; ++k) {
      yr[i * m + k] = bre[(int64_t)k * M + i];
      yi[i * m + k] = bim[(int64_t)k * M + i];
    }
#define FR(i, j) (&Fr[((j) * M + (i)) * m])
#define FI(i, j) (&Fi[((j) * M + (i)) * m])
  int info = 0;
  for (int64_t j = 0; j < K; ++j) {
    const int64_t n = M - j;
    double sigma[MAXM], t[MAXM], a1[MAXM], mu[MAXM], beta[MAXM];
    md_zero(m, sigma);
    for (int64_t i = 1; i < n; ++i) { /* sigma = sum_{i>1} |x_i|^2, ascending */
      z_abs2(m, FR(j + i, j), FI(j + i, j), t);
      md_add(m, sigma, t, sigma);
    }
    const int identity = md_lead(sigma) == 0.0 && md_lead(FI(j, j)) == 0.0;
    if (identity) {
      md_zero(m, beta);
    } else {
      double x1r[MAXM], x1i[MAXM], pr[MAXM], pi[MAXM], ar[MAXM], ai[MAXM], v1r[MAXM], v1i[MAXM];
      md_copy(m, FR(j, j), x1r);
      md_copy(m, FI(j, j), x1i);
      z_abs2(m, x1r, x1i, t);
      md_sqrt(m, t, a1); /* |x_1| */
      md_add(m, t, sigma, t);
      md_sqrt(m, t, mu); /* mu = ||x|| */
      if (md_lead(a1) == 0.0) {
        md_set_d(m, 1.0, pr);
        md_zero(m, pi);
      } else {
        md_div(m, x1r, a1, pr);
        md_div(m, x1i, a1, pi);
      }
      md_mul(m, pr, mu, ar); /* alpha = -phase mu */
      md_neg(m, ar, ar);
      md_mul(m, pi, mu, ai);
      md_neg(m, ai, ai);
      md_add(m, a1, mu, t); /* v_1 = phase (|x_1| + mu) */
      md_mul(m, pr, t, v1r);
      md_mul(m, pi, t, v1i);
      /* v = x / v_1, v_1 = 1 */
      md_set_d(m, 1.0, &vr[0]);
      md_zero(m, &vi[0]);
      for (int64_t i = 1; i < n; ++i) z_div(m, FR(j + i, j), FI(j + i, j), v1r, v1i, &vr[i * m], &vi[i * m]);
      /* beta = 2 / (v^H v) */
      double vv[MAXM], two[MAXM];
      md_set_d(m, 1.0, vv);
      for (int64_t i = 1; i < n; ++i) {
        z_abs2(m, &vr[i * m], &vi[i * m], t);
        md_add(m, vv, t, vv);
      }
      md_set_d(m, 2.0, two);
      md_div(m, two, vv, beta);
      /* columns c > j: w = v^H a_c, a_c -= beta v w */
      for (int64_t c = j + 1; c < K; ++c) {
        double wr[MAXM], wi[MAXM], pr2[MAXM], pi2[MAXM];
        md_zero(m, wr);
        md_zero(m, wi);
        for (int64_t i = 0; i < n; ++i) {
          z_cmul(m, &vr[i * m], &vi[i * m], FR(j + i, c), FI(j + i, c), pr2, pi2);
          md_add(m, wr, pr2, wr);
          md_add(m, wi, pi2, wi);
        }
        md_mul(m, beta, wr, wr);
        md_mul(m, beta, wi, wi);
        for (int64_t i = 0; i < n; ++i) {
          z_mul(m, &vr[i * m], &vi[i * m], wr, wi, pr2, pi2);
          md_sub(m, FR(j + i, c), pr2, FR(j + i, c));
          md_sub(m, FI(j + i, c), pi2, FI(j + i, c));
        }
      }
      /* y = H y on rows j.. (Q^H b, reflectors in order) */
      {
        double wr[MAXM], wi[MAXM], pr2[MAXM], pi2[MAXM];
        md_zero(m, wr);
        md_zero(m, wi);
        for (int64_t i = 0; i < n; ++i) {
          z_cmul(m, &vr[i * m], &vi[i * m], &yr[(j + i) * m], &yi[(j + i) * m], pr2, pi2);
          md_add(m, wr, pr2, wr);
          md_add(m, wi, pi2, wi);
        }
        md_mul(m, beta, wr, wr);
        md_mul(m, beta, wi, wi);
        for (int64_t i = 0; i < n; ++i) {
          z_mul(m, &vr[i * m], &vi[i * m], wr, wi, pr2, pi2);
          md_sub(m, &yr[(j + i) * m], pr2, &yr[(j + i) * m]);
          md_sub(m, &yi[(j + i) * m], pi2, &yi[(j + i) * m]);
        }
      }
      md_copy(m, ar, FR(j, j));
      md_copy(m, ai, FI(j, j));
      for (int64_t i = 1; i < n; ++i) {
        md_zero(m, FR(j + i, j));
        md_zero(m, FI(j + i, j));
      }
    }
    if (md_lead(FR(j, j)) == 0.0 && md_lead(FI(j, j)) == 0.0 && !info) info = (int)(j + 1);
  }
  /* R x = y(1:K), complex back substitution */
  for (int64_t i = K - 1; i >= 0; --i) {
    double sr[MAXM], si[MAXM], pr2[MAXM], pi2[MAXM];
    md_copy(m, &yr[i * m], sr);
    md_copy(m, &yi[i * m], si);
    for (int64_t l = i + 1; l < K; ++l) {
      z_mul(m, FR(i, l), FI(i, l), &xr_[l * m], &xi_[l * m], pr2, pi2);
      md_sub(m, sr, pr2, sr);
      md_sub(m, si, pi2, si);
    }
    z_div(m, sr, si, FR(i, i), FI(i, i), &xr_[i * m], &xi_[i * m]);
  }
  for (int64_t i = 0; i < K; ++i)
    for (int k = 0; k < m; ++k) {
      xre[(int64_t)k * K + i] = xr_[i * m + k];
      xim[(int64_t)k * K + i] = xi_[i * m + k];
    }
  if (Rre && Rim)
    for (int64_t j = 0; j < K; ++j)
      for (int64_t i = 0; i < M; ++i)
        for (int k = 0; k < m; ++k) {
          Rre[(int64_t)k * M * K + j * M + i] = (i <= j) ? FR(i, j)[k] : 0.0;
          Rim[(int64_t)k * M * K + j * M + i] = (i <= j) ? FI(i, j)[k] : 0.0;
        }
#undef FR
#undef FI
  free(Fr);
  free(Fi);
  free(yr);
  free(yi);
  free(vr);
  free(vi);
  free(xr_);
  free(xi_);
  return info;
}

/* runtime self-check of round-to-nearest-even without reassociation:
 * two_sum(2^53, 1) must give (2^53, 1). */
int oracle_selfcheck(void) {
  double s, e;
  two_sum(9007199254740992.0, 1.0, &s, &e);
  return (s == 9007199254740992.0 && e == 1.0) ? 0 : 1;
}

/* silence unused-function warnings for helpers kept for completeness */
void oracle_unused_(void) {
  double a[MAXM] = {0}, b[MAXM] = {0};
  (void)md_lt(2, a, b);
  md_abs(2, a, b);
}
