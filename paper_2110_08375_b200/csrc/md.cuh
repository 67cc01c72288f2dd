// md.cuh -- device multiple-double arithmetic on the FP64 pipe (sm_100a).
//
// A multiple double is an unevaluated sum of M doubles, M = 2 (dd), 4 (qd),
// 8 (od), most significant first.  The operation families
// are the ones the paper names: QDlib for double double
// and CAMPARY's generated quad/octo double code, held in M separate
// scalar registers and force-inlined.  The exact
// variants are the readings listed in DESIGN.md ("md arithmetic readings");
// they are the variants whose base-operation tallies reproduce the paper's
// Table 1, with one deliberate change: two_prod uses the FMA
// (DMUL + DFMA) instead of Dekker's split, which returns the identical exact
// pair (p, e) in 2 instead of 17 FP64 operations.
//
// Every operation is written with explicit __dadd_rn / __dsub_rn / __dmul_rn /
// __fma_rn intrinsics so nvcc can never contract or reassociate an error-free
// transformation.  Renormalisation is branch-free (selects, integer zero
// tests) so warps never diverge inside the arithmetic.
#pragma once
#include <cstdint>

namespace mdls {

template <int M>
struct md {
  double v[M];
};

// ----------------------------------------------------------------------------
// error-free transformations
// ----------------------------------------------------------------------------
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  double ss = __dadd_rn(a, b);
  double bb = __dsub_rn(ss, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(ss, bb)), __dsub_rn(b, bb));
  s = ss;
}

// Fast2Sum, |a| >= |b| (or a == 0)
__device__ __forceinline__ void quick_two_sum(double a, double b, double& s, double& e) {
  double ss = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(ss, a));
  s = ss;
}

// exact product via the fused multiply-add: p + e == a*b
__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  double pp = __dmul_rn(a, b);
  e = __fma_rn(a, b, -pp);
  p = pp;
}

__device__ __forceinline__ bool nonzero(double x) {
  return (static_cast<unsigned long long>(__double_as_longlong(x)) << 1) != 0ull;
}

template <int M>
__device__ __forceinline__ md<M> md_zero() {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = 0.0;
  return r;
}

template <int M>
__device__ __forceinline__ md<M> md_from(double d) {
  md<M> r = md_zero<M>();
  r.v[0] = d;
  return r;
}

template <int M>
__device__ __forceinline__ md<M> neg(const md<M>& a) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = -a.v[k];
  return r;
}

// exact scaling by a power of two
template <int M>
__device__ __forceinline__ md<M> scale_pow2(const md<M>& a, double p2) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = __dmul_rn(a.v[k], p2);
  return r;
}

// ----------------------------------------------------------------------------
// double double (QDlib)
// ----------------------------------------------------------------------------
__device__ __forceinline__ md<2> dd_add(const md<2>& a, const md<2>& b) {
  double s1, s2, t1, t2;
  two_sum(a.v[0], b.v[0], s1, s2);
  two_sum(a.v[1], b.v[1], t1, t2);
  s2 = __dadd_rn(s2, t1);
  quick_two_sum(s1, s2, s1, s2);
  s2 = __dadd_rn(s2, t2);
  md<2> c;
  quick_two_sum(s1, s2, c.v[0], c.v[1]);
  return c;
}

__device__ __forceinline__ md<2> dd_mul(const md<2>& a, const md<2>& b) {
  double p1, p2;
  two_prod(a.v[0], b.v[0], p1, p2);
  p2 = __dadd_rn(p2, __dadd_rn(__dmul_rn(a.v[0], b.v[1]), __dmul_rn(a.v[1], b.v[0])));
  md<2> c;
  quick_two_sum(p1, p2, c.v[0], c.v[1]);
  return c;
}

__device__ __forceinline__ md<2> dd_mul_d(const md<2>& a, double b) {
  double p1, p2;
  two_prod(a.v[0], b, p1, p2);
  p2 = __dadd_rn(p2, __dmul_rn(a.v[1], b));
  md<2> c;
  quick_two_sum(p1, p2, c.v[0], c.v[1]);
  return c;
}

__device__ __forceinline__ md<2> dd_add_d(const md<2>& a, double b) {
  double s1, s2;
  two_sum(a.v[0], b, s1, s2);
  s2 = __dadd_rn(s2, a.v[1]);
  md<2> c;
  quick_two_sum(s1, s2, c.v[0], c.v[1]);
  return c;
}

// QDlib accurate division: three quotient digits
static __device__ __noinline__ md<2> dd_div(const md<2>& a, const md<2>& b) {
  double q1 = __ddiv_rn(a.v[0], b.v[0]);
  md<2> r = dd_add(a, neg(dd_mul_d(b, q1)));
  double q2 = __ddiv_rn(r.v[0], b.v[0]);
  r = dd_add(r, neg(dd_mul_d(b, q2)));
  double q3 = __ddiv_rn(r.v[0], b.v[0]);
  md<2> q;
  quick_two_sum(q1, q2, q.v[0], q.v[1]);
  return dd_add_d(q, q3);
}

// QDlib sqrt: one Newton correction of the double reciprocal square root
static __device__ __noinline__ md<2> dd_sqrt(const md<2>& a) {
  if (a.v[0] == 0.0) return md_zero<2>();
  double x = __ddiv_rn(1.0, __dsqrt_rn(a.v[0]));
  double ax = __dmul_rn(a.v[0], x);
  md<2> sq;
  two_prod(ax, ax, sq.v[0], sq.v[1]);
  md<2> d = dd_add(a, neg(sq));
  md<2> c;
  two_sum(ax, __dmul_rn(d.v[0], __dmul_rn(x, 0.5)), c.v[0], c.v[1]);
  return c;
}

// ----------------------------------------------------------------------------
// quad / octo double (CAMPARY fast family)
// ----------------------------------------------------------------------------

// fast_renorm2L<M+1, M>: bottom-up Fast2Sum sweep over f[0..M], then a
// top-down sweep over its first M outputs that emits a limb whenever the
// Fast2Sum error is nonzero; zero padded.  2M-1 Fast2Sums, branch-free.
template <int M>
__device__ __forceinline__ md<M> renorm(const double (&f)[M + 1]) {
  double g[M + 1];
  double s = f[M];
#pragma unroll
  for (int i = M - 1; i >= 0; --i) quick_two_sum(f[i], s, s, g[i + 1]);
  g[0] = s;
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = 0.0;
  double eps = g[0];
  int j = 0;
#pragma unroll
  for (int i = 1; i <= M - 1; ++i) {
    double rr, e;
    quick_two_sum(eps, g[i], rr, e);
    const bool emit = nonzero(e);
#pragma unroll
    for (int k = 0; k < i; ++k) r.v[k] = (emit && j == k) ? rr : r.v[k];
    j += emit ? 1 : 0;
    eps = emit ? e : rr;
  }
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = (j == k) ? eps : r.v[k];
  return r;
}

// baileyAdd_fast<M,M,M>
template <int M>
__device__ __forceinline__ md<M> gen_add(const md<M>& a, const md<M>& b) {
  double f[M + 1], e;
  f[M] = 0.0;
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    two_sum(a.v[i], b.v[i], f[i], e);
#pragma unroll
    for (int j = i + 1; j < M; ++j) two_sum(f[j], e, f[j], e);
    f[M] = __dadd_rn(f[M], e);
  }
  return renorm<M>(f);
}

template <int M>
__device__ __forceinline__ void carry(double (&f)[M + 1], int n, double x) {
#pragma unroll
  for (int j = n + 1; j < M; ++j) two_sum(f[j], x, f[j], x);
  f[M] = __dadd_rn(f[M], x);
}

// baileyMul_fast<M,LA,LB> with M output limbs (LA, LB in {1, M})
template <int M, int LA, int LB>
__device__ __forceinline__ md<M> gen_mul_gen(const double (&a)[LA], const double (&b)[LB]) {
  double f[M + 1];
  f[M] = 0.0;
  {
    bool first = true;
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int j = M - i;
      if (j < 0 || j >= LB) continue;
      double p = __dmul_rn(a[i], b[j]);
      if (first) {
        f[M] = p;
        first = false;
      } else {
        f[M] = __dadd_rn(f[M], p);
      }
    }
  }
#pragma unroll
  for (int n = M - 1; n >= 0; --n) {
    bool have = false;
#pragma unroll
    for (int i = 0; i <= n; ++i) {
      const int j = n - i;
      if (i >= LA || j >= LB) continue;
      double p, pe, e;
      two_prod(a[i], b[j], p, pe);
      if (!have) {
        f[n] = p;
        have = true;
        carry<M>(f, n, pe);
      } else {
        two_sum(f[n], p, f[n], e);
        carry<M>(f, n, pe);
        carry<M>(f, n, e);
      }
    }
    if (!have) f[n] = 0.0;
  }
  return renorm<M>(f);
}

template <int M>
__device__ __forceinline__ md<M> gen_mul(const md<M>& a, const md<M>& b) {
  return gen_mul_gen<M, M, M>(a.v, b.v);
}

template <int M>
__device__ __forceinline__ md<M> gen_mul_d(const md<M>& a, double b) {
  const double bb[1] = {b};
  return gen_mul_gen<M, M, 1>(a.v, bb);
}

// long division: M+1 quotient digits (not inlined: off the hot loops, keeps code size down)
template <int M>
__device__ __noinline__ md<M> gen_div(const md<M>& a, const md<M>& b) {
  double q[M + 1];
  md<M> r = a;
  q[0] = __ddiv_rn(a.v[0], b.v[0]);
#pragma unroll
  for (int i = 1; i <= M; ++i) {
    md<M> t = gen_mul_d<M>(b, q[i - 1]);
    r = gen_add<M>(r, neg(t));
    q[i] = __ddiv_rn(r.v[0], b.v[0]);
  }
  return renorm<M>(q);
}

// QDlib-style Newton on 1/sqrt, ceil(log2 M)+1 iterations, result a*y
template <int M>
__device__ __noinline__ md<M> gen_sqrt(const md<M>& a) {
  if (a.v[0] == 0.0) return md_zero<M>();
  constexpr int iters = (M == 4) ? 3 : 4;
  md<M> y = md_from<M>(__ddiv_rn(1.0, __dsqrt_rn(a.v[0])));
  const md<M> h = scale_pow2(a, 0.5);
  const md<M> half = md_from<M>(0.5);
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    md<M> t = gen_mul<M>(y, y);
    t = gen_mul<M>(h, t);
    t = gen_add<M>(half, neg(t));
    t = gen_mul<M>(t, y);
    y = gen_add<M>(y, t);
  }
  return gen_mul<M>(a, y);
}

// ----------------------------------------------------------------------------
// precision dispatch
// ----------------------------------------------------------------------------
// M = 1 is plain IEEE double ("1d": the paper's double precision reference rows):
// one correctly rounded operation each, no error-free transformation.
template <int M>
__device__ __forceinline__ md<M> add(const md<M>& a, const md<M>& b) {
  if constexpr (M == 1) return md<1>{{__dadd_rn(a.v[0], b.v[0])}};
  else if constexpr (M == 2) return dd_add(a, b);
  else return gen_add<M>(a, b);
}
template <int M>
__device__ __forceinline__ md<M> sub(const md<M>& a, const md<M>& b) {
  return add<M>(a, neg(b));
}
template <int M>
__device__ __forceinline__ md<M> mul(const md<M>& a, const md<M>& b) {
  if constexpr (M == 1) return md<1>{{__dmul_rn(a.v[0], b.v[0])}};
  else if constexpr (M == 2) return dd_mul(a, b);
  else return gen_mul<M>(a, b);
}
template <int M>
__device__ __forceinline__ md<M> mul_d(const md<M>& a, double b) {
  if constexpr (M == 1) return md<1>{{__dmul_rn(a.v[0], b)}};
  else if constexpr (M == 2) return dd_mul_d(a, b);
  else return gen_mul_d<M>(a, b);
}
template <int M>
__device__ __forceinline__ md<M> div(const md<M>& a, const md<M>& b) {
  if constexpr (M == 1) return md<1>{{__ddiv_rn(a.v[0], b.v[0])}};
  else if constexpr (M == 2) return dd_div(a, b);
  else return gen_div<M>(a, b);
}
template <int M>
__device__ __forceinline__ md<M> sqrt(const md<M>& a) {
  if constexpr (M == 1) return md<1>{{__dsqrt_rn(a.v[0])}};
  else if constexpr (M == 2) return dd_sqrt(a);
  else return gen_sqrt<M>(a);
}
// acc + a*b  (md mul, then md add: one "pair")
template <int M>
__device__ __forceinline__ md<M> fma(const md<M>& acc, const md<M>& a, const md<M>& b) {
  return add<M>(acc, mul<M>(a, b));
}
// acc - a*b
template <int M>
__device__ __forceinline__ md<M> fms(const md<M>& acc, const md<M>& a, const md<M>& b) {
  return add<M>(acc, neg(mul<M>(a, b)));
}

// ----------------------------------------------------------------------------
// latency-lean square root and reciprocal for the panel's scalar chain.
// Newton's iteration doubles the number of correct bits, so the reciprocal
// square root y ~ 1/sqrt(a) and the reciprocal are refined in increasing
// precision (double -> dd -> qd, each step at the precision it produces), and
// the last doubling is Karp's: sqrt(a) = a y + (a - (a y)^2) y / 2, 1/d = y +
// y (1 - d y), with only the leading products at full precision.  About 4x
// (od) / 2x (qd) fewer FP64 operations than QDlib-style sqrt and long
// division; results agree with them to within a few units of 2^(-53 M)
// (tests/test_gpu_arith.py, op codes 5 and 6).
// ----------------------------------------------------------------------------
template <int P, int M>
__device__ __forceinline__ md<P> md_trunc(const md<M>& a) {
  md<P> r;
#pragma unroll
  for (int k = 0; k < P; ++k) r.v[k] = (k < M) ? a.v[k] : 0.0;
  return r;
}

template <int M>
__device__ __forceinline__ md<M> add(const md<M>& a, const md<M>& b);
template <int M>
__device__ __forceinline__ md<M> mul(const md<M>& a, const md<M>& b);

// y <- y + y (1/2 - (a/2) y^2) at precision P
template <int P>
__device__ __forceinline__ md<P> rsqrt_step(const md<P>& a, const md<P>& y) {
  md<P> t = mul<P>(y, y);
  t = mul<P>(scale_pow2<P>(a, 0.5), t);
  t = add<P>(md_from<P>(0.5), neg(t));
  return add<P>(y, mul<P>(t, y));
}
// y ~ 1/sqrt(a) with about 53 * H correct bits (H = 1, 2, 4)
template <int H, int M>
__device__ __forceinline__ md<H> rsqrt_to(const md<M>& a) {
  md<H> y = md_from<H>(__drcp_rn(__dsqrt_rn(a.v[0])));
  if constexpr (H >= 2) {
    md<2> y2 = rsqrt_step<2>(md_trunc<2, M>(a), md_trunc<2, H>(y));
    y = md_trunc<H, 2>(y2);
  }
  if constexpr (H >= 4) {
    md<4> y4 = rsqrt_step<4>(md_trunc<4, M>(a), md_trunc<4, H>(y));
    y = md_trunc<H, 4>(y4);
  }
  return y;
}
template <int M>
__device__ __noinline__ md<M> sqrt_fast(const md<M>& a) {
  if (a.v[0] == 0.0) return md_zero<M>();
  if constexpr (M == 1) {
    return md<1>{{__dsqrt_rn(a.v[0])}};
  } else if constexpr (M == 2) {
    // Karp: sqrt(a) = a x + x (a - (a x)^2) / 2 with x = rsqrt(a0) (hardware-seeded double);
    // a0 - p is exact (Sterbenz), so the residual needs three plain operations
    const double x = ::rsqrt(a.v[0]);
    const double ax = __dmul_rn(a.v[0], x);
    double p, e;
    two_prod(ax, ax, p, e);
    const double d = __dadd_rn(__dsub_rn(__dsub_rn(a.v[0], p), e), a.v[1]);
    md<2> c;
    two_sum(ax, __dmul_rn(d, __dmul_rn(x, 0.5)), c.v[0], c.v[1]);
    return c;
  } else {
  constexpr int H = M / 2;
  const md<H> yh = rsqrt_to<H, M>(a);
  const md<M> y = md_trunc<M, H>(yh);
  const md<M> x = mul<M>(a, y);                         // a y
  const md<M> r = add<M>(a, neg(mul<M>(x, x)));         // a - (a y)^2, tiny
  const md<H> c = mul<H>(md_trunc<H, M>(r), scale_pow2<H>(yh, 0.5));
  return add<M>(x, md_trunc<M, H>(c));
  }
}
template <int P>
__device__ __forceinline__ md<P> recip_step(const md<P>& d, const md<P>& y) {
  const md<P> e = add<P>(md_from<P>(1.0), neg(mul<P>(d, y)));
  return add<P>(y, mul<P>(y, e));
}
template <int M>
__device__ __noinline__ md<M> recip_fast(const md<M>& d) {
  if constexpr (M == 1) {
    return md<1>{{__drcp_rn(d.v[0])}};
  } else if constexpr (M == 2) {
    const double y0 = __drcp_rn(d.v[0]);
    const md<2> e = dd_add(md_from<2>(1.0), neg(dd_mul_d(d, y0)));  // 1 - d y0, tiny
    md<2> r;
    two_sum(y0, __dmul_rn(y0, e.v[0]), r.v[0], r.v[1]);
    return r;
  } else {
  constexpr int H = M / 2;
  md<H> yh = md_from<H>(__drcp_rn(d.v[0]));
  if constexpr (H >= 2) yh = md_trunc<H, 2>(recip_step<2>(md_trunc<2, M>(d), md_trunc<2, H>(yh)));
  if constexpr (H >= 4) yh = md_trunc<H, 4>(recip_step<4>(md_trunc<4, M>(d), md_trunc<4, H>(yh)));
  const md<M> y = md_trunc<M, H>(yh);
  const md<M> e = add<M>(md_from<M>(1.0), neg(mul<M>(d, y)));   // 1 - d y, tiny
  const md<H> c = mul<H>(yh, md_trunc<H, M>(e));
  return add<M>(y, md_trunc<M, H>(c));
  }
}

// inline double-double pieces for the panel's scalar chain (dd only; the
// generic sqrt_fast / recip_fast are out-of-line)
// sqrt(a) by Karp from a double seed y0 ~ 1/sqrt(a0)
__device__ __forceinline__ md<2> dd_sqrt_seeded(const md<2>& a, double y0) {
  const double ax = __dmul_rn(a.v[0], y0);
  double p, e;
  two_prod(ax, ax, p, e);
  const double d = __dadd_rn(__dsub_rn(__dsub_rn(a.v[0], p), e), a.v[1]);
  md<2> c;
  two_sum(ax, __dmul_rn(d, __dmul_rn(y0, 0.5)), c.v[0], c.v[1]);
  return c;
}
// 1/sqrt(a): one Newton step y0 + y0 (1 - a y0^2) / 2 with the residual in double double
__device__ __forceinline__ md<2> dd_rsqrt_seeded(const md<2>& a, double y0) {
  double p, e;
  two_prod(y0, y0, p, e);                                   // y0^2 exactly
  const md<2> q = dd_mul(a, md<2>{{p, e}});                 // a y0^2
  const double r = __dadd_rn(__dsub_rn(1.0, q.v[0]), -q.v[1]);  // 1 - a y0^2 (tiny; Sterbenz)
  md<2> c;
  two_sum(y0, __dmul_rn(__dmul_rn(y0, 0.5), r), c.v[0], c.v[1]);
  return c;
}
// 1/d: y0 = rcp(d0), y = y0 + y0 (1 - d y0)
__device__ __forceinline__ md<2> dd_recip_inl(const md<2>& d) {
  const double y0 = __drcp_rn(d.v[0]);
  const double r = __fma_rn(-d.v[1], y0, __fma_rn(-d.v[0], y0, 1.0));  // 1 - d y0 (first fma exact)
  md<2> c;
  two_sum(y0, __dmul_rn(y0, r), c.v[0], c.v[1]);
  return c;
}

// ----------------------------------------------------------------------------
// dot-product accumulator: sum_k a_k * b_k.  Generic precisions keep a
// renormalised md sum (one md mul + one md add per term, 267 / 1471 FP64 ops
// for qd / od).  Double double keeps an unnormalised pair: the leading
// products are summed with two_sum and every error term (the FMA product
// error, both cross products a0*b1 + a1*b0, the two_sum error) goes into a
// plain double tail -- 12 FP64 ops per term instead of 29 -- and the pair is
// normalised once by get().  Error: |tail rounding| <= k u^2 sum |a_k b_k|,
// far inside the 1e3 n u parity tolerance for k <= 10^5.
// ----------------------------------------------------------------------------
//
// Quad and octo double use the same idea with M "level bins" s[0..M-1]: the
// limb products a_i b_j of level n = i + j <= M-2 are exact two_prods whose
// high part is deposited into bin n and error into bin n+1; a deposit into
// bin L is exact (two_sum, the error carried to bin L+1, ...) down to bin M-2,
// and bin M-1 (levels M-1 and M, the same products baileyMul_fast keeps)
// takes plain FMAs.  Only bin M-1 ever rounds, at magnitude ~u^(M-1) of the
// terms, so the sum is accurate to a few units of u^M per term -- the same
// order as one renormalised md mul + md add per term -- at about 112 (qd) /
// 950 (od) FP64 operations per term instead of 267 / 1471.  renorm_bins()
// (a bottom-up two_sum sweep) keeps the lower bins small; callers run it every
// few terms (each k-tile), get() runs it and renormalises to an md number.
template <int M>
struct Acc {
  double s[M];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int k = 0; k < M; ++k) s[k] = 0.0;
  }
  // exact deposit of t into bin L (two_sum cascade to bin M-2, plain add into bin M-1)
  __device__ __forceinline__ void dep(int L, double t) {
#pragma unroll
    for (int j = 0; j < M - 1; ++j)
      if (j >= L) two_sum(s[j], t, s[j], t);
    s[M - 1] = __dadd_rn(s[M - 1], t);
  }
  __device__ __forceinline__ void add_prod(const md<M>& a, const md<M>& b) {
    double tail = s[M - 1];
#pragma unroll
    for (int i = 0; i < M; ++i) tail = __fma_rn(a.v[i], b.v[M - 1 - i], tail);  // level M-1
#pragma unroll
    for (int i = 1; i < M; ++i) tail = __fma_rn(a.v[i], b.v[M - i], tail);      // level M
    s[M - 1] = tail;
#pragma unroll
    for (int n = 0; n <= M - 2; ++n) {
#pragma unroll
      for (int i = 0; i <= n; ++i) {
        double p, e;
        two_prod(a.v[i], b.v[n - i], p, e);
        dep(n, p);
        dep(n + 1, e);
      }
    }
  }
  __device__ __forceinline__ void renorm_bins() {
#pragma unroll
    for (int j = M - 1; j >= 1; --j) two_sum(s[j - 1], s[j], s[j - 1], s[j]);
  }
  // exact merge of another accumulator (bin by bin)
  __device__ __forceinline__ void merge(const Acc& o) {
#pragma unroll
    for (int L = 0; L < M; ++L) dep(L, o.s[L]);
  }
  static constexpr int NV = M;
  __device__ __forceinline__ double& r(int i) { return s[i]; }
  __device__ __forceinline__ double r(int i) const { return s[i]; }
  __device__ __forceinline__ md<M> get() const {
    double f[M + 1];
#pragma unroll
    for (int k = 0; k < M; ++k) f[k] = s[k];
    f[M] = 0.0;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int j = M - 1; j >= 1; --j) two_sum(f[j - 1], f[j], f[j - 1], f[j]);
    return renorm<M>(f);
  }
};
template <>
struct Acc<2> {
  double hi, lo;
  __device__ __forceinline__ void init() { hi = lo = 0.0; }
  __device__ __forceinline__ void add_prod(const md<2>& a, const md<2>& b) {
    const double p = __dmul_rn(a.v[0], b.v[0]);
    double pe = __fma_rn(a.v[0], b.v[0], -p);
    pe = __fma_rn(a.v[0], b.v[1], pe);
    pe = __fma_rn(a.v[1], b.v[0], pe);
    double t;
    two_sum(hi, p, hi, t);
    lo = __dadd_rn(lo, __dadd_rn(t, pe));
  }
  __device__ __forceinline__ void renorm_bins() { two_sum(hi, lo, hi, lo); }
  __device__ __forceinline__ void merge(const Acc& o) {
    double t;
    two_sum(hi, o.hi, hi, t);
    lo = __dadd_rn(lo, __dadd_rn(o.lo, t));
  }
  static constexpr int NV = 2;
  __device__ __forceinline__ double& r(int i) { return i == 0 ? hi : lo; }
  __device__ __forceinline__ double r(int i) const { return i == 0 ? hi : lo; }
  __device__ __forceinline__ md<2> get() const {
    md<2> r;
    two_sum(hi, lo, r.v[0], r.v[1]);
    return r;
  }
};

template <int M>
__device__ __forceinline__ Acc<M> acc_shfl_xor(const Acc<M>& a, int m) {
  Acc<M> o;
#pragma unroll
  for (int k = 0; k < Acc<M>::NV; ++k) o.r(k) = __shfl_xor_sync(0xffffffffu, a.r(k), m);
  return o;
}
template <int M>
__device__ __forceinline__ Acc<M> acc_shfl_down(const Acc<M>& a, int d) {
  Acc<M> o;
#pragma unroll
  for (int k = 0; k < Acc<M>::NV; ++k) o.r(k) = __shfl_down_sync(0xffffffffu, a.r(k), d);
  return o;
}

// ----------------------------------------------------------------------------
// limb-planar access: limb k of element e at p[k*ps + e]
// ----------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ md<M> ld(const double* __restrict__ p, int64_t ps, int64_t e) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = p[k * ps + e];
  return r;
}
template <int M>
__device__ __forceinline__ md<M> ld_cg(const double* p, int64_t ps, int64_t e) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = __ldcg(p + k * ps + e);
  return r;
}
template <int M>
__device__ __forceinline__ void st(double* __restrict__ p, int64_t ps, int64_t e, const md<M>& x) {
#pragma unroll
  for (int k = 0; k < M; ++k) p[k * ps + e] = x.v[k];
}

template <int M>
__device__ __forceinline__ md<M> shfl(const md<M>& x, int src, unsigned mask = 0xffffffffu) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = __shfl_sync(mask, x.v[k], src);
  return r;
}
template <int M>
__device__ __forceinline__ md<M> shfl_down(const md<M>& x, int d, unsigned mask = 0xffffffffu) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = __shfl_down_sync(mask, x.v[k], d);
  return r;
}
template <int M>
__device__ __forceinline__ md<M> shfl_xor(const md<M>& x, int d, unsigned mask = 0xffffffffu) {
  md<M> r;
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = __shfl_xor_sync(mask, x.v[k], d);
  return r;
}

// warp sum in a fixed tree order (lane 0 holds the result; deterministic)
template <int M>
__device__ __forceinline__ md<M> warp_sum(md<M> x) {
#pragma unroll 1
  for (int d = 16; d >= 1; d >>= 1) x = add<M>(x, shfl_down<M>(x, d));
  return x;
}
// warp sum broadcast to all lanes (butterfly; every lane gets the same bits only
// if add is commutative bitwise -- it is not for CAMPARY add, so use warp_sum +
// shfl when all lanes need the identical value)
template <int M>
__device__ __forceinline__ md<M> warp_sum_all(md<M> x) {
  x = warp_sum<M>(x);
  return shfl<M>(x, 0);
}

}  // namespace mdls
