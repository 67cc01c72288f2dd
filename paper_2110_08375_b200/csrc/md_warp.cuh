// md_warp.cuh -- warp-cooperative quad/octo double multiplication for the
// panel's scalar chain (the Householder scalars, are a chain of a
// dozen dependent md operations per column; an octo double product by one
// thread is ~1200 dependent FP64 operations, the bottleneck of the od panel).
//
// wmul<M>(a, b) is called by all 32 lanes of a warp with the same a, b and
// returns the product in every lane.  The exact limb products of baileyMul_fast
// -- p_ij = fl(a_i b_j) and e_ij = a_i b_j -
// p_ij for levels i + j <= M-1, plain p_ij for level M -- are spread over the
// lanes (one to three terms each).  Instead of carrying every error term down
// a limb chain, each term is split exactly onto a fixed grid of NB "bins"
// (Rump-Ogita-Oishi ExtractScalar: q = fl(fl(s_k + r) - s_k), r = r - q, with
// s_k = 2^(E0 - 46 k)): every bin part is a multiple of 2^(E0 - 46 k - 53) of
// magnitude <= 2^(E0 - 46 k - 7), so the <= 128 parts of a bin sum exactly in
// plain double arithmetic, in any order -- a warp butterfly of plain adds.
// The NB exact bin sums are then renormalised (two_sum sweep + CAMPARY's
// top-down emission) into M limbs.  The operands are first scaled by powers of
// two so that a_0, b_0 are in [1, 2) (exact), which fixes E0 = 9.  Terms below
// the last bin's grid are dropped: relative error < 2^-450 (od) / 2^-220 (qd),
// i.e. at or below one unit of 2^(-53 M) -- the products baileyMul_fast itself
// drops (levels > M) are of the same order.
#pragma once
#include "md.cuh"

namespace mdls {

template <int M>
struct WMulCfg {
  static constexpr int NB = (M == 8) ? 10 : 5;                      // bins: grid 2^-458 (od) / 2^-228 (qd)
  static constexpr int NT = M * (M + 1) / 2 * 2 + (M - 1);         // p + e of levels 0..M-1, p of level M
  static constexpr int ROUNDS = (NT + 31) / 32;
};

__device__ __forceinline__ int exponent_of(double x) {  // floor(log2 |x|) for normal x
  return (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
}
__device__ __forceinline__ double pow2(int e) {  // 2^e, -1022 <= e <= 1023
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// the term of index t of the product of a and b: value and the first bin it may occupy
template <int M>
__device__ __forceinline__ double wmul_term(const md<M>& a, const md<M>& b, int t, int& kfirst) {
  constexpr int NP = M * (M + 1) / 2;
  int kind, i, n;
  if (t < NP) {
    kind = 0;
    n = 0;
    while ((n + 1) * (n + 2) / 2 <= t) ++n;
    i = t - n * (n + 1) / 2;
  } else if (t < 2 * NP) {
    kind = 1;
    const int u = t - NP;
    n = 0;
    while ((n + 1) * (n + 2) / 2 <= u) ++n;
    i = u - n * (n + 1) / 2;
  } else {
    kind = 0;
    n = M;
    i = t - 2 * NP + 1;  // 1..M-1
  }
  const int j = n - i;
  double ai = 0.0, bj = 0.0;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    ai = (k == i) ? a.v[k] : ai;
    bj = (k == j) ? b.v[k] : bj;
  }
  const double p = __dmul_rn(ai, bj);
  const int level = n + kind;
  // |a_i| <= 2^(-52 i) |a_0| (ulp-nonoverlapping limbs): |term| < 2^(2 - 52 level) <= 2^(2 - 46 k) for
  // k = floor(52 level / 46)
  kfirst = (52 * level) / 46 - 1;  // one bin of margin (terms up to 2^46 above the bound stay exact)
  kfirst = kfirst < 0 ? 0 : kfirst;
  return kind ? __fma_rn(ai, bj, -p) : p;
}

template <int M>
__device__ __noinline__ md<M> wmul(const md<M>& a, const md<M>& b) {
  using C = WMulCfg<M>;
  constexpr int NB = C::NB;
  const int lane = threadIdx.x & 31;
  const double a0 = a.v[0], b0 = b.v[0];
  if (a0 == 0.0 || b0 == 0.0) return md_zero<M>();
  const int ea = exponent_of(a0), eb = exponent_of(b0);
  if (ea < -1000 || ea > 1000 || eb < -1000 || eb > 1000 || ea + eb < -500 || ea + eb > 1000)
    return mul<M>(a, b);  // extreme exponents: the sequential product (warp-uniform branch)
  const double sa = pow2(-ea), sb = pow2(-eb);
  md<M> as, bs;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    as.v[k] = __dmul_rn(a.v[k], sa);
    bs.v[k] = __dmul_rn(b.v[k], sb);
  }
  double bin[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) bin[k] = 0.0;
#pragma unroll
  for (int r = 0; r < C::ROUNDS; ++r) {
    const int t = lane + 32 * r;
    if (t < C::NT) {
      int kf;
      double rem = wmul_term<M>(as, bs, t, kf);
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const double s = pow2(9 - 46 * k);
        const double q = __dsub_rn(__dadd_rn(s, rem), s);  // rem on bin k's grid (exact)
        const bool on = k >= kf;
        bin[k] = __dadd_rn(bin[k], on ? q : 0.0);
        rem = on ? __dsub_rn(rem, q) : rem;
      }
    }
  }
  // exact bin sums over the warp (plain adds: all parts on the bin grid, |sum| <= 2^(9 - 46 k))
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1)
#pragma unroll
    for (int k = 0; k < NB; ++k) bin[k] = __dadd_rn(bin[k], __shfl_xor_sync(0xffffffffu, bin[k], d));
  // renormalise: bottom-up two_sum sweep, then the top-down emission of renorm<M>
  double g[NB];
  double s = bin[NB - 1];
#pragma unroll
  for (int k = NB - 2; k >= 0; --k) two_sum(bin[k], s, s, g[k + 1]);
  g[0] = s;
  md<M> r = md_zero<M>();
  double eps = g[0];
  int j = 0;
#pragma unroll
  for (int i = 1; i < NB; ++i) {
    double rr, e;
    quick_two_sum(eps, g[i], rr, e);
    const bool emit = nonzero(e) && j < M - 1;
#pragma unroll
    for (int k = 0; k < M; ++k) r.v[k] = (emit && j == k) ? rr : r.v[k];
    j += emit ? 1 : 0;
    eps = emit ? e : rr;
  }
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = (j == k) ? eps : r.v[k];
  const double sc = pow2(ea + eb);
#pragma unroll
  for (int k = 0; k < M; ++k) r.v[k] = __dmul_rn(r.v[k], sc);
  return r;
}

// dispatch: only the octo double product is faster across the warp (B200, tools/wmul_lat.cu: one dependent
// od product 4.3k cycles by the warp vs 6.7k by one thread; qd 1.9k vs 0.9k), so dd and qd stay per thread
// (every lane computes the same product)
template <int M>
__device__ __forceinline__ md<M> wmul_any(const md<M>& a, const md<M>& b) {
  if constexpr (M == 8) return wmul<M>(a, b);
  else return mul<M>(a, b);
}

// the latency-lean square root / reciprocal / reciprocal square root of md.cuh with every product of
// two or more limbs taken by the warp (same Newton/Karp sequence, same precisions per step)
template <int P>
__device__ __forceinline__ md<P> w_rsqrt_step(const md<P>& a, const md<P>& y) {
  md<P> t = wmul_any<P>(y, y);
  t = wmul_any<P>(scale_pow2<P>(a, 0.5), t);
  t = add<P>(md_from<P>(0.5), neg(t));
  return add<P>(y, wmul_any<P>(t, y));
}
template <int H, int M>
__device__ __forceinline__ md<H> w_rsqrt_to(const md<M>& a) {
  md<H> y = md_from<H>(__drcp_rn(__dsqrt_rn(a.v[0])));
  if constexpr (H >= 2) {
    md<2> y2 = rsqrt_step<2>(md_trunc<2, M>(a), md_trunc<2, H>(y));
    y = md_trunc<H, 2>(y2);
  }
  if constexpr (H >= 4) {
    md<4> y4 = w_rsqrt_step<4>(md_trunc<4, M>(a), md_trunc<4, H>(y));
    y = md_trunc<H, 4>(y4);
  }
  return y;
}
template <int M>
__device__ __forceinline__ md<M> w_sqrt_fast(const md<M>& a) {
  static_assert(M >= 4, "warp sqrt for qd / od");
  if (a.v[0] == 0.0) return md_zero<M>();
  constexpr int H = M / 2;
  const md<H> yh = w_rsqrt_to<H, M>(a);
  const md<M> y = md_trunc<M, H>(yh);
  const md<M> x = wmul_any<M>(a, y);
  const md<M> r = add<M>(a, neg(wmul_any<M>(x, x)));
  const md<H> c = wmul_any<H>(md_trunc<H, M>(r), scale_pow2<H>(yh, 0.5));
  return add<M>(x, md_trunc<M, H>(c));
}
template <int P>
__device__ __forceinline__ md<P> w_recip_step(const md<P>& d, const md<P>& y) {
  const md<P> e = add<P>(md_from<P>(1.0), neg(wmul_any<P>(d, y)));
  return add<P>(y, wmul_any<P>(y, e));
}
template <int M>
__device__ __forceinline__ md<M> w_recip_fast(const md<M>& d) {
  static_assert(M >= 4, "warp reciprocal for qd / od");
  constexpr int H = M / 2;
  md<H> yh = md_from<H>(__drcp_rn(d.v[0]));
  if constexpr (H >= 2) yh = md_trunc<H, 2>(recip_step<2>(md_trunc<2, M>(d), md_trunc<2, H>(yh)));
  if constexpr (H >= 4) yh = md_trunc<H, 4>(w_recip_step<4>(md_trunc<4, M>(d), md_trunc<4, H>(yh)));
  const md<M> y = md_trunc<M, H>(yh);
  const md<M> e = add<M>(md_from<M>(1.0), neg(wmul_any<M>(d, y)));
  const md<H> c = wmul_any<H>(yh, md_trunc<H, M>(e));
  return add<M>(y, md_trunc<M, H>(c));
}
// 1/sqrt(a) to full precision (od: qd seed + one od Newton step)
template <int M>
__device__ __forceinline__ md<M> w_rsqrt(const md<M>& a) {
  if constexpr (M == 8) {
    const md<8> y = md_trunc<8, 4>(w_rsqrt_to<4, 8>(a));
    return w_rsqrt_step<8>(a, y);
  } else {
    return w_rsqrt_to<M, M>(a);
  }
}

}  // namespace mdls
