// kern_leaf.cuh -- A1 + A2 (and the sub-panel T of A3): Householder factorisation of a
// narrow sub-panel ("leaf", B columns) by one thread-block cluster.
//
// Algorithm 2 step 1: for each column, compute v and beta (GVL Alg.
// 5.1.1) and update the rest of the tile.  The tile (rows js..M-1,
// columns js..js+B-1) is partitioned by rows over the C CTAs of a cluster and
// held in shared memory for the whole leaf.  Per column ONE reduction suffices:
// with x the current column below the pivot and v = x / v1 (v(1) = 1),
//     v . a_c   = a_jc + (1/v1) * sum_{i>j} x_i a_ic          (beta R^T v)
//     Y_c^T v   = y_jc + (1/v1) * sum_{i>j} x_i y_ic   (c < l, previous vectors)
//     sigma     = sum_{i>j} x_i^2
// so the B sums g_c = sum_{i>j} x_i t_ic over the whole tile row (t = a or y)
// are reduced together: per-thread products, a warp reduce-scatter (halving),
// a cross-warp smem sum, then one cluster barrier and a fixed-order DSMEM sum
// over the C CTA partials.  Every CTA then computes the Householder scalars
// redundantly (identical bits), updates its rows, and CTA 0 builds the leaf's
// compact-WY factor T (T_ll = beta_l, T(:l, l) = -beta_l T(:l,:l) Y(:,:l)^T v_l,
// which is the paper's z = -beta (v + W Y^T v), with W = -Y T).
#pragma once
#include <cstdio>

#include "launch.cuh"
#include "md_warp.cuh"

namespace mdls {

template <int M>
struct LeafArgs {
  int64_t Mrows;  // rows of A
  int64_t js;     // first column of the leaf (= first pivot row)
  int64_t R;      // tile rows per CTA
  Mat A;          // matrix (R and v written in place)
  Mat Y;          // explicit Y store (same indexing as A)
  double* beta;   // beta of global column j at beta[l*bps + j]
  int64_t bps;
  Mat T;          // B x B leaf T (upper triangular, zeros below)
  int* info;      // min-slot: 1-based first zero / non-finite R_jj
  // register leaf only: apply the previous leaf (columns jsp..jsp+B-1, same width) to this
  // leaf's columns first, C -= Yp Tp^T (Yp^T C) on rows jsp..Mrows-1 (jsp < 0: none)
  Mat Yp;         // explicit Y (global column indexing, as Y)
  Mat Tp;         // previous leaf's T (B x B, upper)
  int64_t jsp;
};

// Reduce-scatter sum of V md values over the lanes of a warp that share
// (lane % TPR): halving exchanges on the lane bits above TPR.  On return the
// lane holds the full sums of values base..base+W_END-1 in v[0..W_END).
// `plain` collects the lane bits of the levels that ended as plain pairwise
// adds (lanes with those bits clear hold the canonical copy).
template <int M, int W, int MASK, int TPR>
struct HalveSum {
  static constexpr int W_END = (MASK < TPR) ? W : HalveSum<M, (W > 1 ? W / 2 : 1), MASK / 2, TPR>::W_END;
  __device__ __forceinline__ static void run(md<M>* v, int lane, int& base, int& plain) {
    if constexpr (MASK >= TPR && MASK > 0) {
      if constexpr (W > 1) {
        constexpr int half = W / 2;
        const bool up = (lane & MASK) != 0;
#pragma unroll
        for (int q = 0; q < half; ++q) {
          md<M> send, keep;
#pragma unroll
          for (int k = 0; k < M; ++k) {
            send.v[k] = up ? v[q].v[k] : v[q + half].v[k];
            keep.v[k] = up ? v[q + half].v[k] : v[q].v[k];
          }
          v[q] = add<M>(keep, shfl_xor<M>(send, MASK));
        }
        if (up) base += half;
        HalveSum<M, half, MASK / 2, TPR>::run(v, lane, base, plain);
      } else {
        v[0] = add<M>(v[0], shfl_xor<M>(v[0], MASK));
        plain |= MASK;
        HalveSum<M, 1, MASK / 2, TPR>::run(v, lane, base, plain);
      }
    }
  }
};
template <int M, int W, int TPR>
struct HalveSum<M, W, 0, TPR> {
  static constexpr int W_END = W;
  __device__ __forceinline__ static void run(md<M>*, int, int&, int&) {}
};

// Householder scalars (GVL Alg. 5.1.1): from sigma and x1, mu = sqrt(x1^2 +
// sigma), v1 = x1 - mu (x1 <= 0) or -sigma / (x1 + mu).  sigma = 0: P = I.
template <int M>
__device__ __noinline__ void house_v1(const md<M>& sigma, const md<M>& x1, md<M>& mu, md<M>& v1) {
  mu = sqrt<M>(add<M>(mul<M>(x1, x1), sigma));
  if (x1.v[0] <= 0.0) v1 = sub<M>(x1, mu);
  else v1 = div<M>(neg(sigma), add<M>(x1, mu));
}
// beta = 2 v1^2 / (sigma + v1^2)
template <int M>
__device__ __noinline__ md<M> house_beta(const md<M>& sigma, const md<M>& v1) {
  const md<M> v1sq = mul<M>(v1, v1);
  return div<M>(scale_pow2<M>(v1sq, 2.0), add<M>(sigma, v1sq));
}
template <int M>
__device__ __noinline__ md<M> md_recip(const md<M>& v1) {
  return recip_fast<M>(v1);
}

#ifdef MDLS_LEAF_PROF
__device__ long long g_leaf_prof[64 * 12];
#define LEAF_MARK(l, ph) \
  if (rank == 0 && tid == 0 && (l) < 64) g_leaf_prof[(l) * 12 + (ph)] = clock64();
#else
#define LEAF_MARK(l, ph)
#endif

template <int M, int B, int TPR, int NT>
__global__ void __launch_bounds__(NT) leaf_kernel(LeafArgs<M> a) {
  constexpr int V = B / TPR;      // tile columns per thread
  constexpr int NW = NT / 32;     // warps
  constexpr int NRG = NT / TPR;   // row groups
  constexpr int GS = (NT / B >= 32) ? 32 : (NT / B >= 16 ? 16 : (NT / B >= 8 ? 8 : (NT / B >= 4 ? 4 : (NT / B >= 2 ? 2 : 1))));
  static_assert(V >= 1 && B % TPR == 0, "leaf shape");
  static_assert(NT % B == 0 && B * NW <= NT && 32 % NW == 0 && NW >= 4, "leaf threads");

  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = tid % TPR, rg = tid / TPR;

  extern __shared__ double smem_leaf[];
  const int64_t R = a.R;
  double* tile = smem_leaf;                       // [M][B][R]
  double* vsm = smem_leaf + (int64_t)M * B * R;   // [M][R]
  __shared__ md<M> wpart[NW][B];
  __shared__ md<M> red[2][B];
  __shared__ md<M> piv[2][B];
  __shared__ md<M> G[B], pv[B], wv[B], betas[B];
  __shared__ md<M> SY[B][B];  // SY[p][l] = Y_p^T v_l (p < l)
  __shared__ md<M> Ts[B][B];  // leaf T, Ts[row][col]
  __shared__ md<M> sc_mu, sc_v1, sc_beta, sc_rv1;

  auto T_ = [&](int64_t i, int c, int l) -> double& { return tile[((int64_t)l * B + c) * R + i]; };

  const int64_t total = a.Mrows - a.js;
  const int64_t row0 = a.js + (int64_t)rank * R;
  int64_t Rp = total - (int64_t)rank * R;
  Rp = Rp < 0 ? 0 : (Rp > R ? R : Rp);

  // ---- load the tile ----
  for (int64_t e = tid; e < Rp * B; e += NT) {
    const int64_t i = e % Rp;
    const int c = (int)(e / Rp);
#pragma unroll
    for (int l = 0; l < M; ++l) T_(i, c, l) = a.A.p[l * a.A.ps + (a.js + c) * a.A.ld + row0 + i];
  }
  __syncthreads();

  for (int l = 0; l < B; ++l) {
    const int64_t j = a.js + l;
    const int buf = l & 1;
    const int64_t pr_abs = j - a.js;
    const int p_piv = (int)(pr_abs / R);
    const int64_t pr = pr_abs - (int64_t)p_piv * R;

    LEAF_MARK(l, 0);
    // (1) per-thread products x_i * t_ic over own rows below the pivot
    md<M> acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = md_zero<M>();
    for (int64_t i = rg; i < Rp; i += NRG) {
      if (row0 + i <= j) continue;
      md<M> x;
#pragma unroll
      for (int k = 0; k < M; ++k) x.v[k] = T_(i, l, k);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        md<M> t;
#pragma unroll
        for (int k = 0; k < M; ++k) t.v[k] = T_(i, h * V + q, k);
        acc[q] = fma<M>(acc[q], x, t);
      }
    }
    LEAF_MARK(l, 1);
    // (2) warp reduce-scatter, (3) cross-warp sum -> CTA partial
    int base = 0, plain = 0;
    HalveSum<M, V, 16, TPR>::run(acc, lane, base, plain);
    constexpr int WE = HalveSum<M, V, 16, TPR>::W_END;
    if ((lane & plain) == 0) {
#pragma unroll
      for (int q = 0; q < WE; ++q) wpart[warp][h * V + base + q] = acc[q];
    }
    __syncthreads();
    if (tid < ((B * NW + 31) / 32) * 32) {  // cross-warp sum, fixed shuffle tree (whole warps)
      const int c = tid / NW, w = tid % NW;
      md<M> s = (c < B) ? wpart[w][c] : md_zero<M>();
#pragma unroll
      for (int d = NW / 2; d >= 1; d >>= 1) {
        md<M> o = shfl_down<M>(s, d);
        if (w + d < NW) s = add<M>(s, o);
      }
      if (w == 0 && c < B) red[buf][c] = s;
    }
    if (rank == p_piv && tid >= NT - B) {
      const int c = tid - (NT - B);
      md<M> pvv;
#pragma unroll
      for (int k = 0; k < M; ++k) pvv.v[k] = T_(pr, c, k);
      piv[buf][c] = pvv;
    }
    LEAF_MARK(l, 2);
    cluster.sync();
    LEAF_MARK(l, 3);

    // (4) fixed-order sum of the C partials (DSMEM), pivot row from its owner
    if (tid < B * GS) {
      const int c = tid / GS, sub = tid % GS;
      constexpr int QPL = 16 / GS > 0 ? 16 / GS : 1;  // partials per lane (C <= 16)
      md<M> t[QPL];
#pragma unroll
      for (int u = 0; u < QPL; ++u) {  // issue all DSMEM loads first
        const int q = sub + u * GS;
        t[u] = (q < C) ? *cluster.map_shared_rank(&red[buf][c], q) : md_zero<M>();
      }
      md<M> s = t[0];
#pragma unroll
      for (int u = 1; u < QPL; ++u)
        if (sub + u * GS < C) s = add<M>(s, t[u]);
#pragma unroll
      for (int d = GS / 2; d >= 1; d >>= 1) {
        md<M> o = shfl_down<M>(s, d);
        if (sub + d < GS && sub + d < C) s = add<M>(s, o);  // lanes beyond C hold nothing
      }
      if (sub == 0) {
        G[c] = s;
        pv[c] = *cluster.map_shared_rank(&piv[buf][c], p_piv);
      }
    }
    __syncthreads();
    LEAF_MARK(l, 4);

    // (5) Householder scalars, every CTA identically (GVL Alg. 5.1.1, rewritten so
    // the three divisions are independent): mu = sqrt(x1^2 + sigma);
    //   x1 > 0:  s = x1 + mu, v1 = -sigma/s, 1/v1 = -s/sigma, beta = sigma/(mu s)
    //   x1 <= 0: v1 = x1 - mu,               beta = -v1/mu
    // (beta = 2 v1^2/(sigma + v1^2) in both cases, as sigma + v1^2 = -2 mu v1).
    // Meanwhile this CTA's warp 1 extends its rows of the leaf T by column l-1.
    const md<M> sigma = G[l], x1 = pv[l];
    const bool deg = sigma.v[0] == 0.0;
    const bool pos = x1.v[0] > 0.0;
    if (tid == 0) {
      sc_mu = deg ? x1 : sqrt_fast<M>(add<M>(mul<M>(x1, x1), sigma));
    } else if (tid == 32 % NT && !deg && pos) {
      sc_rv1 = md_recip<M>(sigma);  // 1/sigma for now
    } else if (warp == 2 && l > 0) {
      // T(r, ll) = -beta_ll sum_{p=r}^{ll-1} T(r, p) SY[p][ll] for the rows r = rank (mod C)
      const int ll = l - 1;
      for (int r = rank; r <= ll; r += C) {
        if (r == ll) {
          if (lane == 0) Ts[ll][ll] = betas[ll];
          continue;
        }
        md<M> s = (lane >= r && lane < ll) ? mul<M>(Ts[r][lane], SY[lane][ll]) : md_zero<M>();
        s = warp_sum<M>(s);
        if (lane == 0) Ts[r][ll] = neg(mul<M>(betas[ll], s));
      }
    }
    __syncthreads();
    LEAF_MARK(l, 5);
    if (!deg) {
      if (tid == 0) {
        sc_beta = md_recip<M>(sc_mu);  // 1/mu for now
      } else if (tid == 32 % NT) {
        if (pos) sc_v1 = md_recip<M>(add<M>(x1, sc_mu));  // 1/s for now
        else sc_rv1 = md_recip<M>(sub<M>(x1, sc_mu));
      }
    }
    __syncthreads();
    LEAF_MARK(l, 6);
    md<M> beta, rv1;
    if (deg) {
      beta = md_zero<M>();
      rv1 = md_from<M>(1.0);
    } else if (pos) {
      const md<M> s = add<M>(x1, sc_mu);
      rv1 = neg(mul<M>(s, sc_rv1));              // -s / sigma
      beta = mul<M>(mul<M>(sigma, sc_v1), sc_beta);  // sigma (1/s) (1/mu)
    } else {
      rv1 = sc_rv1;
      beta = neg(mul<M>(sub<M>(x1, sc_mu), sc_beta));  // -v1 / mu
    }
    // (6) w_c = beta (a_jc + rv1 g_c) for c > l; Y_c^T v = y_jc + rv1 g_c for c < l
    if (tid < B) {
      const int c = tid;
      if (c != l) {
        const md<M> t = deg ? pv[c] : add<M>(pv[c], mul<M>(rv1, G[c]));
        if (c > l) wv[c] = mul<M>(beta, t);
        else SY[c][l] = t;
      } else {
        betas[l] = beta;
      }
    }
    // v below the pivot (owner threads of column l)
    if (h == l / V) {
      for (int64_t i = rg; i < Rp; i += NRG) {
        if (row0 + i <= j) continue;
        md<M> x;
#pragma unroll
        for (int k = 0; k < M; ++k) x.v[k] = T_(i, l, k);
        const md<M> v = deg ? x : mul<M>(x, rv1);
#pragma unroll
        for (int k = 0; k < M; ++k) vsm[(int64_t)k * R + i] = v.v[k];
      }
    }
    __syncthreads();
    LEAF_MARK(l, 7);
    // (7) update own rows: t_ic -= v_i w_c (c > l); column l <- v (R_jj = mu on the pivot row)
    for (int64_t i = rg; i < Rp; i += NRG) {
      const int64_t gi = row0 + i;
      if (gi < j) continue;
      md<M> v;
      if (gi == j) {
        v = md_from<M>(1.0);
      } else {
#pragma unroll
        for (int k = 0; k < M; ++k) v.v[k] = vsm[(int64_t)k * R + i];
      }
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const int c = h * V + q;
        if (c > l) {
          md<M> t;
#pragma unroll
          for (int k = 0; k < M; ++k) t.v[k] = T_(i, c, k);
          t = (gi == j) ? add<M>(t, neg(wv[c])) : fms<M>(t, v, wv[c]);
#pragma unroll
          for (int k = 0; k < M; ++k) T_(i, c, k) = t.v[k];
        } else if (c == l) {
          const md<M> out = (gi == j) ? sc_mu : v;
#pragma unroll
          for (int k = 0; k < M; ++k) T_(i, c, k) = out.v[k];
        }
      }
    }
    if (tid == 0 && rank == 0) {
      const double m0 = sc_mu.v[0];
      if (!(m0 != 0.0) || !isfinite(m0)) atomicMin(a.info, (int)(j + 1));
    }
    __syncthreads();
    LEAF_MARK(l, 8);
  }

  // ---- last T column, write-back of R/v, explicit Y, beta, T ----
  if (warp == 2) {
    const int ll = B - 1;
    for (int r = rank; r <= ll; r += C) {
      if (r == ll) {
        if (lane == 0) Ts[ll][ll] = betas[ll];
        continue;
      }
      md<M> s = (lane >= r && lane < ll) ? mul<M>(Ts[r][lane], SY[lane][ll]) : md_zero<M>();
      s = warp_sum<M>(s);
      if (lane == 0) Ts[r][ll] = neg(mul<M>(betas[ll], s));
    }
  }
  for (int64_t e = tid; e < Rp * B; e += NT) {
    const int64_t i = e % Rp;
    const int c = (int)(e / Rp);
    const int64_t gi = row0 + i, jc = a.js + c;
#pragma unroll
    for (int l = 0; l < M; ++l) {
      const double t = T_(i, c, l);
      a.A.p[l * a.A.ps + jc * a.A.ld + gi] = t;
      a.Y.p[l * a.Y.ps + jc * a.Y.ld + gi] = (gi < jc) ? 0.0 : (gi == jc ? (l == 0 ? 1.0 : 0.0) : t);
    }
  }
  __syncthreads();
  if (rank == 0 && tid < B) st<M>(a.beta, a.bps, a.js + tid, betas[tid]);
  for (int e = tid; e < B * B; e += NT) {  // this CTA's rows of T (r = rank mod C), zeros below the diagonal
    const int r = e % B, c = e / B;
    if (r % C != rank) continue;
    st<M>(a.T.p, a.T.ps, r + (int64_t)c * a.T.ld, (r <= c) ? Ts[r][c] : md_zero<M>());
  }
  cluster.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

// ===========================================================================
// Register-resident leaf (rows per CTA <= NT/TPR): the same column step as
// leaf_kernel with the latency taken out of the chain.
//  * each thread keeps its row's V = B/TPR tile entries in registers; the TPR
//    threads of a row are adjacent lanes, so the current column x_i reaches
//    them by a shuffle and the update needs no block barrier;
//  * products and every reduction level use the unnormalised accumulators of
//    md.cuh (Acc: dd pair / qd-od level bins) -- exact merges, one
//    normalisation per column sum;
//  * the CTA partials are PUSHED into every CTA's shared memory (DSMEM stores,
//    double buffered) together with the pivot row before the cluster barrier,
//    so after it each CTA sums 16 local partials (no remote-load latency);
//  * Householder scalars split over three threads: mu = sqrt(x1^2 + sigma)
//    then 1/(x1 +- mu); 1/sigma; 1/mu = rsqrt(x1^2 + sigma) -- all
//    independent after the reduction except the first chain.
// Three __syncthreads and one cluster barrier per column.
// ===========================================================================
template <int M>
__device__ __forceinline__ md<M> rsqrt_md(const md<M>& a) {
  if constexpr (M == 8) {
    const md<8> y = md_trunc<8, 4>(rsqrt_to<4, 8>(a));
    return rsqrt_step<8>(a, y);
  } else {
    return rsqrt_to<M, M>(a);
  }
}

template <int M, int V, int MASK, int TPR>
struct HalveAcc {
  // reduce-scatter of V accumulators over the lane bits >= TPR (see HalveSum)
  __device__ __forceinline__ static void run(Acc<M>* v, int lane, int& base, int& plain) {
    if constexpr (MASK >= TPR && MASK > 0) {
      if constexpr (V > 1) {
        constexpr int half = V / 2;
        const bool up = (lane & MASK) != 0;
#pragma unroll
        for (int q = 0; q < half; ++q) {
          Acc<M> send, keep;
#pragma unroll
          for (int k = 0; k < Acc<M>::NV; ++k) {
            const double lo_k = v[q].r(k), hi_k = v[q + half].r(k);  // values, not addresses
            send.r(k) = up ? lo_k : hi_k;
            keep.r(k) = up ? hi_k : lo_k;
          }
          keep.merge(acc_shfl_xor<M>(send, MASK));
          v[q] = keep;
        }
        if (up) base += half;
        HalveAcc<M, half, MASK / 2, TPR>::run(v, lane, base, plain);
      } else {
        v[0].merge(acc_shfl_xor<M>(v[0], MASK));
        plain |= MASK;
        HalveAcc<M, 1, MASK / 2, TPR>::run(v, lane, base, plain);
      }
    }
  }
  static constexpr int V_END = (MASK < TPR) ? V : HalveAcc<M, (V > 1 ? V / 2 : 1), MASK / 2, TPR>::V_END;
};
template <int M, int V, int TPR>
struct HalveAcc<M, V, 0, TPR> {
  __device__ __forceinline__ static void run(Acc<M>*, int, int&, int&) {}
  static constexpr int V_END = V;
};

// --- async DSMEM helpers (st.async + mbarrier complete_tx) ---
__device__ __forceinline__ uint32_t cluster_addr(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double x, double y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               :: "r"(raddr), "d"(x), "d"(y), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double x, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
               :: "r"(raddr), "d"(x), "r"(rbar) : "memory");
}
// push an md-like value of NV doubles to the same smem slot of CTA `rank` (pairs as v2 stores; NV = 1,
// plain double, as one 8-byte store)
template <int NV>
__device__ __forceinline__ void push_vals(const double* v, const void* local_slot, int rank, uint32_t local_bar) {
  const uint32_t ra = cluster_addr(smem_addr(local_slot), rank);
  const uint32_t rb = cluster_addr(local_bar, rank);
  if constexpr (NV % 2 == 1) {
    static_assert(NV == 1, "odd md widths other than plain double");
    st_async_f64(ra, v[0], rb);
  } else {
#pragma unroll
    for (int k = 0; k < NV; k += 2) st_async_v2(ra + 8 * k, v[k], v[k + 1], rb);
  }
}

// t - v w through the level-bin accumulator (one normalisation)
template <int M>
__device__ __forceinline__ md<M> fms_acc(const md<M>& t, const md<M>& v, const md<M>& w) {
  Acc<M> a;
#pragma unroll
  for (int k = 0; k < Acc<M>::NV; ++k) a.r(k) = (k < M) ? t.v[k] : 0.0;
  a.add_prod(neg(v), w);
  return a.get();
}

// ---------------------------------------------------------------------------
// Prologue of the chained register leaf: apply the previous leaf's block
// reflector to this leaf's B columns (the "beta R^T v" + "update R" work of the
// panel, for the one block the chain waits on):
//     C <- C - Yp Tp^T (Yp^T C)      rows jsp..M-1 (P_WY = I + W Y^T, W = -Y T)
// Z = Yp^T C is reduced over the cluster by reduce-scatter (column c of Z to
// CTA c mod C, async pushes + mbarrier), the owner forms Z'(:,c) = Tp^T Z(:,c)
// and pushes it to every CTA, and each CTA updates its rows (CTA 0 also the B
// rows jsp..js-1 above the leaf, which become rows of R).  Shared memory
// (dynamic): Ys, Cs [RX][B] md, zred [CMAX][2][B] Acc, Zp [B][B] md.
// ---------------------------------------------------------------------------
template <int M, int B, int NT>
struct LeafPro {
  static constexpr int RX = ((NT / 4 + B) + 63) / 64 * 64;  // rows staged per CTA (tile rows + the B rows above), padded
  static constexpr int BP = B + 1;  // padded row stride (no bank conflicts across rows)
  static constexpr size_t ys = 0, cs = sizeof(md<M>) * RX * BP, zr = 2 * cs;
  static constexpr size_t zp = zr + sizeof(Acc<M>) * 16 * 2 * B;
  static constexpr size_t tp = zp + sizeof(md<M>) * B * B;
  static constexpr size_t zs = tp + sizeof(md<M>) * B * B;
  static constexpr size_t bytes = zs + sizeof(md<M>) * 2 * B;
};

template <int M, int B, int TPR, int NT>
__device__ __forceinline__ void leaf_prologue(const LeafArgs<M>& a, cg::cluster_group& cluster, int C, int rank,
                                              md<M> (&t)[B / TPR], int64_t Rp, bool valid, int64_t gi, int64_t row0,
                                              bool zinit, uint32_t zpar, int ncols = B) {
  using P = LeafPro<M, B, NT>;
  constexpr int BP = P::BP;
  constexpr int V = B / TPR;
  constexpr int BB = B * B;
  constexpr int RS = (NT / BB) >= 1 ? NT / BB : 1;  // lanes per Z entry (row split)
  static_assert(NT % BB == 0 || BB % NT == 0, "prologue threads");
  extern __shared__ __align__(16) unsigned char leaf_dyn[];
  md<M>* Ys = reinterpret_cast<md<M>*>(leaf_dyn + P::ys);
  md<M>* Cs = reinterpret_cast<md<M>*>(leaf_dyn + P::cs);
  Acc<M>* zred = reinterpret_cast<Acc<M>*>(leaf_dyn + P::zr);  // [src][cc][p]
  md<M>* Zp = reinterpret_cast<md<M>*>(leaf_dyn + P::zp);      // [p][c]
  md<M>* Tsm = reinterpret_cast<md<M>*>(leaf_dyn + P::tp);     // [pp][p] = Tp(p, pp)
  md<M>* Zsum = reinterpret_cast<md<M>*>(leaf_dyn + P::zs);    // [cc][p] summed Z(:, c)
  __shared__ __align__(8) unsigned long long zbar[2];
  const int tid = threadIdx.x, lane = tid & 31;
  // the B rows above the leaf (jsp..js-1) are spread over the CTAs: row jsp + rank + k C, k < ex
  const int ex = (rank < B) ? (B - 1 - rank) / C + 1 : 0;
  const int Rx = (int)Rp + ex;
  const int ncol = (B - 1 - rank) / C + 1 > 0 && rank < B ? (B - 1 - rank) / C + 1 : 0;  // owned Z columns
  if (tid == 0) {
    if (zinit) {
      mbar_init(smem_addr(&zbar[0]), 1);
      mbar_init(smem_addr(&zbar[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    mbar_arm(smem_addr(&zbar[0]), (uint32_t)(C * B * ncol * sizeof(Acc<M>)));
    mbar_arm(smem_addr(&zbar[1]), (uint32_t)(BB * sizeof(md<M>)));
  }
  // stage Yp and C rows: local row i < ex -> global jsp + i, else row0 + (i - ex); zero padding
  // to a multiple of 4 RS rows so the partial-product loop is branch free
  constexpr int RS0 = (NT / BB) >= 1 ? NT / BB : 1;
  const int Rxp = (Rx + 4 * RS0 - 1) / (4 * RS0) * (4 * RS0);
  for (int e = tid; e < Rxp * B; e += NT) {
    const int i = e % Rxp, p = e / Rxp;  // consecutive threads walk a column: coalesced global loads
    const int64_t g = (i < ex) ? a.jsp + rank + (int64_t)i * C : row0 + (i - ex);
    md<M> y = md_zero<M>(), c = md_zero<M>();
    if (i < Rx) {
#pragma unroll
      for (int k = 0; k < M; ++k) {
        y.v[k] = __ldcg(a.Yp.p + k * a.Yp.ps + (a.jsp + p) * a.Yp.ld + g);
        c.v[k] = (p < ncols) ? __ldcg(a.A.p + k * a.A.ps + (a.js + p) * a.A.ld + g) : 0.0;
      }
    }
    Ys[i * BP + p] = y;
    Cs[i * BP + p] = c;
  }
  for (int e = tid; e < BB; e += NT) {
    const int p = e % B, pp = e / B;
    md<M> tv;
#pragma unroll
    for (int k = 0; k < M; ++k) tv.v[k] = __ldcg(a.Tp.p + k * a.Tp.ps + pp * a.Tp.ld + p);
    Tsm[e] = tv;
  }
  LEAF_MARK(63, 0);
  cluster.sync();  // barriers armed everywhere, staging visible
  LEAF_MARK(63, 1);
  // Z partial (p, c) over the staged rows, RS lanes per entry, 4 interleaved accumulators (od: 2, its
  // operands loaded just in time -- four od accumulators and their operands do not fit the registers)
  {
    const int e = tid / RS, r0 = tid % RS;
    if (e < BB) {
      const int p = e % B, c = e / B;
      Acc<M> acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u].init();
      if constexpr (M == 8) {
#pragma unroll 1
        for (int i = 2 * r0; i < Rxp; i += 2 * RS) {
          acc[0].add_prod(Ys[i * BP + p], Cs[i * BP + c]);
          acc[1].add_prod(Ys[(i + 1) * BP + p], Cs[(i + 1) * BP + c]);
        }
      } else {
#pragma unroll 2
        for (int i = 4 * r0; i < Rxp; i += 4 * RS) {
          md<M> yv[4], cv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            yv[u] = Ys[(i + u) * BP + p];
            cv[u] = Cs[(i + u) * BP + c];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u].add_prod(yv[u], cv[u]);
        }
      }
      acc[0].merge(acc[1]);
      if constexpr (M != 8) {
        acc[2].merge(acc[3]);
        acc[0].merge(acc[2]);
      }
#pragma unroll
      for (int d = RS / 2; d >= 1; d >>= 1) {
        Acc<M> o = acc_shfl_down<M>(acc[0], d);
        if (r0 + d < RS) acc[0].merge(o);
      }
      if (r0 == 0) {
        const int q = c % C, cc = c / C;
        double sv[Acc<M>::NV];
#pragma unroll
        for (int k = 0; k < Acc<M>::NV; ++k) sv[k] = acc[0].r(k);
        push_vals<Acc<M>::NV>(sv, &zred[(rank * 2 + cc) * B + p], q, smem_addr(&zbar[0]));
      }
    }
  }
  LEAF_MARK(63, 2);
  // owner: Z(:, c) = sum of the C partials (fixed order), Z'(:, c) = Tp^T Z(:, c), push to all CTAs
  if (ncol > 0) {
    mbar_wait(smem_addr(&zbar[0]), zpar);
    __syncthreads();
    LEAF_MARK(63, 3);
    // Z(p, c) = fixed-order tree over the C source partials: thread (cc, p, q), 16 lanes per entry
    for (int e = tid; e < ncol * B * 16; e += NT) {
      const int q = e % 16, p = (e / 16) % B, cc = e / (16 * B);
      Acc<M> z;
      if (q < C) z = zred[(q * 2 + cc) * B + p];
      else z.init();
#pragma unroll
      for (int d = 8; d >= 1; d >>= 1) {
        Acc<M> o = acc_shfl_down<M>(z, d);
        if (q + d < 16) z.merge(o);
      }
      if (q == 0) Zsum[cc * B + p] = z.get();
    }
    __syncthreads();
    for (int cc = 0; cc < ncol; ++cc) {
      const int c = rank + cc * C;
      // Z'(pp, c) = sum_{p <= pp} Tp(p, pp) Z(p, c): thread (pp, p), B lanes per output
      if (tid < BB) {
        const int pp = tid / B, p = tid % B;
        Acc<M> pr;
        pr.init();
        if (p <= pp) pr.add_prod(Tsm[pp * B + p], Zsum[cc * B + p]);
#pragma unroll
        for (int d = B / 2; d >= 1; d >>= 1) {
          Acc<M> o = acc_shfl_down<M>(pr, d);
          if (p + d < B) pr.merge(o);
        }
        const md<M> zz = pr.get();
        // lanes p < C of each group push to CTA p (parallel pushes)
        md<M> zb;
#pragma unroll
        for (int k = 0; k < M; ++k) zb.v[k] = __shfl_sync(0xffffffffu, zz.v[k], (tid & 31) & ~(B - 1));
        for (int q = p; q < C; q += B) push_vals<M>(zb.v, &Zp[pp * B + c], q, smem_addr(&zbar[1]));
      }
    }
  }
  LEAF_MARK(63, 4);
  mbar_wait(smem_addr(&zbar[1]), zpar);
  __syncthreads();
  LEAF_MARK(63, 5);
  // update own rows (registers) and the B rows above the leaf (global; row jsp + rank + k C on CTA rank)
  if (valid) {
    const int h = tid % TPR;
    const int i = ex + (int)(gi - row0);
    Acc<M> u[V];
#pragma unroll
    for (int q = 0; q < V; ++q)
#pragma unroll
      for (int k = 0; k < Acc<M>::NV; ++k) u[q].r(k) = (k < M) ? t[q].v[k] : 0.0;
    if constexpr (M == 8) {
      // two chains per column (even / odd terms), merged at the end: half the dependent od products
      Acc<M> u2[V];
#pragma unroll
      for (int q = 0; q < V; ++q) u2[q].init();
#pragma unroll 1
      for (int p = 0; p < B; p += 2) {
        const md<M> y0 = neg(Ys[i * BP + p]), y1 = neg(Ys[i * BP + p + 1]);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          u[q].add_prod(y0, Zp[p * B + h * V + q]);
          u2[q].add_prod(y1, Zp[(p + 1) * B + h * V + q]);
        }
      }
#pragma unroll
      for (int q = 0; q < V; ++q) u[q].merge(u2[q]);
    } else {
#pragma unroll 4
      for (int p = 0; p < B; ++p) {
        const md<M> y = neg(Ys[i * BP + p]);
#pragma unroll
        for (int q = 0; q < V; ++q) u[q].add_prod(y, Zp[p * B + h * V + q]);
      }
    }
#pragma unroll
    for (int q = 0; q < V; ++q) t[q] = u[q].get();
  }
  if constexpr (M == 8) {
    // od: each row above the leaf by the last warp, lane = (column c, term quarter), one or two products per
    // lane merged over the quarters by shuffles -- instead of one thread per entry summing all B terms
    static_assert(B <= 32 && 32 % B == 0, "od leaf width");
    constexpr int NPART = 32 / B;
    if (tid >= NT - 32) {
      const int ln = tid & 31, c = ln % B, part = ln / B;
      for (int i = 0; i < ex; ++i) {  // warp-uniform
        Acc<M> u;
        u.init();
        if (part == 0) {
          const md<M> c0 = Cs[i * BP + c];
#pragma unroll
          for (int k = 0; k < M; ++k) u.r(k) = c0.v[k];
        }
        for (int p = part; p < B; p += NPART) u.add_prod(neg(Ys[i * BP + p]), Zp[p * B + c]);
#pragma unroll
        for (int d = B; d < 32; d <<= 1) u.merge(acc_shfl_xor<M>(u, d));
        const md<M> r = u.get();
        if (part == 0 && c < ncols)
#pragma unroll
          for (int k = 0; k < M; ++k) a.A.p[k * a.A.ps + (a.js + c) * a.A.ld + a.jsp + rank + (int64_t)i * C] = r.v[k];
      }
    }
  } else {
    for (int e = tid; e < ex * B; e += NT) {
      const int i = e / B, c = e % B;
      Acc<M> u;
      const md<M> c0 = Cs[i * BP + c];
#pragma unroll
      for (int k = 0; k < Acc<M>::NV; ++k) u.r(k) = (k < M) ? c0.v[k] : 0.0;
      for (int p = 0; p < B; ++p) u.add_prod(neg(Ys[i * BP + p]), Zp[p * B + c]);
      const md<M> r = u.get();
      if (c < ncols)
#pragma unroll
        for (int k = 0; k < M; ++k) a.A.p[k * a.A.ps + (a.js + c) * a.A.ld + a.jsp + rank + (int64_t)i * C] = r.v[k];
    }
  }
  LEAF_MARK(63, 6);
  (void)lane;
}

// Column ll of the leaf's compact-WY T for the rows r = rank (mod C):
//   T(ll, ll) = beta_ll,  T(r, ll) = -beta_ll sum_{p=r}^{ll-1} T(r, p) Y_p^T v_ll   (W = -Y T)
// one lane per row, the <= B-1 terms accumulated in a level-bin / pair accumulator (no warp tree).
template <int M, int BT>
__device__ __forceinline__ void leaf_t_column(md<M> (&Ts)[BT][BT], const md<M> (&SY)[BT][BT], const md<M> (&betas)[BT],
                                              int ll, int rank, int C, int lane) {
  const int r = rank + lane * C;
  if (r > ll) return;
  if (r == ll) {
    Ts[ll][ll] = betas[ll];
    return;
  }
  Acc<M> acc;
  acc.init();
  for (int p = r; p < ll; ++p) acc.add_prod(Ts[r][p], SY[p][ll]);
  Ts[r][ll] = neg(mul<M>(betas[ll], acc.get()));
}

// the same column with the <= BT-1 terms of a row spread over lanes (one product each, merged by a shuffle tree)
// and the scaling by -beta_ll taken by the warp: the octo double version (a row's sequential sum of up to seven
// od products is ~5k cycles per term)
template <int M, int BT>
__device__ __forceinline__ void leaf_t_column_warp(md<M> (&Ts)[BT][BT], const md<M> (&SY)[BT][BT],
                                                   const md<M> (&betas)[BT], int ll, int rank, int C, int lane) {
  static_assert(BT <= 32, "one lane per term");
  for (int r = rank; r < ll; r += C) {  // warp-uniform
    const int p = r + lane;
    Acc<M> acc;
    acc.init();
    if (p < ll) acc.add_prod(Ts[r][p], SY[p][ll]);
#pragma unroll
    for (int d = BT / 2; d >= 1; d >>= 1) {
      Acc<M> o = acc_shfl_down<M>(acc, d);
      if (lane + d < BT) acc.merge(o);
    }
    md<M> sum = acc.get();
#pragma unroll
    for (int k = 0; k < M; ++k) sum.v[k] = __shfl_sync(0xffffffffu, sum.v[k], 0);
    const md<M> t = neg(wmul_any<M>(betas[ll], sum));
    if (lane == 0) Ts[r][ll] = t;
  }
  if (lane == 0 && ll % C == rank) Ts[ll][ll] = betas[ll];
}

// One leaf (the body of leaf_reg_kernel; leaf_chain_kernel runs it for every leaf of the
// factorisation).  init_bars: initialise the column mbarriers (first leaf of the kernel);
// zinit / zpar: initialise the prologue mbarriers / their phase parity for this leaf.
template <int M, int B, int TPR, int NT>
__device__ __forceinline__ void leaf_body(const LeafArgs<M>& a, bool init_bars, bool zinit, uint32_t zpar) {
  constexpr int V = B / TPR;
  constexpr int NW = NT / 32;
  constexpr int CMAX = 16;
  constexpr int GS = 16;  // lanes per column in the final partial sum
  static_assert(V >= 1 && B % TPR == 0 && 32 % TPR == 0, "leaf shape");
  static_assert(B * NW <= NT && 32 % NW == 0 && NW >= 4 && B * GS <= NT && (B * NW) % 32 == 0, "leaf threads");

  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = tid % TPR, rg = tid / TPR;

  __shared__ __align__(16) Acc<M> red[2][CMAX][B];  // pushed CTA partials [buffer][source rank][column]
  __shared__ __align__(16) md<M> piv[2][B];         // pushed pivot row
  __shared__ __align__(16) md<M> pvl[B];            // pivot row staging in the owner CTA
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ Acc<M> wpart[NW][B];
  __shared__ md<M> G[B], W[B], betas[B], Uc[B], Qc[B];
  __shared__ md<M> SY[B][B];  // SY[p][l] = Y_p^T v_l (p < l)
  __shared__ md<M> Ts[B][B];
  __shared__ md<M> sc_mu, sc_rs, sc_rsig, sc_rmu, sc_rv1, sc_s, sc_bq;

  const int64_t total = a.Mrows - a.js;
  const int64_t row0 = a.js + (int64_t)rank * a.R;
  int64_t Rp = total - (int64_t)rank * a.R;
  Rp = Rp < 0 ? 0 : (Rp > a.R ? a.R : Rp);
  const bool valid = rg < Rp;
  const int64_t gi = row0 + rg;
  const uint32_t tx_bytes = (uint32_t)(C * B * sizeof(Acc<M>) + B * sizeof(md<M>));

  if (tid == 0) {
    if (init_bars) {
      mbar_init(smem_addr(&bar[0]), 1);
      mbar_init(smem_addr(&bar[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    mbar_arm(smem_addr(&bar[0]), tx_bytes);
    if (B > 1) mbar_arm(smem_addr(&bar[1]), tx_bytes);
  }
  md<M> t[V];
#pragma unroll
  for (int q = 0; q < V; ++q) {
    const int c = h * V + q;
#pragma unroll
    for (int k = 0; k < M; ++k) t[q].v[k] = valid ? __ldcg(a.A.p + k * a.A.ps + (a.js + c) * a.A.ld + gi) : 0.0;
  }
  // PDL (leaf_reg_launch): the leaf's own columns are final before the previous leaf ends (they are written only
  // by the near-window updates, a full event dependency), so they load above; the previous leaf's Y, T (prologue)
  // only after its grid has completed
  pdl_wait();
  if (a.jsp >= 0) leaf_prologue<M, B, TPR, NT>(a, cluster, C, rank, t, Rp, valid, gi, row0, zinit, zpar);
  else cluster.sync();  // every CTA's barriers initialised and armed before the first push

  for (int l = 0; l < B; ++l) {
    const int64_t j = a.js + l;
    const int buf = l & 1;
    const int p_piv = (int)((j - a.js) / a.R);
    const int hl = l / V, ql = l % V;

    LEAF_MARK(l, 0);
    // (1) x_i from the row's owner lane of column l; products over the own row
    md<M> x = t[0];  // column l of the own row (static register selects, no local memory)
#pragma unroll
    for (int q = 1; q < V; ++q)
#pragma unroll
      for (int k = 0; k < M; ++k) x.v[k] = (q == ql) ? t[q].v[k] : x.v[k];
#pragma unroll
    for (int k = 0; k < M; ++k) x.v[k] = __shfl_sync(0xffffffffu, x.v[k], (lane & ~(TPR - 1)) + hl);
    const bool below = valid && gi > j;
    Acc<M> acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) {
      acc[q].init();
      if (below) acc[q].add_prod(x, t[q]);
    }
    if (valid && gi == j) {
#pragma unroll
      for (int q = 0; q < V; ++q) pvl[h * V + q] = t[q];
    }
    LEAF_MARK(l, 1);
    // (2) warp reduce-scatter, cross-warp sum, async push to every CTA
    int base = 0, plain = 0;
    HalveAcc<M, V, 16, TPR>::run(acc, lane, base, plain);
    constexpr int VE = HalveAcc<M, V, 16, TPR>::V_END;
    if ((lane & plain) == 0) {
#pragma unroll
      for (int q = 0; q < VE; ++q) wpart[warp][h * V + base + q] = acc[q];
    }
    __syncthreads();
    const uint32_t lbar = smem_addr(&bar[buf]);
    if (tid < B * NW) {
      const int c = tid / NW, w = tid % NW;
      Acc<M> s = wpart[w][c];
#pragma unroll
      for (int d = NW / 2; d >= 1; d >>= 1) {
        Acc<M> o = acc_shfl_down<M>(s, d);
        if (w + d < NW) s.merge(o);
      }
      double sv[Acc<M>::NV];
#pragma unroll
      for (int k = 0; k < Acc<M>::NV; ++k) sv[k] = __shfl_sync(0xffffffffu, s.r(k), (lane & ~(NW - 1)));
      for (int q = w; q < C; q += NW) push_vals<Acc<M>::NV>(sv, &red[buf][rank][c], q, lbar);
    } else if (rank == p_piv) {
      for (int e = tid - B * NW; e < B * C; e += NT - B * NW) {
        const int c = e % B, q = e / B;
        push_vals<M>(pvl[c].v, &piv[buf][c], q, lbar);
      }
    }
    LEAF_MARK(l, 2);
    // (3) wait for the C partials and the pivot row; fixed-order sum, GS lanes per column
    if (tid < B * GS) {
      mbar_wait(lbar, (uint32_t)((l >> 1) & 1));
      LEAF_MARK(l, 3);
      const int c = tid / GS, q = tid % GS;
      Acc<M> s;
      if (q < C) s = red[buf][q][c];
      else s.init();
#pragma unroll
      for (int d = GS / 2; d >= 1; d >>= 1) {
        Acc<M> o = acc_shfl_down<M>(s, d);
        if (q + d < GS) s.merge(o);
      }
      if (q == 0) G[c] = s.get();
      if (tid == 0 && l + 2 < B) mbar_arm(lbar, tx_bytes);
    }
    __syncthreads();
    LEAF_MARK(l, 4);

    // (4) Householder scalars (GVL Alg. 5.1.1 with independent reciprocals):
    //   x1 > 0:  s = x1 + mu, 1/v1 = -s/sigma, beta = sigma/(mu s)
    //   x1 <= 0: v1 = x1 - mu (= s), beta = -v1/mu
    // then u_c = a_jc + g_c/v1 for every column: Y_c^T v (c < l) and w_c = beta u_c (c > l).
    const md<M> sigma = G[l], x1 = piv[buf][l];
    const bool deg = sigma.v[0] == 0.0;
    const bool pos = x1.v[0] > 0.0;
    if constexpr (M == 1) {
      // plain double: the same chain as double double, one rounded operation per step
      if (warp == 0) {
        const double x = x1.v[0], sg = sigma.v[0];
        double mu = x, beta = 0.0, rv1 = 1.0;
        if (!deg) {
          mu = __dsqrt_rn(__dadd_rn(__dmul_rn(x, x), sg));
          const double sv = pos ? __dadd_rn(x, mu) : __dsub_rn(x, mu);
          const double rmu = __drcp_rn(mu);
          rv1 = pos ? -__ddiv_rn(sv, sg) : __drcp_rn(sv);                           // 1/v1
          beta = pos ? __dmul_rn(__ddiv_rn(sg, sv), rmu) : -__dmul_rn(sv, rmu);    // 2 v1^2 / (sigma + v1^2)
        }
        if (lane < B) {
          const int c = lane;
          const double pc = piv[buf][c].v[0];
          const double u = deg ? pc : __fma_rn(rv1, G[c].v[0], pc);
          if (c < l) SY[c][l] = md<1>{{u}};
          W[c] = md<1>{{(c > l && !deg) ? __dmul_rn(beta, u) : 0.0}};
        }
        if (lane == 0) {
          sc_mu = md<1>{{mu}};
          sc_rv1 = md<1>{{rv1}};
          betas[l] = md<1>{{beta}};
        }
      }
    } else if constexpr (M == 2) {
      // double double: warp 0 computes the three independent chains inline (ILP), no extra barrier
      if (warp == 0) {
        md<2> mu = x1, beta = md_zero<2>(), rv1 = md_from<2>(1.0);
        if (!deg) {
          const md<2> aa = dd_add(dd_mul(x1, x1), sigma);
          const double y0 = ::rsqrt(aa.v[0]);
          mu = dd_sqrt_seeded(aa, y0);
          const md<2> rmu = dd_rsqrt_seeded(aa, y0);
          const md<2> sv = pos ? dd_add(x1, mu) : dd_add(x1, neg(mu));
          const md<2> rs = dd_recip_inl(sv);
          const md<2> rsig = dd_recip_inl(sigma);
          rv1 = pos ? neg(dd_mul(sv, rsig)) : rs;
          beta = pos ? dd_mul(dd_mul(sigma, rs), rmu) : neg(dd_mul(sv, rmu));
        }
        if (lane < B) {
          const int c = lane;
          const md<2> pc = piv[buf][c];
          const md<2> u = deg ? pc : dd_add(pc, dd_mul(rv1, G[c]));
          const md<2> w = dd_mul(beta, u);
          if (c < l) SY[c][l] = u;
          W[c] = (c > l && !deg) ? w : md_zero<2>();  // zero w: the update below is branch free
        }
        if (lane == 0) {
          sc_mu = mu;
          sc_rv1 = rv1;
          betas[l] = beta;
        }
      }
    } else {
      // qd/od, phase A: every md product of the scalar chain is computed by a whole warp (od: warp-cooperative,
      // md_warp.cuh; qd: redundantly per lane):
      // warp 0: mu = sqrt(x1^2 + sigma), s = x1 +- mu; warp 1: 1/sigma (x1 > 0); warp 2: 1/mu = rsqrt(x1^2 + sigma)
      if (!deg) {
        if (warp == 0) {
          const md<M> mu = w_sqrt_fast<M>(add<M>(wmul_any<M>(x1, x1), sigma));
          const md<M> sv = pos ? add<M>(x1, mu) : sub<M>(x1, mu);
          if (lane == 0) {
            sc_mu = mu;
            sc_s = sv;
          }
        } else if (warp == 1) {
          if (pos) {
            const md<M> r = w_recip_fast<M>(sigma);
            if (lane == 0) sc_rsig = r;
          }
        } else if (warp == 2) {
          const md<M> r = w_rsqrt<M>(add<M>(wmul_any<M>(x1, x1), sigma));
          if (lane == 0) sc_rmu = r;
        }
      } else if (tid == 0) {
        sc_mu = x1;
      }
    }
    if (warp == 3 && l > 0) {
      if constexpr (M == 8) leaf_t_column_warp<M>(Ts, SY, betas, l - 1, rank, C, lane);
      else leaf_t_column<M>(Ts, SY, betas, l - 1, rank, C, lane);
    }  // this CTA's rows of T(:, l-1)
    __syncthreads();
    LEAF_MARK(l, 5);
    if constexpr (M > 2) {
      static_assert(NT >= 32 * B, "one warp per leaf column");
      // phase B: warp 0 forms rs = 1/s (the long reciprocal); warps 1..B-1 meanwhile, in two steps (named
      // barrier 1): x1 > 0: rv1 = 1/v1 = -s/sigma (warp 1), bq = sigma/mu (warp 2), then per column c != l
      // (warp 1 + slot): u_c = a_jc + g_c/v1 and q_c = bq u_c (c > l), so that after rs only w_c = rs q_c and
      // beta = rs bq remain; x1 <= 0: bq = -v1/mu = beta (warp 2)
      const int slot = warp - 1;                               // column slot of warps 1..B-1
      const int cw = (slot >= 0 && slot < B - 1) ? (slot < l ? slot : slot + 1) : -1;  // its column (!= l)
      if (!deg) {
        if (warp == 0) {
          const md<M> r = w_recip_fast<M>(sc_s);
          if (lane == 0) sc_rs = r;
        } else if (warp < B) {
          const md<M> sv = sc_s, rmu = sc_rmu;
          if (warp == 1 && pos) {
            const md<M> r = neg(wmul_any<M>(sv, sc_rsig));
            if (lane == 0) sc_rv1 = r;
          } else if (warp == 2) {
            const md<M> r = pos ? wmul_any<M>(sigma, rmu) : neg(wmul_any<M>(sv, rmu));
            if (lane == 0) sc_bq = r;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(32 * (B - 1)) : "memory");
          if (pos && cw >= 0) {
            const md<M> pc = piv[buf][cw];
            const md<M> u = add<M>(pc, wmul_any<M>(sc_rv1, G[cw]));
            const md<M> q = (cw > l) ? wmul_any<M>(sc_bq, u) : md_zero<M>();
            if (lane == 0) {
              Uc[cw] = u;
              Qc[cw] = q;
            }
          }
        }
      }
      __syncthreads();
      // phase C: beta and u_c / w_c, one warp per column (warp 0: beta for x1 > 0)
      if (deg) {
        if (tid < B) {
          const int c = tid;
          if (c < l) SY[c][l] = piv[buf][c];
          else if (c == l) betas[l] = md_zero<M>();
          W[c] = md_zero<M>();
          if (c == 0) sc_rv1 = md_from<M>(1.0);
        }
      } else if (pos) {
        if (warp == 0) {
          const md<M> bt = wmul_any<M>(sc_rs, sc_bq);
          if (lane == 0) betas[l] = bt;
        } else if (cw >= 0) {
          const md<M> w = (cw > l) ? wmul_any<M>(sc_rs, Qc[cw]) : md_zero<M>();
          if (lane == 0) {
            if (cw < l) SY[cw][l] = Uc[cw];
            W[cw] = w;
          }
        }
        if (tid == 1) W[l] = md_zero<M>();
      } else {
        const md<M> rv1 = sc_rs, bt = sc_bq;
        if (cw >= 0) {
          const md<M> u = add<M>(piv[buf][cw], wmul_any<M>(rv1, G[cw]));
          const md<M> w = (cw > l) ? wmul_any<M>(bt, u) : md_zero<M>();
          if (lane == 0) {
            if (cw < l) SY[cw][l] = u;
            W[cw] = w;
          }
        }
        if (tid == 0) {
          betas[l] = bt;
          sc_rv1 = rv1;
          W[l] = md_zero<M>();
        }
      }
      __syncthreads();
    }
    LEAF_MARK(l, 6);
    LEAF_MARK(l, 7);
    // (6) update the own row: t_c -= v_i w_c (c > l, v = 1 on the pivot row); column l <- v (mu on the pivot row)
    if (valid && gi >= j) {
      const bool piv_row = gi == j;
      const md<M> v = piv_row ? md_from<M>(1.0) : (deg ? x : mul<M>(x, sc_rv1));
      const md<M> mu = sc_mu;
      md<M> nt[V];
#pragma unroll
      for (int q = 0; q < V; ++q) nt[q] = fms_acc<M>(t[q], v, W[h * V + q]);  // w = 0 for c <= l: t unchanged
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const bool isl = (h * V + q) == l;
#pragma unroll
        for (int k = 0; k < M; ++k) t[q].v[k] = isl ? (piv_row ? mu.v[k] : v.v[k]) : nt[q].v[k];
      }
    }
    if (tid == 0 && rank == 0) {
      const double m0 = sc_mu.v[0];
      if (!(m0 != 0.0) || !isfinite(m0)) atomicMin(a.info, (int)(j + 1));
    }
    LEAF_MARK(l, 8);
  }

  // ---- last T column, write-back of R/v, explicit Y, beta, T ----
  pdl_trigger();  // only the write-back remains: the next leaf's cluster may launch now
  __syncthreads();
  if (warp == 3) {
    if constexpr (M == 8) leaf_t_column_warp<M>(Ts, SY, betas, B - 1, rank, C, lane);
    else leaf_t_column<M>(Ts, SY, betas, B - 1, rank, C, lane);
  }
  if (valid) {
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int64_t jc = a.js + h * V + q;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        a.A.p[k * a.A.ps + jc * a.A.ld + gi] = t[q].v[k];
        a.Y.p[k * a.Y.ps + jc * a.Y.ld + gi] = (gi < jc) ? 0.0 : (gi == jc ? (k == 0 ? 1.0 : 0.0) : t[q].v[k]);
      }
    }
  }
  __syncthreads();
  if (rank == 0 && tid < B) st<M>(a.beta, a.bps, a.js + tid, betas[tid]);
  for (int e = tid; e < B * B; e += NT) {
    const int r = e % B, c = e / B;
    if (r % C != rank) continue;
    st<M>(a.T.p, a.T.ps, r + (int64_t)c * a.T.ld, (r <= c) ? Ts[r][c] : md_zero<M>());
  }
  __threadfence();  // R, v, Y, beta, T visible device-wide before the leaf is published
  cluster.sync();   // no CTA exits while another may still push into it
}

template <int M, int B, int TPR, int NT>
__global__ void __launch_bounds__(NT) leaf_reg_kernel(LeafArgs<M> a) {
  leaf_body<M, B, TPR, NT>(a, true, true, 0u);
}

template <int M, int B, int TPR, int NT>
cudaError_t leaf_reg_launch(cudaStream_t st, const LeafArgs<M>& la, int C, bool pdl = false) {
  auto kern = leaf_reg_kernel<M, B, TPR, NT>;
  // Exclusive SMs: request enough shared memory that no other CTA (the concurrent trailing / Q
  // GEMMs of the other streams) can share the leaf's SMs and their FP64 pipes -- the leaf is a
  // latency chain and would otherwise queue behind throughput-bound GEMM warps.  MDLS_LEAF_EXCL=0 off.
  static size_t excl_d[kMaxDev];  // kernel attributes are per device context
  static bool attr_set[kMaxDev];
  const int dev = cur_dev();
  if (!attr_set[dev]) {
    const char* v = getenv("MDLS_LEAF_EXCL");
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    const size_t room = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
    excl_d[dev] = (v && v[0] == '0') ? 0 : room;  // the whole opt-in shared memory: one leaf CTA per SM, alone
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(LeafPro<M, B, NT>::bytes, excl_d[dev]));
    attr_set[dev] = true;
  }
  const size_t excl = excl_d[dev];
  const size_t dyn = std::max((la.jsp >= 0) ? LeafPro<M, B, NT>::bytes : (size_t)0, excl);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the launch with the previous leaf's tail
  attr[1].val.programmaticStreamSerializationAllowed = (pdl && pdl_enabled()) ? 1 : 0;  // chain only
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  trace_begin(st, F_PANEL);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, la);
  trace_end(st, F_PANEL);
  return e;
}

// ---------------------------------------------------------------------------
// launcher: cluster size C (16, non-portable; 8 fallback), leaf width B
// (power of two dividing nb, capped per precision and by shared memory)
// ---------------------------------------------------------------------------
// The shared-memory leaf is compiled in its own translation unit per precision
// (leafsm_<p>.cu, MDLS_LEAF_SMEM_TU) to keep the od build parallel.
template <int M, int B, int TPR>
cudaError_t leaf_launch_impl(cudaStream_t st, const LeafArgs<M>& la, int C);
#if defined(MDLS_LEAF_SMEM_TU)
template <int M, int B, int TPR>
cudaError_t leaf_launch_impl(cudaStream_t st, const LeafArgs<M>& la, int C) {
  constexpr int NT = (64 * TPR < 128) ? 128 : 64 * TPR;  // >= 4 warps: warp 2 is free for T
  auto kern = leaf_kernel<M, B, TPR, NT>;
  const size_t smem = sizeof(double) * (size_t)M * (B + 1) * la.R;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  trace_begin(st, F_PANEL);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, la);
  trace_end(st, F_PANEL);
  return e;
}
#endif
#define MDLS_INSTANTIATE_LEAF_SMEM_WIDE(MM)                                             \
  template cudaError_t leaf_launch_impl<MM, 32, 4>(cudaStream_t, const LeafArgs<MM>&, int); \
  template cudaError_t leaf_launch_impl<MM, 16, 4>(cudaStream_t, const LeafArgs<MM>&, int);
#define MDLS_INSTANTIATE_LEAF_SMEM(MM)                                                  \
  template cudaError_t leaf_launch_impl<MM, 8, 4>(cudaStream_t, const LeafArgs<MM>&, int);  \
  template cudaError_t leaf_launch_impl<MM, 4, 4>(cudaStream_t, const LeafArgs<MM>&, int);  \
  template cudaError_t leaf_launch_impl<MM, 2, 2>(cudaStream_t, const LeafArgs<MM>&, int);  \
  template cudaError_t leaf_launch_impl<MM, 1, 1>(cudaStream_t, const LeafArgs<MM>&, int);

inline size_t leaf_smem_bytes(int M, int B, int64_t R) { return sizeof(double) * (size_t)M * (B + 1) * R; }

// factor columns [js, js+B) of A (rows js..Mrows-1); returns B used via *bw
template <int M>
cudaError_t launch_leaf(cudaStream_t st, int64_t Mrows, int64_t js, int64_t bmax, Mat A, Mat Y, double* beta,
                        int64_t bps, Mat T, int* info, int* bw) {
  int csize = leaf_cluster_size();
  const int64_t rows = Mrows - js;
  const size_t cap = 200 * 1024;
  int B = 1;
  while (B * 2 <= bmax && B * 2 <= (M <= 2 ? 16 : 8)) B *= 2;  // B = 32 measured slower per column
  for (;;) {
    const int C = (int)std::max<int64_t>(1, std::min<int64_t>(csize, rows));
    const int64_t R = cdiv(rows, C);
    while (B > 1 && leaf_smem_bytes(M, B, R) > cap) B /= 2;
    if (leaf_smem_bytes(M, B, R) > cap) return cudaErrorInvalidValue;
    LeafArgs<M> la{Mrows, js, R, A, Y, beta, bps, T, info, Mat{nullptr, 0, 0}, Mat{nullptr, 0, 0}, -1};
    cudaError_t e;
    static const bool force_smem = [] {
      const char* v = getenv("MDLS_LEAF");
      return v && v[0] == 's';
    }();
    if (!force_smem && B >= 4 && R <= 64) {
      if constexpr (M <= 2) e = (B == 16) ? leaf_reg_launch<M, 16, 4, 256>(st, la, C)
                                          : (B == 8 ? leaf_reg_launch<M, 8, 4, 256>(st, la, C)
                                                    : leaf_reg_launch<M, 4, 4, 256>(st, la, C));
      else e = (B == 8) ? leaf_reg_launch<M, 8, 4, 256>(st, la, C) : leaf_reg_launch<M, 4, 4, 256>(st, la, C);
    } else if (!force_smem && M <= 4 && B >= 4 && R <= 128) {
      if constexpr (M <= 2) e = (B == 16) ? leaf_reg_launch<M, 16, 4, 512>(st, la, C)
                                          : (B == 8 ? leaf_reg_launch<M, 8, 4, 512>(st, la, C)
                                                    : leaf_reg_launch<M, 4, 4, 512>(st, la, C));
      else e = (B == 8) ? leaf_reg_launch<M, 8, 4, 512>(st, la, C) : leaf_reg_launch<M, 4, 4, 512>(st, la, C);
    } else {
    switch (B) {
      case 32:
        if constexpr (M <= 2) {
          e = leaf_launch_impl<M, 32, 4>(st, la, C);
          break;
        }
        [[fallthrough]];
      case 16:
        if constexpr (M <= 2) {
          e = leaf_launch_impl<M, 16, 4>(st, la, C);
          break;
        }
        [[fallthrough]];
      case 8: e = leaf_launch_impl<M, 8, 4>(st, la, C); break;
      case 4: e = leaf_launch_impl<M, 4, 4>(st, la, C); break;
      case 2: e = leaf_launch_impl<M, 2, 2>(st, la, C); break;
      default: e = leaf_launch_impl<M, 1, 1>(st, la, C); break;
    }
    }
    if (e == cudaSuccess || csize == 8) {
      *bw = B;
      return e;
    }
    cudaGetLastError();
    csize = 8;  // non-portable cluster size refused: fall back to 8
  }
}

// ---------------------------------------------------------------------------
// chained leaves (whole-factorisation critical path): the register leaf with
// the previous-leaf prologue.  chain_leaf_width() returns the leaf width the
// chain uses at column js (0: shape not supported by the register leaf; the
// caller then runs the GEMM-chained panel path).
// ---------------------------------------------------------------------------
template <int M>
cudaError_t launch_leaf_chain(cudaStream_t st, int64_t Mrows, int64_t js, int B, Mat A, Mat Y, double* beta,
                              int64_t bps, Mat T, int* info, Mat Tp, int64_t jsp) {
  const int64_t rows = Mrows - js;
  const int C = (int)std::max<int64_t>(1, std::min<int64_t>(leaf_cluster_size(), rows));
  const int64_t R = cdiv(rows, C);
  LeafArgs<M> la{Mrows, js, R, A, Y, beta, bps, T, info, Y, Tp, jsp};
  if constexpr (M <= 2) {
    if (R <= 64) return B == 16 ? leaf_reg_launch<M, 16, 4, 256>(st, la, C, true) : leaf_reg_launch<M, 8, 4, 256>(st, la, C, true);
    return B == 16 ? leaf_reg_launch<M, 16, 4, 512>(st, la, C, true) : leaf_reg_launch<M, 8, 4, 512>(st, la, C, true);
  } else if constexpr (M == 4) {
    if (R <= 64) return leaf_reg_launch<M, 8, 4, 256>(st, la, C, true);
    return leaf_reg_launch<M, 8, 4, 512>(st, la, C, true);
  } else {
    return leaf_reg_launch<M, 8, 4, 256>(st, la, C, true);
  }
}

#define MDLS_INSTANTIATE_LEAF(MM)                                                                               \
  template cudaError_t launch_leaf<MM>(cudaStream_t, int64_t, int64_t, int64_t, Mat, Mat, double*, int64_t, Mat, \
                                       int*, int*);                                                                \
  template cudaError_t launch_leaf_chain<MM>(cudaStream_t, int64_t, int64_t, int, Mat, Mat, double*, int64_t, Mat, \
                                             int*, Mat, int64_t);

}  // namespace mdls
