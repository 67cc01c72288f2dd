// kern_bs.cuh -- tile inversion and tiled back substitution kernels (A7-A9).
#pragma once
#include "types.cuh"

namespace mdls {

// ============================================================================
// A7: inverse of upper-triangular nb x nb tiles, one warp per inverse column
// ("the k-th thread solves U v = e_k"; here the k-th WARP, its lanes
// sharing the rows of the column-oriented back substitution).  Output is the
// transposed inverse: Vt(c, tile*nb + r) = (U_tile^-1)(r, c).
//
// With a scaled copy Us (nb x n workspace, the back-substitution path), the
// diagonal is absorbed first: U = D U' with U' unit upper triangular,
// Us(i, l) = u_il / u_ii (i < l) and Us(l, l) = 1/u_ll, so U v = e_k becomes
// U' v = e_k / u_kk and each step of the chain is x_l = s_l (no md product on
// the latency chain, only the pivot row's normalisation and the row updates
// s_i -= u'_il x_l, whose U' loads are issued one step ahead).  Without it
// (mdls_invert_tiles, no workspace) every step multiplies by 1/u_ll.
// ============================================================================
// Us(i, tile*nb + l) = u_il / u_ii for i < l, 1 / u_ll on the diagonal (one CTA per tile)
template <int M>
__global__ void __launch_bounds__(256) scale_tiles_kernel(int64_t nb, CMat U, Mat Us, int* info) {
  extern __shared__ double smem_inv[];  // rinv: M planes of nb
  const int64_t base = (int64_t)blockIdx.x * nb;
  for (int64_t r = threadIdx.x; r < nb; r += blockDim.x) {
    const md<M> d = ld<M>(U.p, U.ps, (base + r) + (base + r) * U.ld);
    if (!(d.v[0] != 0.0) || !isfinite(d.v[0])) atomicMin(info, (int)(base + r + 1));
    const md<M> q = div<M>(md_from<M>(1.0), d);
#pragma unroll
    for (int l = 0; l < M; ++l) smem_inv[l * nb + r] = q.v[l];
    st<M>(Us.p, Us.ps, r + (base + r) * Us.ld, q);
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int64_t i = e % nb, l = e / nb;  // consecutive threads walk a column: coalesced
    if (i >= l) continue;
    md<M> ri;
#pragma unroll
    for (int q = 0; q < M; ++q) ri.v[q] = smem_inv[q * nb + i];
    st<M>(Us.p, Us.ps, i + (base + l) * Us.ld, mul<M>(ld<M>(U.p, U.ps, (base + i) + (base + l) * U.ld), ri));
  }
}

template <int M, int NPL, bool SCALED>
__global__ void __launch_bounds__(256) invert_tiles_kernel(int64_t nb, CMat U, CMat Us, Mat Vt, int* info) {
  extern __shared__ double smem_inv[];  // rinv: M planes of nb (unscaled path)
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * nb;  // tile rows/cols offset
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;

  if constexpr (!SCALED) {
    for (int64_t r = tid; r < nb; r += blockDim.x) {
      const md<M> d = ld<M>(U.p, U.ps, (base + r) + (base + r) * U.ld);
      if (!(d.v[0] != 0.0) || !isfinite(d.v[0])) atomicMin(info, (int)(base + r + 1));
      const md<M> q = div<M>(md_from<M>(1.0), d);
#pragma unroll
      for (int l = 0; l < M; ++l) smem_inv[l * nb + r] = q.v[l];
    }
    __syncthreads();
  }
  // element (i, l) of the tile's (scaled) strictly upper part
  auto u_at = [&](int64_t i, int64_t l) -> md<M> {
    if constexpr (SCALED) return ld<M>(Us.p, Us.ps, i + (base + l) * Us.ld);
    else return ld<M>(U.p, U.ps, (base + i) + (base + l) * U.ld);
  };

  for (int64_t k = (int64_t)blockIdx.y * nwarp + warp; k < nb; k += (int64_t)gridDim.y * nwarp) {
    // row accumulators s_i = rhs_i - sum_l u_il x_l (md.cuh Acc: exact deposits, normalised only when
    // row i becomes the pivot row l); rhs = e_k (unscaled) or e_k / u_kk (scaled)
    Acc<M> s[NPL];
    md<M> rk = md_from<M>(1.0);
    if constexpr (SCALED) rk = u_at(k, k);
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      s[t].init();
      if (lane + 32 * t == k)
#pragma unroll
        for (int q = 0; q < M; ++q) s[t].r(q) = rk.v[q];
    }
    md<M> un[NPL];  // column l of the strict upper part, loaded one step ahead
#pragma unroll
    for (int t = 0; t < NPL; ++t) {
      const int64_t i = lane + 32 * t;
      un[t] = (i < k) ? u_at(i, k) : md_zero<M>();
    }
    for (int64_t l = k; l >= 0; --l) {
      const int ol = (int)(l & 31), tl = (int)(l >> 5);
      Acc<M> sa = s[0];
#pragma unroll
      for (int t = 1; t < NPL; ++t)
#pragma unroll
        for (int q = 0; q < Acc<M>::NV; ++q) sa.r(q) = (t == tl) ? s[t].r(q) : sa.r(q);
      md<M> x = sa.get();
      if constexpr (!SCALED) {
        md<M> rinv;
#pragma unroll
        for (int q = 0; q < M; ++q) rinv.v[q] = smem_inv[q * nb + l];
        x = mul<M>(x, rinv);
      }
      x = shfl<M>(x, ol);
      if (lane == 0) st<M>(Vt.p, Vt.ps, k + (base + l) * Vt.ld, x);
      const md<M> nx = neg(x);
      md<M> uc[NPL];
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        uc[t] = un[t];
        const int64_t i = lane + 32 * t;
        un[t] = (l >= 1 && i < l - 1) ? u_at(i, l - 1) : md_zero<M>();  // next step's column, in flight
      }
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        const int64_t i = lane + 32 * t;
        if (i < l) s[t].add_prod(uc[t], nx);
      }
    }
    // zeros below the diagonal of the inverse: Vt(k, base + r) for r > k
    for (int64_t r = k + 1 + lane; r < nb; r += 32) st<M>(Vt.p, Vt.ps, k + (base + r) * Vt.ld, md_zero<M>());
  }
}

// ============================================================================
// A8: x_i = U_i^-1 b_i, one warp per output row (lanes over the columns)
// ============================================================================
template <int M>
__global__ void __launch_bounds__(256) bs_mulinv_kernel(int64_t nb, int64_t tile, CMat Vt, const double* b,
                                                        int64_t psb, double* x, int64_t psx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nb) return;
  const int64_t base = tile * nb;
  Acc<M> acc;
  acc.init();
  for (int64_t c = r + lane; c < nb; c += 32) {  // upper triangular: c >= r
    md<M> t = ld<M>(Vt.p, Vt.ps, c + (base + r) * Vt.ld);
    md<M> bb = ld<M>(b, psb, base + c);
    acc.add_prod(t, bb);
  }
  // fixed-order tree of exact accumulator merges (no renormalised md add per level)
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) acc.merge(acc_shfl_down<M>(acc, d));
  if (lane == 0) st<M>(x, psx, base + r, acc.get());
}

// ============================================================================
// A9: b(rho) -= sum_c U(rho, tile*nb + c) x_tile(c) for rho in [row0, row1).
// CTA = 32*RPT rows x G column groups: each thread keeps RPT independent row
// accumulators over the columns c = g, g+G, ... (coalesced column reads of U),
// then a fixed-order smem reduction over the G groups.
// ============================================================================
template <int M, int G, int RPT>
__global__ void __launch_bounds__(32 * G) bs_update_kernel(int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U,
                                                           const double* x, int64_t psx, double* b, int64_t psb) {
  __shared__ Acc<M> part[G][32 * RPT];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t rbase = row0 + (int64_t)blockIdx.x * 32 * RPT;
  const int64_t base = tile * nb;
  Acc<M> acc[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) acc[t].init();
  for (int64_t c = g; c < nb; c += G) {
    const md<M> xx = ld<M>(x, psx, base + c);
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int64_t rho = rbase + lane + 32 * t;
      if (rho < row1) acc[t].add_prod(ld<M>(U.p, U.ps, rho + (base + c) * U.ld), xx);
    }
  }
#pragma unroll
  for (int t = 0; t < RPT; ++t) part[g][lane + 32 * t] = acc[t];
  __syncthreads();
  // fixed-order tree over the G column groups (exact accumulator merges)
#pragma unroll
  for (int stride = G / 2; stride >= 1; stride >>= 1) {
    if (g < stride) {
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        Acc<M> a = part[g][lane + 32 * t];
        a.merge(part[g + stride][lane + 32 * t]);
        part[g][lane + 32 * t] = a;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < 32 * RPT; e += 32 * G) {
    const int64_t rho = rbase + e;
    if (rho >= row1) continue;
    const md<M> t = part[0][e].get();
    md<M> bb = ld<M>(b, psb, rho);
    st<M>(b, psb, rho, add<M>(bb, neg(t)));
  }
}

// Us (nullable): nb x (ntiles nb) workspace for the row-scaled copy (the diagonal absorbed, see A7)
template <int M>
void launch_invert(cudaStream_t st, int64_t ntiles, int64_t nb, CMat U, Mat Vt, Mat Us, int* info) {
  const int threads = 256, nwarp = threads / 32;
  const int64_t ny = cdiv(nb, nwarp);
  dim3 grid((unsigned)ntiles, (unsigned)ny);
  const size_t smem = sizeof(double) * M * nb;
  if (Us.p) {
    MDLS_LAUNCH(F_INVERT, st, scale_tiles_kernel<M><<<(unsigned)ntiles, threads, smem, st>>>(nb, U, Us, info));
    const CMat C = cm(Us);
    if (nb <= 32) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 1, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info));
    else if (nb <= 64) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 2, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info));
    else if (nb <= 128) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 4, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info));
    else MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 8, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info));
    return;
  }
  const CMat C{nullptr, 0, 0};
  if (nb <= 32) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 1, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info));
  else if (nb <= 64) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 2, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info));
  else if (nb <= 128) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 4, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info));
  else MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 8, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info));
}

template <int M>
void launch_bs_mulinv(cudaStream_t st, int64_t nb, int64_t tile, CMat Vt, const double* b, int64_t psb, double* x,
                      int64_t psx) {
  MDLS_LAUNCH(F_BS, st, bs_mulinv_kernel<M><<<(unsigned)cdiv(nb, 8), 256, 0, st>>>(nb, tile, Vt, b, psb, x, psx));
}

// rows [row0, row1): CTA = 32 rows x GC column groups (1024 / 512 threads), so
// even the short late steps spread over many SMs; `critical` (one tile of rows on the
// back substitution's chain): twice the column groups, half the sequential products
template <int M>
void launch_bs_update(cudaStream_t st, int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U, const double* x,
                      int64_t psx, double* b, int64_t psb) {
  const int64_t rows = row1 - row0;
  if (rows <= 0) return;
  constexpr int GC = (M == 2) ? 32 : 16;  // column groups (registers / smem bound)
  MDLS_LAUNCH(F_BS, st, bs_update_kernel<M, GC, 1><<<(unsigned)cdiv(rows, 32), 32 * GC, 0, st>>>(nb, tile, row0, row1, U, x, psx, b, psb));
}

#define MDLS_INSTANTIATE_BS(MM)                                                                                \
  template void launch_invert<MM>(cudaStream_t, int64_t, int64_t, CMat, Mat, Mat, int*);                                     \
  template void launch_bs_mulinv<MM>(cudaStream_t, int64_t, int64_t, CMat, const double*, int64_t, double*,    \
                                     int64_t);                                                                 \
  template void launch_bs_update<MM>(cudaStream_t, int64_t, int64_t, int64_t, int64_t, CMat, const double*,  \
                                     int64_t, double*, int64_t);

}  // namespace mdls
