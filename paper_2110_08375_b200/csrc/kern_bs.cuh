// kern_bs.cuh -- tile inversion and tiled back substitution kernels (A7-A9).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

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
// Us(i, tile*nb + l) = u_il / u_ii for i < l, 1 / u_ll on the diagonal.  Grid (tile, column slice):
// every CTA forms the tile's nb reciprocal diagonal entries (cheap, nb md divisions spread over the
// threads) and scales its own slice of columns, so a chunk of tiles fills the SMs.
template <int M>
__global__ void __launch_bounds__(256) scale_tiles_kernel(int64_t nb, CMat U, Mat Us, int* info, int64_t info_off) {
  extern __shared__ double smem_inv[];  // rinv: M planes of nb
  const int64_t base = (int64_t)blockIdx.x * nb;
  const int64_t c0 = nb * blockIdx.y / gridDim.y, c1 = nb * (blockIdx.y + 1) / gridDim.y;
  for (int64_t r = threadIdx.x; r < nb; r += blockDim.x) {
    const md<M> d = ld<M>(U.p, U.ps, (base + r) + (base + r) * U.ld);
    if (blockIdx.y == 0 && (!(d.v[0] != 0.0) || !isfinite(d.v[0]))) atomicMin(info, (int)(info_off + base + r + 1));
    const md<M> q = div<M>(md_from<M>(1.0), d);
#pragma unroll
    for (int l = 0; l < M; ++l) smem_inv[l * nb + r] = q.v[l];
    if (r >= c0 && r < c1) st<M>(Us.p, Us.ps, r + (base + r) * Us.ld, q);
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < nb * (c1 - c0); e += blockDim.x) {
    const int64_t i = e % nb, l = c0 + e / nb;  // consecutive threads walk a column: coalesced
    if (i >= l) continue;
    md<M> ri;
#pragma unroll
    for (int q = 0; q < M; ++q) ri.v[q] = smem_inv[q * nb + i];
    st<M>(Us.p, Us.ps, i + (base + l) * Us.ld, mul<M>(ld<M>(U.p, U.ps, (base + i) + (base + l) * U.ld), ri));
  }
}

template <int M, int NPL, bool SCALED>
__global__ void __launch_bounds__(256) invert_tiles_kernel(int64_t nb, CMat U, CMat Us, Mat Vt, int* info,
                                                           int64_t info_off) {
  extern __shared__ double smem_inv[];  // rinv: M planes of nb (unscaled path)
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * nb;  // tile rows/cols offset
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;

  if constexpr (!SCALED) {
    for (int64_t r = tid; r < nb; r += blockDim.x) {
      const md<M> d = ld<M>(U.p, U.ps, (base + r) + (base + r) * U.ld);
      if (!(d.v[0] != 0.0) || !isfinite(d.v[0])) atomicMin(info, (int)(info_off + base + r + 1));
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
        if (32 * t >= l) break;  // warp-uniform: row blocks at or below the pivot hold no work
        uc[t] = un[t];
        const int64_t i = lane + 32 * t;
        un[t] = (l >= 1 && i < l - 1) ? u_at(i, l - 1) : md_zero<M>();  // next step's column, in flight
      }
#pragma unroll
      for (int t = 0; t < NPL; ++t) {
        if (32 * t >= l) break;
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
template <int M, int NPL>
__global__ void __launch_bounds__(256) bs_mulinv_kernel(int64_t nb, int64_t tile, CMat Vt, const double* b,
                                                        int64_t psb, double* x, int64_t psx, BsFlow fl, int first) {
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool live = r < nb;
  const int64_t base = tile * nb;
  // the lane's columns c = r + lane + 32 t (upper triangular: c >= r), every load issued before any product;
  // the inverse (complete: a full dependency) before waiting, b (the updates' output) after
  md<M> tv[NPL], bv[NPL];
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int64_t c = r + lane + 32 * t;
    tv[t] = (live && c < nb) ? ld<M>(Vt.p, Vt.ps, c + (base + r) * Vt.ld) : md_zero<M>();
  }
  if (fl.rows && !first) {
    // dataflow: b_tile final once every later step's update reached its nb rows
    if (threadIdx.x == 0) spin_geq(fl.rows + tile, (int)(nb * (fl.N - 1 - tile)));
    __syncthreads();
  } else {
    pdl_wait();
  }
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int64_t c = r + lane + 32 * t;
    md<M> v = md_zero<M>();
    if (live && c < nb)
#pragma unroll
      for (int k = 0; k < M; ++k) v.v[k] = __ldcg(b + k * psb + base + c);
    bv[t] = v;
  }
  Acc<M> acc, acc2;  // two independent chains (even / odd t), merged before the tree
  acc.init();
  acc2.init();
#pragma unroll
  for (int t = 0; t < NPL; t += 2) {
    acc.add_prod(tv[t], bv[t]);
    if (t + 1 < NPL) acc2.add_prod(tv[t + 1], bv[t + 1]);
  }
  acc.merge(acc2);
  // fixed-order tree of exact accumulator merges (no renormalised md add per level)
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) acc.merge(acc_shfl_down<M>(acc, d));
  if (lane == 0 && live) {
    st<M>(x, psx, base + r, acc.get());
    if (fl.rows) __threadfence();
  }
  if (fl.rows) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t r0 = (int64_t)blockIdx.x * (blockDim.x >> 5);
      const int64_t r1 = r0 + (blockDim.x >> 5), rows = (r1 < nb ? r1 : nb) - r0;
      red_release_gpu(fl.xrdy + tile, (int)rows);  // x_tile rows published
    }
  }
}

// ============================================================================
// A9: b(rho) -= sum_c U(rho, tile*nb + c) x_tile(c) for rho in [row0, row1).
// CTA = RB rows x (256 / RB) column groups: thread (r, g) owns row rb + r and, in
// every stage, the stage's columns g, g + 256/RB, ...  The CTA's RB x nb block of
// U streams through shared memory in stages of 2048 doubles (SC = 2048 / (M RB)
// columns x M limb planes x RB rows) by cp.async (LDGSTS), NS - 1 stages in
// flight, so the HBM latency overlaps the md arithmetic with no register staging;
// x_tile is staged once per CTA; two accumulator chains per thread (alternate
// columns).  Then a fixed-order smem tree over the column groups.
// RB = 32 for the wide steps; RB = 8 spreads a short step over 4x the SMs.
// Coalesced: consecutive threads copy consecutive rows of one column plane.
// ============================================================================
template <int M, int RB, int NS, int MINB, int NACC>
__global__ void __launch_bounds__(256, MINB) bs_update_kernel(int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U,
                                                           const double* x, int64_t psx, double* b, int64_t psb,
                                                           const __grid_constant__ CUtensorMap tmap, int use_tma,
                                                           BsFlow fl) {
  constexpr int NT = 256, GR = NT / RB, STAGE = 2048, SC = STAGE / (M * RB);
  static_assert(SC >= GR && SC % GR == 0, "stage shape");
  extern __shared__ __align__(128) double sm_bs[];
  double* xs = sm_bs;                                  // M planes of nb: x_tile
  double* ring = sm_bs + ((M * nb + 15) & ~15);        // NS stages of [limb][column][row] (128-byte aligned)
  __shared__ Acc<M> part[GR][RB];
  __shared__ __align__(8) unsigned long long full[NS];  // TMA path: stage slot filled
  const int tid = threadIdx.x, r = tid % RB, gq = tid / RB;
  const int64_t base = tile * nb;
  // dataflow mode: row blocks from the diagonal upward (the critical tile first); launch order otherwise
  const int64_t rb = fl.rows ? row1 - (int64_t)(blockIdx.x + 1) * RB : row0 + (int64_t)blockIdx.x * RB;
  const int nst = (int)((nb + SC - 1) / SC);
  // TMA path (use_tma: the host encoded a 3-D tensor map rows x columns x limb planes of U, box RB x SC x M):
  // one cp.async.bulk.tensor per stage, issued by one thread, lands exactly in the stage's [limb][column][row]
  // layout, zero-filled outside U, completing on the slot's mbarrier -- no per-element address arithmetic.
  // Otherwise 8-byte cp.async (LDGSTS) per element with zero fill.
  if (use_tma) {
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < NS; ++q) mbar_init(smem_addr(&full[q]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("prefetch.tensormap [%0];" :: "l"(&tmap) : "memory");
    }
    __syncthreads();
  }
  auto issue = [&](int st) {
    if (use_tma) {
      if (st < nst && tid == 0) {
        const int slot = st % NS;
        const uint32_t bar = smem_addr(&full[slot]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's earlier generic reads first
        mbar_arm(bar, (uint32_t)(STAGE * sizeof(double)));
        const int c0 = (int)rb, c1 = (int)(base + (int64_t)st * SC), c2 = 0;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            :: "r"(smem_addr(ring + slot * STAGE)), "l"(&tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
      }
      return;
    }
    if (st < nst) {
      double* dst = ring + (st % NS) * STAGE;
      for (int e = tid; e < STAGE; e += NT) {
        const int rr = e % RB, c = (e / RB) % SC, k = e / (RB * SC);
        const int64_t col = (int64_t)st * SC + c, row = rb + rr;
        const bool ok = col < nb && row < row1;
        cp_async8(dst + e, ok ? U.p + k * U.ps + (base + col) * U.ld + row : U.p, ok);
      }
    }
    cp_async_commit();  // one group per stage, empty past the end (uniform wait counts)
  };
  pdl_trigger();
#pragma unroll
  for (int st = 0; st < NS - 1; ++st) issue(st);  // U is read-only here: prefetched before the PDL wait
  if (fl.rows) {
    // dataflow: x_tile written (mulinv) and this row block's tile updated by every later step
    if (tid == 0) {
      spin_geq(fl.xrdy + tile, (int)nb);
      spin_geq(fl.rows + rb / nb, (int)(nb * (fl.N - 1 - tile)));
    }
    __syncthreads();
  } else {
    pdl_wait();  // x (mulinv) and b (the previous update) from here on
  }
  for (int64_t e = tid; e < nb; e += NT)
#pragma unroll
    for (int k = 0; k < M; ++k) xs[k * nb + e] = __ldcg(x + k * psx + base + e);
  constexpr int CPT = SC / GR;  // columns per thread per stage
  Acc<M> acc[NACC];              // NACC independent chains (round-robin over the thread's columns), merged at the end
#pragma unroll
  for (int a = 0; a < NACC; ++a) acc[a].init();
  for (int st = 0; st < nst; ++st) {
    if (use_tma) mbar_wait(smem_addr(&full[st % NS]), (uint32_t)((st / NS) & 1));  // stage st has landed
    else cp_async_wait<NS - 2>();  // this thread's copies of stage st have landed
    __syncthreads();               // everyone's; and stage st - 1 is consumed, its slot free
    issue(st + NS - 1);
    const double* sg = ring + (st % NS) * STAGE;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = gq + j * GR;
      const int64_t col = (int64_t)st * SC + c;
      if (col < nb) {
        md<M> u, xx;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          u.v[k] = sg[(k * SC + c) * RB + r];
          xx.v[k] = xs[k * nb + col];
        }
        // chain (st CPT + j) mod NACC: j is a compile-time constant, the stage parity a warp-uniform branch
        // (constant indices only, so the chains stay in registers)
        if constexpr (NACC == 1) {
          acc[0].add_prod(u, xx);
        } else if constexpr (CPT % NACC == 0) {
          acc[j % NACC].add_prod(u, xx);
        } else {
          const int sel = (int)((st * CPT) % NACC);
#pragma unroll
          for (int a = 0; a < NACC; ++a)
            if (sel == a) acc[(a + j) % NACC].add_prod(u, xx);
        }
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 1; a < NACC; ++a) acc[0].merge(acc[a]);
  part[gq][r] = acc[0];
  __syncthreads();
  // fixed-order tree over the column groups (exact accumulator merges)
#pragma unroll
  for (int stride = GR / 2; stride >= 1; stride >>= 1) {
    if (gq < stride) {
      Acc<M> a = part[gq][r];
      a.merge(part[gq + stride][r]);
      part[gq][r] = a;
    }
    __syncthreads();
  }
  if (gq == 0 && rb + r < row1) {
    const md<M> t = part[0][r].get();
    md<M> bb;
#pragma unroll
    for (int k = 0; k < M; ++k) bb.v[k] = __ldcg(b + k * psb + rb + r);
    st<M>(b, psb, rb + r, add<M>(bb, neg(t)));
    if (fl.rows) __threadfence();
  }
  if (fl.rows) {
    __syncthreads();
    if (tid == 0) red_release_gpu(fl.rows + rb / nb, RB);  // this block's rows of the tile updated
  }
}

// Us (nullable): nb x (ntiles nb) workspace for the row-scaled copy (the diagonal absorbed, see A7)
template <int M>
// info_off: global row index of the first tile's first row (dev_info reports global 1-based rows)
void launch_invert(cudaStream_t st, int64_t ntiles, int64_t nb, CMat U, Mat Vt, Mat Us, int* info, int64_t info_off) {
  const int threads = 256, nwarp = threads / 32;
  const int64_t ny = cdiv(nb, nwarp);
  dim3 grid((unsigned)ntiles, (unsigned)ny);
  const size_t smem = sizeof(double) * M * nb;
  if (Us.p) {
    const dim3 sgrid((unsigned)ntiles, (unsigned)std::max<int64_t>(1, std::min<int64_t>(8, nb / 16)));
    MDLS_LAUNCH(F_INVERT, st, scale_tiles_kernel<M><<<sgrid, threads, smem, st>>>(nb, U, Us, info, info_off));
    const CMat C = cm(Us);
    if (nb <= 32) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 1, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info, info_off));
    else if (nb <= 64) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 2, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info, info_off));
    else if (nb <= 128) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 4, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info, info_off));
    else MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 8, true><<<grid, threads, 0, st>>>(nb, U, C, Vt, info, info_off));
    return;
  }
  const CMat C{nullptr, 0, 0};
  if (nb <= 32) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 1, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info, info_off));
  else if (nb <= 64) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 2, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info, info_off));
  else if (nb <= 128) MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 4, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info, info_off));
  else MDLS_LAUNCH(F_INVERT, st, invert_tiles_kernel<M, 8, false><<<grid, threads, smem, st>>>(nb, U, C, Vt, info, info_off));
}

template <int M>
void launch_bs_mulinv(cudaStream_t st, int64_t nb, int64_t tile, CMat Vt, const double* b, int64_t psb, double* x,
                      int64_t psx, BsFlow fl, bool first) {
  const dim3 grid((unsigned)cdiv(nb, 8));
  if (nb <= 64) MDLS_LAUNCH(F_BS, st, launch_pdl(bs_mulinv_kernel<M, 2>, grid, dim3(256), 0, st, nb, tile, Vt, b, psb, x, psx, fl, (int)first));
  else if (nb <= 128) MDLS_LAUNCH(F_BS, st, launch_pdl(bs_mulinv_kernel<M, 4>, grid, dim3(256), 0, st, nb, tile, Vt, b, psb, x, psx, fl, (int)first));
  else MDLS_LAUNCH(F_BS, st, launch_pdl(bs_mulinv_kernel<M, 8>, grid, dim3(256), 0, st, nb, tile, Vt, b, psb, x, psx, fl, (int)first));
}

// 3-D tensor map of U for the update kernel's TMA stages: dims (rows, columns, limb planes), strides
// (ld, ps) doubles, box (RB, SC, M); 0 (use the LDGSTS path) when the operand is not 16-byte aligned, the
// driver entry point is missing, encoding fails, or MDLS_BS_TMA=0
inline int64_t base_cols_end(int64_t nb, int64_t tile) { return (tile + 1) * nb; }
inline int bs_tensor_map(CUtensorMap* tm, CMat U, int64_t rows, int64_t cols, int M, int RB, int SC) {
  static const bool env_on = [] {
    const char* v = getenv("MDLS_BS_TMA");
    return !(v && v[0] == '0');
  }();
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  std::memset(tm, 0, sizeof(*tm));
  if (!env_on || !encode || (U.ld % 2) || (U.ps % 2) || ((uintptr_t)U.p & 15)) return 0;
  const cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)cols, (cuuint64_t)M};
  const cuuint64_t strides[2] = {(cuuint64_t)U.ld * sizeof(double), (cuuint64_t)U.ps * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)RB, (cuuint32_t)SC, (cuuint32_t)M};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult rc = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(U.p), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS ? 1 : 0;
}

// rows [row0, row1): RB = 32 rows per CTA when that still gives two CTAs per SM, else RB = 8;
// NS stages of 16 KB (dynamic shared memory beyond 48 KB: attribute set once per device)
template <int M, int RB, int NS, int MINB, int NACC>
void bs_update_launch(cudaStream_t st, int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U, const double* x,
                      int64_t psx, double* b, int64_t psb, BsFlow fl) {
  static bool attr_set[kMaxDev];
  const int dev = cur_dev();
  const size_t smem = sizeof(double) * ((((size_t)M * nb + 15) & ~(size_t)15) + (size_t)NS * 2048);
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(bs_update_kernel<M, RB, NS, MINB, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * ((size_t)M * 256 + 16 + (size_t)NS * 2048)));
    attr_set[dev] = true;
  }
  CUtensorMap tm;
  const int use_tma = bs_tensor_map(&tm, U, row1, base_cols_end(nb, tile), M, RB, 2048 / (M * RB));
  MDLS_LAUNCH(F_BS, st, launch_pdl(bs_update_kernel<M, RB, NS, MINB, NACC>, dim3((unsigned)cdiv(row1 - row0, RB)),
                                    dim3(256), smem, st, nb, tile, row0, row1, U, x, psx, b, psb, tm, use_tma, fl));
}
// variant (MDLS_BSU): 0 = NS 4, two CTAs per SM, two accumulator chains per thread (default, measured
// 4.44 ms at config 4); 1 = the same with one chain (4.52 ms); 2 = NS 3, three CTAs per SM, two chains (5.17);
// 3 = NS 4, two CTAs per SM, four chains

template <int M, int RB>
void bs_update_variant(cudaStream_t st, int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U, const double* x,
                       int64_t psx, double* b, int64_t psb, BsFlow fl) {
  static const int v = [] {
    const char* e = getenv("MDLS_BSU");
    return e ? atoi(e) : 0;
  }();
  if (v == 1) bs_update_launch<M, RB, 4, 2, 1>(st, nb, tile, row0, row1, U, x, psx, b, psb, fl);
  else if (v == 3) bs_update_launch<M, RB, 4, 2, 4>(st, nb, tile, row0, row1, U, x, psx, b, psb, fl);
  else if (v == 2) bs_update_launch<M, RB, 3, 3, 2>(st, nb, tile, row0, row1, U, x, psx, b, psb, fl);
  else bs_update_launch<M, RB, 4, 2, 2>(st, nb, tile, row0, row1, U, x, psx, b, psb, fl);
}
template <int M>
void launch_bs_update(cudaStream_t st, int64_t nb, int64_t tile, int64_t row0, int64_t row1, CMat U, const double* x,
                      int64_t psx, double* b, int64_t psb, BsFlow fl) {
  const int64_t rows = row1 - row0;
  if (rows <= 0) return;
  if (cdiv(rows, 32) >= 2 * num_sms()) bs_update_variant<M, 32>(st, nb, tile, row0, row1, U, x, psx, b, psb, fl);
  else bs_update_variant<M, 8>(st, nb, tile, row0, row1, U, x, psx, b, psb, fl);
}

#define MDLS_INSTANTIATE_BS(MM)                                                                                \
  template void launch_invert<MM>(cudaStream_t, int64_t, int64_t, CMat, Mat, Mat, int*, int64_t);                                     \
  template void launch_bs_mulinv<MM>(cudaStream_t, int64_t, int64_t, CMat, const double*, int64_t, double*,    \
                                     int64_t, BsFlow, bool);                                                   \
  template void launch_bs_update<MM>(cudaStream_t, int64_t, int64_t, int64_t, int64_t, CMat, const double*,  \
                                     int64_t, double*, int64_t, BsFlow);

}  // namespace mdls
