// kern_gemm.cuh -- md GEMM on the FP64 pipe (trailing update, WY build, Q formation, Q^T b).
#pragma once
#include <cstdlib>

#include "types.cuh"

namespace mdls {

// ============================================================================
// md GEMM on the FP64 pipe: C (mode)= op(A) op(B)
//   op(A)(i, k) = TA ? A[k + i*lda] : A[i + k*lda]   (m x k)
//   op(B)(k, j) = TB ? B[j + k*ldb] : B[k + j*ldb]   (k x n)
// Shared-memory staged (limb-planar smem tiles), TM x TN register tile per
// thread, one md mul + one md add per output and k.  Split-K: blockIdx.z takes
// k range [z*kc, (z+1)*kc) and writes its partial tile to `part` (m x n per
// split, ld m, split z at column offset z*n, plane stride m*n*S); a fixed-order
// reduction kernel finishes.  mode: 0 C = P, 1 C += P, 2 C -= P, 3 C = -P.
// ============================================================================
template <int M>
__device__ __forceinline__ md<M> apply_mode(int mode, const md<M>& c, const md<M>& p) {
  switch (mode) {
    case 0: return p;
    case 1: return add<M>(c, p);
    case 2: return add<M>(c, neg(p));
    default: return neg(p);
  }
}


// pipeline depth and padded shared-memory rows per precision (dynamic shared memory)
template <int M, int V, bool TA, bool TB>
struct GemmSmem {
  using Tl = GemmTile<M, V>;
  static constexpr int STAGES = (M == 8) ? 2 : 3;
  // a +1 pad where the copy walks k fastest (transposed A, plain B): conflict-free scattered stores
  static constexpr int BMP = Tl::BM + (TA ? 1 : 0);
  static constexpr int BNP = Tl::BN + (TB ? 0 : 1);
  static constexpr int A_ST = M * Tl::BK * BMP;  // doubles per stage
  static constexpr int B_ST = M * Tl::BK * BNP;
  static constexpr size_t bytes = sizeof(double) * (size_t)STAGES * (A_ST + B_ST);
};

template <int M, int V, bool TA, bool TB>
__global__ void __launch_bounds__(GemmTile<M, V>::NT, GemmTile<M, V>::MINB) gemm_kernel(GemmArgs g) {
  using Tl = GemmTile<M, V>;
  using Sm = GemmSmem<M, V, TA, TB>;
  constexpr int BM = Tl::BM, BN = Tl::BN, BK = Tl::BK;
  constexpr int TM = Tl::TM, TN = Tl::TN;
  constexpr int NX = BN / TN, NY = BM / TM, NT = NX * NY;
  constexpr int STAGES = Sm::STAGES, BMP = Sm::BMP, BNP = Sm::BNP;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                           // [STAGES][M][BK][BMP]
  double* Bs = gsm + STAGES * Sm::A_ST;       // [STAGES][M][BK][BNP]

  const int tid = threadIdx.x;
  // consecutive lanes own consecutive output ROWS: the epilogue's C loads/stores and the split-K
  // partial stores are coalesced along the column-major planes (they dominate when k is small)
  const int ty = tid % NY, tx = tid / NY;
  const int64_t ntx = (g.n + BN - 1) / BN, nty = (g.m + BM - 1) / BM;

  // the k-tiles [kb, ke) of the output tile (i0, j0) into acc, through the cp.async stage ring
  auto run_tile = [&](int64_t i0, int64_t j0, int64_t kb, int64_t ke, Acc<M> (&acc)[TM][TN]) {
    const int nkt = (int)((ke - kb + BK - 1) / BK);
    // issue the copies of k-tile t into stage t % STAGES (consecutive threads walk the contiguous
    // direction of each operand: coalesced global reads)
    auto load_tile = [&](int t) {
      const int stg = t % STAGES;
      const int64_t k0 = kb + (int64_t)t * BK;
      double* as = As + stg * Sm::A_ST;
      double* bs = Bs + stg * Sm::B_ST;
      for (int e = tid; e < BM * BK; e += NT) {
        int ii, kk;
        if (TA) { kk = e % BK; ii = e / BK; } else { ii = e % BM; kk = e / BM; }
        const int64_t gi = i0 + ii, gk = k0 + kk;
        const bool ok = gi < g.m && gk < ke;
        const int64_t off = ok ? (TA ? (gk + gi * g.lda) : (gi + gk * g.lda)) : 0;
#pragma unroll
        for (int l = 0; l < M; ++l) cp_async8(as + (l * BK + kk) * BMP + ii, g.A + l * g.psa + off, ok);
      }
      for (int e = tid; e < BK * BN; e += NT) {
        int kk, jj;
        if (TB) { jj = e % BN; kk = e / BN; } else { kk = e % BK; jj = e / BK; }
        const int64_t gj = j0 + jj, gk = k0 + kk;
        const bool ok = gj < g.n && gk < ke;
        const int64_t off = ok ? (TB ? (gj + gk * g.ldb) : (gk + gj * g.ldb)) : 0;
#pragma unroll
        for (int l = 0; l < M; ++l) cp_async8(bs + (l * BK + kk) * BNP + jj, g.B + l * g.psb + off, ok);
      }
    };
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
      for (int u = 0; u < TN; ++u) acc[t][u].init();
#pragma unroll
    for (int t = 0; t < STAGES - 1; ++t) {
      if (t < nkt) load_tile(t);
      cp_async_commit();  // one group per tile slot, empty past the end (keeps the wait counts uniform)
    }
    for (int t = 0; t < nkt; ++t) {
      cp_async_wait<STAGES - 2>();  // this thread's copies of tile t have landed
      __syncthreads();              // everyone's have; and everyone finished computing tile t-1
      if (t + STAGES - 1 < nkt) load_tile(t + STAGES - 1);  // refill the stage tile t-1 used
      cp_async_commit();
      const double* as = As + (t % STAGES) * Sm::A_ST;
      const double* bs = Bs + (t % STAGES) * Sm::B_ST;
#pragma unroll 2
      for (int kk = 0; kk < BK; ++kk) {
        md<M> a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int l = 0; l < M; ++l) a[i].v[l] = as[(l * BK + kk) * BMP + ty + i * NY];
#pragma unroll
        for (int u = 0; u < TN; ++u)
#pragma unroll
          for (int l = 0; l < M; ++l) b[u].v[l] = bs[(l * BK + kk) * BNP + tx + u * NX];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int u = 0; u < TN; ++u) acc[i][u].add_prod(a[i], b[u]);
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int u = 0; u < TN; ++u) acc[i][u].renorm_bins();
    }
    cp_async_wait<0>();
    __syncthreads();  // every thread done with the stages before the next tile refills them
  };

  // C (mode)= acc, or the split-K partial z
  auto epilogue = [&](int64_t i0, int64_t j0, int64_t z, Acc<M> (&acc)[TM][TN]) {
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const int64_t gi = i0 + ty + t * NY;
      if (gi >= g.m) continue;
#pragma unroll
      for (int u = 0; u < TN; ++u) {
        const int64_t gj = j0 + tx + u * NX;
        if (gj >= g.n) continue;
        if (g.part) {
          const int64_t pps = g.m * g.n * g.S;
          st<M>(g.part, pps, gi + (gj + z * g.n) * g.m, acc[t][u].get());
        } else {
          const int64_t e = gi + gj * g.ldc;
          md<M> c = (g.mode == 1 || g.mode == 2) ? ld<M>(g.C, g.psc, e) : md_zero<M>();
          st<M>(g.C, g.psc, e, apply_mode<M>(g.mode, c, acc[t][u].get()));
        }
      }
    }
  };

  Acc<M> acc[TM][TN];
  if (g.sk_w == 0) {
    // work items (column tile fastest, then row tile, then split) in a grid-stride loop: one item per
    // CTA normally; a capped grid (GemmCap) keeps a low-priority product to part of the device
    const int64_t nitems = ntx * nty * g.S;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
      const int64_t z = item / (ntx * nty);
      const int64_t i0 = ((item / ntx) % nty) * BM, j0 = (item % ntx) * BN;
      const int64_t kb = z * g.kc;
      run_tile(i0, j0, kb, min(g.k, kb + g.kc), acc);
      epilogue(i0, j0, z, acc);
    }
    return;
  }
  // stream-K: this CTA's contiguous range of the tile-major iteration space, taken from its END: the last
  // segment (the head of a tile finished by a later CTA) is published first, and the first segment (the
  // tail of a tile started by earlier CTAs, which published their parts first) is finished last -- so no
  // CTA ever waits for more than the first segment of its predecessors
  constexpr int RS = TM * TN * Acc<M>::NV;  // partial doubles per thread
  const int64_t I = g.sk_I, W = g.sk_w, total = ntx * nty * I;
  const int64_t p = blockIdx.x;
  const int64_t beg = p * W;
  int64_t hi = min(total, beg + W);
  while (hi > beg) {
    const int64_t tile = (hi - 1) / I;
    const int64_t lo = max(beg, tile * I);
    const int64_t kf = lo - tile * I, kl = hi - tile * I;
    const int64_t i0 = ((tile / ntx) % nty) * BM, j0 = (tile % ntx) * BN;
    run_tile(i0, j0, kf * BK, min(g.k, kl * BK), acc);
    if (kf == 0 && kl == I) {
      epilogue(i0, j0, 0, acc);
    } else if (kl < I) {
      // not the tile's last k-tile: publish the partial (slot p; only a CTA's last segment can be partial)
      double* slot = g.sk_part + p * (int64_t)RS * NT;
#pragma unroll
      for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int u = 0; u < TN; ++u)
#pragma unroll
          for (int v = 0; v < Acc<M>::NV; ++v) __stcg(slot + ((t * TN + u) * Acc<M>::NV + v) * NT + tid, acc[t][u].r(v));
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicAdd(g.sk_flags + tile, 1);
    } else {
      // the tile's last k-tile: wait for the earlier segments (CTAs pf..p-1), merge their partials into this
      // CTA's part in CTA order (fixed: bitwise reproducible)
      const int64_t pf = (tile * I) / W;
      const int need = (int)(p - pf);
      if (tid == 0) {
        volatile int* f = g.sk_flags + tile;
        while (*f < need) __nanosleep(32);
        __threadfence();
      }
      __syncthreads();
      for (int64_t q = pf; q < p; ++q) {
        const double* slot = g.sk_part + q * (int64_t)RS * NT;
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
          for (int u = 0; u < TN; ++u) {
            Acc<M> o;
#pragma unroll
            for (int v = 0; v < Acc<M>::NV; ++v) o.r(v) = __ldcg(slot + ((t * TN + u) * Acc<M>::NV + v) * NT + tid);
            acc[t][u].merge(o);
          }
      }
      epilogue(i0, j0, 0, acc);
    }
    hi = lo;
  }
}

// launch one gemm_kernel with its dynamic shared memory (attribute set once per device)
template <int M, int V, bool TA, bool TB>
void gemm_set_attr() {
  using Sm = GemmSmem<M, V, TA, TB>;
  static bool attr_set[kMaxDev];
  const int dev = cur_dev();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(gemm_kernel<M, V, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sm::bytes);
    attr_set[dev] = true;
  }
}
template <int M, int V, bool TA, bool TB>
void gemm_kernel_launch(cudaStream_t st, const GemmArgs& g) {
  using Tl = GemmTile<M, V>;
  gemm_set_attr<M, V, TA, TB>();
  int64_t items = cdiv(g.m, Tl::BM) * cdiv(g.n, Tl::BN) * g.S;
  if (g_gemm_cta_cap > 0) items = std::min<int64_t>(items, g_gemm_cta_cap);
  const dim3 grid((unsigned)std::max<int64_t>(1, items));
  MDLS_LAUNCH(F_GEMM, st,
              gemm_kernel<M, V, TA, TB><<<grid, Tl::NT, GemmSmem<M, V, TA, TB>::bytes, st>>>(g));
}
// resident CTAs of this variant on the whole device (occupancy x SMs), once per device
template <int M, int V, bool TA, bool TB>
int64_t gemm_slots() {
  static int64_t slots[kMaxDev];
  const int dev = cur_dev();
  if (slots[dev] <= 0) {
    gemm_set_attr<M, V, TA, TB>();
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_kernel<M, V, TA, TB>, GemmTile<M, V>::NT,
                                                  GemmSmem<M, V, TA, TB>::bytes);
    slots[dev] = (int64_t)std::max(1, per_sm) * num_sms();
  }
  return slots[dev];
}

// C (mode)= sum_{z=0..S-1} part_z, in split order
template <int M>
__global__ void splitk_reduce_kernel(int64_t m, int64_t n, int64_t S, const double* __restrict__ part, double* C,
                                     int64_t ldc, int64_t psc, int mode) {
  const int64_t total = m * n, pps = m * n * S;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    // exact merges of the split partials (md.cuh Acc: bins = limbs), one normalisation
    Acc<M> acc;
    const md<M> p0 = ld<M>(part, pps, e);
#pragma unroll
    for (int k = 0; k < Acc<M>::NV; ++k) acc.r(k) = (k < M) ? p0.v[k] : 0.0;
#pragma unroll 4
    for (int64_t z = 1; z < S; ++z) {
      const md<M> pz = ld<M>(part, pps, i + (j + z * n) * m);
      Acc<M> o;
#pragma unroll
      for (int k = 0; k < Acc<M>::NV; ++k) o.r(k) = (k < M) ? pz.v[k] : 0.0;
      acc.merge(o);
    }
    const md<M> s = acc.get();
    const int64_t ce = i + j * ldc;
    md<M> c = (mode == 1 || mode == 2) ? ld<M>(C, psc, ce) : md_zero<M>();
    st<M>(C, psc, ce, apply_mode<M>(mode, c, s));
  }
}


// ---------------------------------------------------------------------------
// GEMM launcher: tile variant and split-K chosen from the shape so that small
// and skinny products (panel-internal updates, W^T C with few rows) still fill
// the 148 SMs; long reductions are split with a fixed-order partial reduction.
// ---------------------------------------------------------------------------
template <int M, int V, bool TA, bool TB>
void gemm_launch(cudaStream_t st, int64_t m, int64_t n, int64_t k, CMat A, CMat B, Mat C, int mode, double* part,
                 int64_t part_cap_elems) {
  using Tl = GemmTile<M, V>;
  const int64_t tiles = cdiv(m, Tl::BM) * cdiv(n, Tl::BN);
  // split-K: choose the split that minimises (waves of resident CTAs) x (k-tiles per CTA) plus the
  // partial round trip (written by the GEMM, read by the fixed-order reduction: ~0.3 (S + 2) k-tile
  // waves of the tiles' share of the device)
  const int64_t slots = g_gemm_cta_cap > 0 ? std::min<int64_t>(g_gemm_cta_cap, gemm_slots<M, V, TA, TB>())
                                           : gemm_slots<M, V, TA, TB>();
  const int64_t kt = cdiv(k, Tl::BK);
  int64_t S = 1;
  if (part && kt >= 4) {
    double best = 1e300;
    for (int64_t s = 1; s <= std::min<int64_t>(kMaxSplitK, kt / 2); ++s) {
      const int64_t per = cdiv(kt, s), se = cdiv(kt, per);
      if (se > 1 && m * n * se > part_cap_elems) break;
      const double cost = (double)(cdiv(tiles * se, slots) * per) +
                          (se > 1 ? 0.3 * (double)(se + 2) * (double)tiles / (double)slots : 0.0);
      if (cost < best - 1e-9) {
        best = cost;
        S = se;
      }
    }
  }
  int64_t kc = cdiv(cdiv(k, S), Tl::BK) * Tl::BK;
  S = std::max<int64_t>(1, cdiv(k, kc));
  GemmArgs g{m, n, k, A.p, A.ld, A.ps, B.p, B.ld, B.ps, C.p, C.ld, C.ps, mode, kc, S > 1 ? part : nullptr, S};
  // stream-K for a product of one or two waves of tiles (no split): the tiles x k-tiles iteration space is
  // cut into equal contiguous ranges, one per resident CTA slot, so every SM holds the same work
  // (256 tiles of 64 x 64 on 296 dd slots leave 40 SMs with one CTA otherwise)
  static const bool sk_on = [] {
    const char* v = getenv("MDLS_STREAMK");
    return !(v && v[0] == '0');
  }();
  if (sk_on && S == 1 && part && kt >= 2 && tiles <= 2 * slots && tiles % slots != 0 && tiles * kt >= slots) {
    const int64_t units = tiles * kt;
    const int64_t W = cdiv(units, slots), P = cdiv(units, W);
    constexpr int64_t RS = (int64_t)Tl::TM * Tl::TN * Acc<M>::NV * Tl::NT;  // partial doubles per CTA
    const int64_t flag_d = cdiv(tiles * (int64_t)sizeof(int), (int64_t)sizeof(double));
    if ((flag_d + P * RS) <= part_cap_elems * M) {
      g.sk_w = W;
      g.sk_I = kt;
      g.sk_flags = reinterpret_cast<int*>(part);
      g.sk_part = part + flag_d;
      cudaMemsetAsync(g.sk_flags, 0, (size_t)tiles * sizeof(int), st);
      gemm_set_attr<M, V, TA, TB>();
      MDLS_LAUNCH(F_GEMM, st,
                  gemm_kernel<M, V, TA, TB><<<(unsigned)P, Tl::NT, GemmSmem<M, V, TA, TB>::bytes, st>>>(g));
      return;
    }
  }
  gemm_kernel_launch<M, V, TA, TB>(st, g);
  if (S > 1)
    MDLS_LAUNCH(F_GEMM, st, splitk_reduce_kernel<M><<<grid_for(m * n, 256), 256, 0, st>>>(m, n, S, part, C.p, C.ld, C.ps, mode));
}

template <int M, bool TA, bool TB>
void gemm(cudaStream_t st, int64_t m, int64_t n, int64_t k, CMat A, CMat B, Mat C, int mode, double* part,
          int64_t part_cap_elems) {
  if (m <= 0 || n <= 0) return;
  const int64_t target = 2 * num_sms();
  if (m <= GemmTile<M, 2>::BM && n > m) {
    gemm_launch<M, 2, TA, TB>(st, m, n, k, A, B, C, mode, part, part_cap_elems);
  } else if (n <= GemmTile<M, 3>::BN && m > n) {
    gemm_launch<M, 3, TA, TB>(st, m, n, k, A, B, C, mode, part, part_cap_elems);
  } else {
    const int64_t t0 = cdiv(m, GemmTile<M, 0>::BM) * cdiv(n, GemmTile<M, 0>::BN);
    const bool can_split = part && k >= 8 * GemmTile<M, 0>::BK;
    // the large tile once it fills about a wave (2 CTAs per SM resident), or with split-K
    const int64_t v0_min = (2 * num_sms()) / 3;  // the large tile once it fills about 2/3 of a wave
    if (t0 >= v0_min || (can_split && t0 >= target / 8))
      gemm_launch<M, 0, TA, TB>(st, m, n, k, A, B, C, mode, part, part_cap_elems);
    else gemm_launch<M, 1, TA, TB>(st, m, n, k, A, B, C, mode, part, part_cap_elems);
  }
}

// ---------------------------------------------------------------------------
// X = -T^T (Y^T C) for a leaf's trailing update without forming W = -Y T:
// the split-K partials of Z = Y^T C (B x n) are summed (exact accumulator
// merges, fixed order) and multiplied by -T^T (T: B x B upper, ld 32) in one
// kernel; a CTA = 16 columns x B rows.  X then feeds C += Y X.
// ---------------------------------------------------------------------------
template <int M, int B, int ZG>
__global__ void __launch_bounds__(16 * B * ZG) splitk_reduce_t_kernel(int64_t n, int64_t S, const double* __restrict__ part,
                                                                      CMat T, double* X, int64_t ldx, int64_t psx) {
  // ZG thread groups split the S partials (group g sums z = g, g + ZG, ...: S / ZG dependent merges instead of S),
  // then group 0 merges the ZG sums in group order (fixed: bitwise reproducible)
  __shared__ Acc<M> Zp[ZG][16][B];
  __shared__ md<M> Z[16][B];
  const int p = threadIdx.x % B, jl = (threadIdx.x / B) % 16, zg = threadIdx.x / (16 * B);
  const int64_t j = (int64_t)blockIdx.x * 16 + jl;
  const int64_t pps = (int64_t)B * n * S;
  Acc<M> acc;
  acc.init();
  if (j < n) {
#pragma unroll 4
    for (int64_t z = zg; z < S; z += ZG) {  // unrolled: the partial loads are issued ahead of the merges
      const md<M> pz = ld<M>(part, pps, p + (j + z * n) * B);
      Acc<M> o;
#pragma unroll
      for (int k = 0; k < Acc<M>::NV; ++k) o.r(k) = (k < M) ? pz.v[k] : 0.0;
      acc.merge(o);
    }
  }
  Zp[zg][jl][p] = acc;
  __syncthreads();
  if (zg == 0 && j < n) {
#pragma unroll
    for (int g = 1; g < ZG; ++g) acc.merge(Zp[g][jl][p]);
    Z[jl][p] = acc.get();
  }
  __syncthreads();
  if (zg == 0 && j < n) {
    Acc<M> a2;
    a2.init();
    for (int q = 0; q <= p; ++q) a2.add_prod(ld<M>(T.p, T.ps, q + (int64_t)p * T.ld), Z[jl][q]);
    st<M>(X, psx, p + j * ldx, neg(a2.get()));
  }
}

// X (B x n) = -T^T (Y^T C): Y r x B, C r x n (both column-major), X with ld B
template <int M>
void leaf_t_product(cudaStream_t st, int B, int64_t n, int64_t r, CMat Y, CMat T, CMat C, Mat X, double* part,
                    int64_t part_cap_elems) {
  using Tl = GemmTile<M, 2>;
  const int64_t tiles = cdiv(B, Tl::BM) * cdiv(n, Tl::BN);
  const int64_t target = 2 * num_sms();
  int64_t S = std::min<int64_t>(kMaxSplitK, std::max<int64_t>(1, cdiv(target, tiles)));
  S = std::max<int64_t>(1, std::min<int64_t>(S, r / (2 * Tl::BK)));
  while (S > 1 && (int64_t)B * n * S > part_cap_elems) --S;
  const int64_t kc = cdiv(cdiv(r, S), Tl::BK) * Tl::BK;
  S = std::max<int64_t>(1, cdiv(r, kc));
  GemmArgs g{B, n, r, Y.p, Y.ld, Y.ps, C.p, C.ld, C.ps, nullptr, B, 0, 0, kc, part, S};
  gemm_kernel_launch<M, 2, true, false>(st, g);
  // z-groups per output: 4 (2 for od: registers and static shared memory); od leaves are 8 wide
  constexpr int ZG8 = (M == 8) ? 2 : 4, ZG16 = (M == 8) ? 1 : 4;
  if (B == 16)
    MDLS_LAUNCH(F_GEMM, st, splitk_reduce_t_kernel<M, 16, ZG16><<<(unsigned)cdiv(n, 16), 16 * 16 * ZG16, 0, st>>>(n, S, part, T, X.p, X.ld, X.ps));
  else
    MDLS_LAUNCH(F_GEMM, st, splitk_reduce_t_kernel<M, 8, ZG8><<<(unsigned)cdiv(n, 16), 16 * 8 * ZG8, 0, st>>>(n, S, part, T, X.p, X.ld, X.ps));
}


// leaf_t_product is instantiated once per precision (with the TA = true, TB = false GEMM)
#define MDLS_INSTANTIATE_LEAF_T(MM, TA, TB) MDLS_INSTANTIATE_LEAF_T_##TA##_##TB(MM)
#define MDLS_INSTANTIATE_LEAF_T_true_false(MM) \
  template void leaf_t_product<MM>(cudaStream_t, int, int64_t, int64_t, CMat, CMat, CMat, Mat, double*, int64_t);
#define MDLS_INSTANTIATE_LEAF_T_false_true(MM)
#define MDLS_INSTANTIATE_LEAF_T_false_false(MM)
#define MDLS_INSTANTIATE_LEAF_T_true_true(MM)

#define MDLS_INSTANTIATE_GEMM(MM, TA, TB)                                                                   \
  template void gemm<MM, TA, TB>(cudaStream_t, int64_t, int64_t, int64_t, CMat, CMat, Mat, int, double*, int64_t); \
  MDLS_INSTANTIATE_LEAF_T(MM, TA, TB)

}  // namespace mdls
