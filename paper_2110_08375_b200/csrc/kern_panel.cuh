// kern_panel.cuh -- Householder panel factorisation by one thread-block cluster (A1 + A2).
#pragma once
#include "types.cuh"

namespace mdls {

// ============================================================================
// A1 + A2: panel factorisation by one thread-block cluster.
// Panel = columns [j0, j0+w) of A, rows [j0, Mrows).  Column l of the panel is
// owned by CTA (l mod C) of the cluster.  For each column j = j0+l:
//   owner: sigma = x(2:)^T x(2:) (block reduction), Householder scalars by
//          GVL Alg. 5.1.1: mu = sqrt(x1^2+sigma), v1 = x1-mu if
//          x1 <= 0 else -sigma/(x1+mu), beta = 2 v1^2/(sigma+v1^2); v = x * (1/v1);
//          writes v below the diagonal of A, the explicit Y column (1 on the
//          diagonal, 0 above), beta, and R_jj = mu; then one cluster barrier;
//   every CTA: for its own columns c > j: w_c = beta * (v . A(j:, c))
//          ("beta R^T * v"), A(j:, c) -= v w_c ("update R").
// ============================================================================
// Householder scalars, GVL Alg. 5.1.1, from sigma = x(2:)^T x(2:) and
// x1: mu = sqrt(x1^2 + sigma); v1 = x1 - mu if x1 <= 0 else -sigma/(x1 + mu);
// beta = 2 v1^2 / (sigma + v1^2); rv1 = 1/v1.  sigma = 0: beta = 0, mu = x1
// (P = I), returns 1.  Not inlined: one thread per column runs it.
template <int M>
__device__ __noinline__ int house_scalars(const md<M>& sigma, const md<M>& x1, md<M>& beta, md<M>& rv1, md<M>& mu) {
  if (sigma.v[0] == 0.0) {
    beta = md_zero<M>();
    rv1 = md_from<M>(1.0);
    mu = x1;
    return 1;
  }
  mu = sqrt<M>(add<M>(mul<M>(x1, x1), sigma));
  md<M> v1;
  if (x1.v[0] <= 0.0) v1 = sub<M>(x1, mu);
  else v1 = div<M>(neg(sigma), add<M>(x1, mu));
  const md<M> v1sq = mul<M>(v1, v1);
  beta = div<M>(mul<M>(md_from<M>(2.0), v1sq), add<M>(sigma, v1sq));
  rv1 = div<M>(md_from<M>(1.0), v1);
  return 0;
}

template <int M, int NT>
__global__ void __launch_bounds__(NT) panel_kernel(PanelArgs<M> a) {
  constexpr int NW = NT / 32;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  __shared__ md<M> red[NW];
  __shared__ md<M> colsum[NW];
  __shared__ md<M> sh_w[NW];  // w_c of the columns handled this step (indexed by local slot)
  __shared__ md<M> sh_scal[3];  // beta, 1/v1, mu
  __shared__ int sh_flag[2];

  const Mat A = a.A, Y = a.Y;
  for (int64_t l = 0; l < a.w; ++l) {
    const int64_t j = a.j0 + l;
    const int64_t nrow = a.Mrows - j;  // rows j..Mrows-1
    const int owner = (int)(l % C);
    if (rank == owner) {
      // ---- sigma = sum_{i>j} x_i^2 ----
      md<M> s = md_zero<M>();
      for (int64_t i = 1 + tid; i < nrow; i += NT) {
        md<M> x = ld<M>(A.p, A.ps, (j + i) + j * A.ld);
        s = fma<M>(s, x, x);
      }
      s = warp_sum<M>(s);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      if (tid == 0) {
        md<M> sigma = red[0];
        for (int q = 1; q < NW; ++q) sigma = add<M>(sigma, red[q]);
        md<M> x1 = ld<M>(A.p, A.ps, j + j * A.ld);
        md<M> beta, rv1, mu;
        const int deg = house_scalars<M>(sigma, x1, beta, rv1, mu);
        sh_scal[0] = beta;
        sh_scal[1] = rv1;
        sh_scal[2] = mu;
        sh_flag[0] = deg;
        st<M>(a.beta, a.bps, j, beta);
        st<M>(A.p, A.ps, j + j * A.ld, mu);
        bool bad = !(mu.v[0] != 0.0) || !isfinite(mu.v[0]);
        if (bad) atomicMin(a.info, (int)(j + 1));
      }
      __syncthreads();
      const md<M> rv1 = sh_scal[1];
      const int deg = sh_flag[0];
      // ---- v = x / v1 below the diagonal; explicit Y column ----
      for (int64_t i = tid; i < a.Mrows - a.j0; i += NT) {
        const int64_t gi = a.j0 + i;
        md<M> yv;
        if (gi < j) yv = md_zero<M>();
        else if (gi == j) yv = md_from<M>(1.0);
        else {
          md<M> x = ld<M>(A.p, A.ps, gi + j * A.ld);
          yv = deg ? x : mul<M>(x, rv1);
          st<M>(A.p, A.ps, gi + j * A.ld, yv);
        }
        st<M>(Y.p, Y.ps, gi + j * Y.ld, yv);
      }
      __threadfence();
    }
    cluster.sync();

    // ---- apply the reflector to this CTA's remaining panel columns ----
    // own columns c = j0 + l' with l' > l, l' = rank (mod C)
    int64_t first = l + 1 + (((int64_t)rank - (l + 1)) % C + C) % C;
    const int nc = (first < a.w) ? (int)((a.w - 1 - first) / C + 1) : 0;
    if (nc > 0) {
      const md<M> beta = ld_cg<M>(a.beta, a.bps, j);
      // warps -> (column slot, row part): G parts per column
      for (int cbase = 0; cbase < nc; cbase += NW) {
        const int ncb = min(NW, nc - cbase);
        const int G = NW / ncb;  // row parts per column
        const int slot = warp % ncb, part = warp / ncb;
        md<M> s = md_zero<M>();
        if (part < G) {
          const int64_t c = a.j0 + first + (int64_t)(cbase + slot) * C;
          for (int64_t i = part * 32 + lane; i < nrow; i += 32 * G) {
            md<M> v = (i == 0) ? md_from<M>(1.0) : ld_cg<M>(Y.p, Y.ps, (j + i) + j * Y.ld);
            md<M> x = ld<M>(A.p, A.ps, (j + i) + c * A.ld);
            s = fma<M>(s, v, x);
          }
        }
        s = warp_sum<M>(s);
        if (lane == 0) colsum[warp] = s;
        __syncthreads();
        if (tid < ncb) {
          md<M> t = colsum[tid];  // part 0 of slot tid
          for (int p = 1; p < G; ++p) t = add<M>(t, colsum[tid + p * ncb]);
          sh_w[tid] = mul<M>(beta, t);
        }
        __syncthreads();
        // update A(j:, c) -= v * w_c
        for (int64_t e = tid; e < nrow * ncb; e += NT) {
          const int64_t i = e % nrow;
          const int sl = (int)(e / nrow);
          const int64_t c = a.j0 + first + (int64_t)(cbase + sl) * C;
          md<M> v = (i == 0) ? md_from<M>(1.0) : ld_cg<M>(Y.p, Y.ps, (j + i) + j * Y.ld);
          md<M> x = ld<M>(A.p, A.ps, (j + i) + c * A.ld);
          x = fms<M>(x, v, sh_w[sl]);
          st<M>(A.p, A.ps, (j + i) + c * A.ld, x);
        }
        __syncthreads();
      }
    }
  }
}


// ---------------------------------------------------------------------------
// panel launch (one cluster)
// ---------------------------------------------------------------------------
template <int M>
struct PanelCfg {
  static constexpr int NT = (M == 8) ? 256 : 512;
};

template <int M>
cudaError_t launch_panel(cudaStream_t st, const PanelArgs<M>& pa) {
  constexpr int NT = PanelCfg<M>::NT;
  auto kern = panel_kernel<M, NT>;
  static bool attr_done = false;
  static int csize = 16;
  if (!attr_done) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      csize = 8;
    }
    attr_done = true;
  }
  int C = (int)std::min<int64_t>(csize, pa.w);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  trace_begin(st, F_PANEL);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, pa);
  if (e != cudaSuccess && C > 8) {  // fall back to a portable cluster size
    cudaGetLastError();
    csize = 8;
    C = (int)std::min<int64_t>(8, pa.w);
    cfg.gridDim = dim3(C, 1, 1);
    attr[0].val.clusterDim.x = C;
    e = cudaLaunchKernelEx(&cfg, kern, pa);
  }
  trace_end(st, F_PANEL);
  return e;
}

#define MDLS_INSTANTIATE_PANEL(MM) template cudaError_t launch_panel<MM>(cudaStream_t, const PanelArgs<MM>&);

}  // namespace mdls
