// ledger.cu -- A10: canonical md-operation counts and Table-1-weighted flops,
// plus the precision-independent C-ABI helpers (strerror, version, limbs).
//
// The paper accumulates per kernel the md operations and converts them with its
// Table 1 sums.  Here the counts are closed forms of the
// minimum work of the algorithm as specified: Householder vectors
// (GVL Alg. 5.1.1), the in-panel reflector application, the W recurrence
// z = -beta (v + W Y^T v), the trailing update Y (W^T C), backward Q
// accumulation, the explicit Q^T b, zero-exploiting tile inversion, and the
// tiled back substitution.  Redundant work a kernel may do (dense
// products over structural zeros) is NOT counted.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/mdls.h"
#include "types.cuh"

// ---------------------------------------------------------------------------
// launch accounting and per-stage tracing (declared in types.cuh)
// ---------------------------------------------------------------------------
namespace mdls {
namespace {
std::atomic<int64_t> g_launches{0};
std::atomic<bool> g_trace{false};
thread_local int t_stage = MDLS_NSTAGES;
struct Rec {
  int stage, family;
  cudaEvent_t e0, e1;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
thread_local cudaEvent_t t_open = nullptr;

cudaEvent_t get_event() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void set_stage(int stage) { t_stage = stage; }

// library-owned non-blocking side streams, kGroupStreams per group and kMaxGroups
// groups per device (joined into the caller's stream by events in every call,
// so graph capture and ordering hold)
cudaStream_t side_stream(int which) {
  static std::mutex mu;
  static std::vector<cudaStream_t> streams;  // [(device * kMaxGroups + group) * kGroupStreams + which]
  int dev = 0;
  cudaGetDevice(&dev);
  const int w = which % kGroupStreams;
  const int grp = g_stream_group % kMaxGroups;
  std::lock_guard<std::mutex> lk(mu);
  const size_t idx = ((size_t)dev * kMaxGroups + (size_t)grp) * kGroupStreams + (size_t)w;
  if (streams.size() <= idx) streams.resize(idx + 1, nullptr);
  if (!streams[idx]) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    // priority levels (greatest is numerically smallest): the leaf chain (0) above the near-window and
    // far-window leaf updates (1, 5), inversion and the group main stream (6), above the W build and panel
    // products (2, 4), above Q (3)
    const int rank = (w == 0) ? 0 : (w == 1 || w == 5 || w == 6) ? 1 : (w == 3) ? 3 : 2;
    const int prio = (rank == 3) ? least : std::min(least, greatest + rank);
    cudaStreamCreateWithPriority(&streams[idx], cudaStreamNonBlocking, prio);
  }
  return streams[idx];
}

// round-robin pool of timing-free events (an event may be re-recorded once the
// waits on its previous record have been enqueued, which program order ensures)
cudaEvent_t pool_event() {
  static std::mutex mu;
  static std::vector<cudaEvent_t> pool;
  static size_t next = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (pool.empty()) {
    pool.resize(4096);
    for (auto& e : pool) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return pool[next++ % pool.size()];
}

void trace_begin(cudaStream_t st, int family) {
  (void)family;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_trace.load(std::memory_order_relaxed)) return;
  t_open = get_event();
  cudaEventRecord(t_open, st);
}

void trace_end(cudaStream_t st, int family) {
  if (!g_trace.load(std::memory_order_relaxed) || !t_open) return;
  cudaEvent_t e1 = get_event();
  cudaEventRecord(e1, st);
  std::lock_guard<std::mutex> lk(g_mu);
  g_recs.push_back(Rec{t_stage, family, t_open, e1});
  t_open = nullptr;
}
// cluster-size probe: a 16-CTA cluster of whole-SM CTAs (the register leaf takes the opt-in shared
// memory) needs the non-portable size; fall back to the portable 8 when the device cannot place it
__global__ void cluster_probe_kernel() {}
int max_cluster_size() {
  static int c[kMaxDev] = {0};
  const int d = cur_dev();
  if (c[d] == 0) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    cudaFuncSetAttribute(cluster_probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cluster_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = (size_t)optin;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, cluster_probe_kernel, &cfg);
    if (e != cudaSuccess) cudaGetLastError();
    c[d] = (e == cudaSuccess && n >= 1) ? 16 : 8;
  }
  return c[d];
}

}  // namespace mdls

namespace {

struct T1 {
  double add, mul, div, sqrt;
};
// Table 1 sums; an md sqrt is priced as 1 div + 2 mul (Z12).
// Index 3 is plain double (1d): every operation is one double flop.
constexpr T1 kT1[4] = {{20, 23, 70, 70 + 2 * 23}, {89, 336, 893, 893 + 2 * 336}, {269, 1742, 5126, 5126 + 2 * 1742},
                       {1, 1, 1, 1}};

void count_house(int64_t n_j, mdls_counts* c) {
  // sigma: n-1 squares and sums; x1^2 + sigma; v1; beta = 2 v1^2 / (sigma + v1^2);
  // 1/v1 and v = x * (1/v1).  A column of length 1 (the last of a square matrix) has
  // sigma = 0 (an empty sum): GVL Alg. 5.1.1 sets beta = 0 with no arithmetic.  The
  // x1 > 0 branch is counted (v1 = -sigma / (x1 + mu): one division more than x1 <= 0).
  if (n_j <= 1) return;
  c->mul[MDLS_ST_HOUSE] += (n_j - 1) + 1 + 2 + (n_j - 1);
  c->add[MDLS_ST_HOUSE] += (n_j - 1) + 1 + 1 + 1;
  c->div[MDLS_ST_HOUSE] += 3;
  c->sqrt[MDLS_ST_HOUSE] += 1;
}

void count_qr(int64_t M, int64_t K, int64_t nb, bool form_q, mdls_counts* c) {
  const int64_t N = K / nb;
  for (int64_t k = 0; k < N; ++k) {
    const int64_t j0 = k * nb, r = M - j0, ct = K - j0 - nb;
    for (int64_t l = 0; l < nb; ++l) {
      const int64_t j = j0 + l, n_j = M - j, q = nb - l - 1;
      count_house(n_j, c);
      // beta R^T v (q dots of length n_j, q scalings) + update R (q * n_j)
      c->mul[MDLS_ST_PANEL] += q * n_j + q + q * n_j;
      c->add[MDLS_ST_PANEL] += q * n_j + q * n_j;
      // W recurrence, column l: Y^T v (l dots over the overlap r - l), W (Y^T v) (r x l), v + ., -beta *
      c->mul[MDLS_ST_WY] += l * (r - l) + r * l + r;
      c->add[MDLS_ST_WY] += l * (r - l) + r * l + r;
    }
    if (ct > 0) {  // T = W^T C (nb x ct, reductions over r), C += Y T (r x ct, reductions over nb)
      c->mul[MDLS_ST_TRAILING] += nb * ct * r + r * ct * nb;
      c->add[MDLS_ST_TRAILING] += nb * ct * r + r * ct * nb;
    }
  }
  if (form_q) {
    for (int64_t k = N - 1; k >= 0; --k) {  // X = Y^T Q_tr (nb x r), Q_tr += W X (r x r)
      const int64_t r = M - k * nb;
      c->mul[MDLS_ST_FORM_Q] += 2 * nb * r * r;
      c->add[MDLS_ST_FORM_Q] += 2 * nb * r * r;
    }
  }
}

void count_qtb(int64_t M, int64_t K, int64_t nb, bool explicit_q, mdls_counts* c) {
  if (explicit_q) {
    c->mul[MDLS_ST_QTB] += M * M;
    c->add[MDLS_ST_QTB] += M * M;
  } else {
    for (int64_t k = 0; k < K / nb; ++k) {
      const int64_t r = M - k * nb;
      c->mul[MDLS_ST_QTB] += 2 * r * nb;
      c->add[MDLS_ST_QTB] += 2 * r * nb;
    }
  }
}

void count_bs(int64_t n, int64_t nb, mdls_counts* c) {
  const int64_t N = n / nb;
  // tile inversion exploiting zeros: column k (1-based) needs k(k-1)/2 pairs and
  // k-1 multiplications by the reciprocal diagonal (v_k = 1/u_kk itself is the
  // reciprocal); nb reciprocals per tile
  const int64_t pairs = nb * (nb * nb - 1) / 6;
  c->mul[MDLS_ST_INVERT] += N * (pairs + nb * (nb - 1) / 2);
  c->add[MDLS_ST_INVERT] += N * pairs;
  c->div[MDLS_ST_INVERT] += N * nb;
  // x_i = U_i^-1 b_i: upper-triangular matvec
  c->mul[MDLS_ST_MULINV] += N * nb * (nb + 1) / 2;
  c->add[MDLS_ST_MULINV] += N * nb * (nb + 1) / 2;
  // b_j -= A_ji x_i for j < i
  const int64_t upd = nb * nb * N * (N - 1) / 2;
  c->mul[MDLS_ST_BSUPDATE] += upd;
  c->add[MDLS_ST_BSUPDATE] += upd;
}

int count(int pidx, int op, int64_t M, int64_t K, int64_t nb, mdls_counts* out) {
  if (!out) return -6;
  if (nb < 1 || K < 1 || K % nb) return -4;
  if (op != MDLS_OP_BACKSUB && M < K) return -2;
  std::memset(out, 0, sizeof(*out));
  switch (op) {
    case MDLS_OP_QR: count_qr(M, K, nb, true, out); break;
    case MDLS_OP_BACKSUB: count_bs(K, nb, out); break;
    case MDLS_OP_LSTSQ:
      count_qr(M, K, nb, true, out);
      count_qtb(M, K, nb, true, out);
      count_bs(K, nb, out);
      break;
    case MDLS_OP_LSTSQ_NOQ:
      count_qr(M, K, nb, false, out);
      count_qtb(M, K, nb, false, out);
      count_bs(K, nb, out);
      break;
    case MDLS_OP_APPLY_QT: count_qtb(M, K, nb, false, out); break;
    default: return -1;
  }
  const T1 t = kT1[pidx];
  out->total_flops = 0;
  for (int s = 0; s < MDLS_NSTAGES; ++s) {
    out->flops[s] = out->add[s] * t.add + out->mul[s] * t.mul + out->div[s] * t.div +
                    out->sqrt[s] * t.sqrt;
    out->total_flops += out->flops[s];
  }
  return 0;
}

}  // namespace

namespace mdls {

cudaStream_t capture_begin() {
  static std::mutex mu;
  static std::vector<cudaStream_t> cs;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t st;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (cs.size() <= (size_t)dev) cs.resize((size_t)dev + 1, nullptr);
    if (!cs[(size_t)dev]) cudaStreamCreateWithFlags(&cs[(size_t)dev], cudaStreamNonBlocking);
    st = cs[(size_t)dev];
  }
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return nullptr;
  return st;
}

int capture_end(cudaStream_t cs, int64_t launches, void** plan_out) {
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(cs, &g);
  if (e != cudaSuccess || !g) {
    if (g) cudaGraphDestroy(g);
    return MDLS_ERR_CUDA;
  }
  cudaGraphExec_t x = nullptr;
  if (cudaGraphInstantiate(&x, g, 0) != cudaSuccess) {
    cudaGraphDestroy(g);
    return MDLS_ERR_CUDA;
  }
  auto* p = new PlanImpl;
  p->graph = g;
  p->exec = x;
  cudaGetDevice(&p->device);
  p->launches = launches;
  *plan_out = p;
  return 0;
}

}  // namespace mdls

extern "C" {

int mdls_plan_launch(void* plan, void* stream) {
  if (!plan) return -1;
  auto* p = static_cast<mdls::PlanImpl*>(plan);
  // the launches are counted like direct calls (the instrumentation's kernels per step)
  mdls::g_launches.fetch_add(p->launches, std::memory_order_relaxed);
  return cudaGraphLaunch(p->exec, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? 0 : MDLS_ERR_CUDA;
}

int64_t mdls_plan_launches(void* plan) { return plan ? static_cast<mdls::PlanImpl*>(plan)->launches : 0; }

void mdls_plan_destroy(void* plan) {
  if (!plan) return;
  auto* p = static_cast<mdls::PlanImpl*>(plan);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  delete p;
}

const char* mdls_strerror(int code) {
  if (code == 0) return "success";
  if (code == MDLS_ERR_CUDA) return "CUDA launch failed";
  if (code == MDLS_ERR_UNSUPPORTED) return "operation not supported for these arguments";
  if (code < 0 && code > -40) return "invalid argument (see include/mdls.h: -i = argument i)";
  return "unknown error";
}

int mdls_version(void) { return 1; }

int64_t mdls_launch_count(void) { return mdls::g_launches.load(); }

void mdls_trace_enable(int on) { mdls::g_trace.store(on != 0); }

int mdls_trace_collect(double* stage_ms, double* family_ms, int64_t* family_launches) {
  using namespace mdls;
  std::vector<Rec> recs;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    recs.swap(g_recs);
  }
  if (stage_ms) std::memset(stage_ms, 0, sizeof(double) * (MDLS_NSTAGES + 1));
  if (family_ms) std::memset(family_ms, 0, sizeof(double) * 5);
  if (family_launches) std::memset(family_launches, 0, sizeof(int64_t) * 5);
  int rc = 0;
  for (const Rec& r : recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) rc = -1;
    if (stage_ms) stage_ms[(r.stage >= 0 && r.stage <= MDLS_NSTAGES) ? r.stage : MDLS_NSTAGES] += ms;
    if (family_ms) family_ms[r.family] += ms;
    if (family_launches) family_launches[r.family] += 1;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  for (const Rec& r : recs) {
    g_pool.push_back(r.e0);
    g_pool.push_back(r.e1);
  }
  return rc ? MDLS_ERR_CUDA : (int)recs.size();
}

int mdls_limbs(int prec_index) {
  return prec_index == 0 ? 2 : prec_index == 1 ? 4 : prec_index == 2 ? 8 : prec_index == 3 ? 1 : -1;
}

int mdls_count_dd(int op, int64_t M, int64_t K, int64_t nb, mdls_counts* out) { return count(0, op, M, K, nb, out); }
int mdls_count_qd(int op, int64_t M, int64_t K, int64_t nb, mdls_counts* out) { return count(1, op, M, K, nb, out); }
int mdls_count_od(int op, int64_t M, int64_t K, int64_t nb, mdls_counts* out) { return count(2, op, M, K, nb, out); }
int mdls_count_d(int op, int64_t M, int64_t K, int64_t nb, mdls_counts* out) { return count(3, op, M, K, nb, out); }

}  // extern "C"
