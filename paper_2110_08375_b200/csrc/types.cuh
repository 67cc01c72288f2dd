// types.cuh -- operand descriptors shared by the kernels and the host drivers.
//
// All operands are limb-planar ("staggered"): limb l of element
// (i, j) of an (ptr, ld, ps) operand is ptr[l*ps + j*ld + i].  Kernels are
// templated on the limb count M (2 dd, 4 qd, 8 od) and run on the FP64 pipe;
// no tensor cores (multiple-double arithmetic is error-free transformations,
// not a plain contraction).  Every reduction has a fixed tree, so results are
// bitwise reproducible run to run.
#pragma once
#include <cooperative_groups.h>

#include <climits>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "md.cuh"

namespace mdls {
namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// launch accounting / per-stage tracing (defined in ledger.cu).  Every kernel
// launch of the library goes through MDLS_LAUNCH: it is counted, and when
// tracing is on it is bracketed by CUDA events on its own stream and charged to
// the current stage (the paper's per-stage tables) and kernel family.
// ---------------------------------------------------------------------------
enum Family { F_GEMM = 0, F_PANEL = 1, F_INVERT = 2, F_BS = 3, F_MISC = 4, F_NFAM = 5 };
void trace_begin(cudaStream_t st, int family);
void trace_end(cudaStream_t st, int family);
void set_stage(int stage);
// side streams / event pool for the look-ahead QR (ledger.cu).  Streams come in
// groups of kGroupStreams per device; side_stream(which) returns stream `which`
// of the calling thread's current group (StreamGroup), so independent problems of
// a batch run on disjoint stream sets and overlap on the device.
constexpr int kGroupStreams = 8;  // 0..5: the QR lanes (solver.cuh), 6: the group's main stream
constexpr int kMaxGroups = 16;
inline thread_local int g_stream_group = 0;
struct StreamGroup {
  int prev;
  explicit StreamGroup(int g) : prev(g_stream_group) { g_stream_group = g; }
  ~StreamGroup() { g_stream_group = prev; }
};
cudaStream_t side_stream(int which);
// library-owned CUDA graphs (plans, ledger.cu): capture_begin() returns a private stream of the
// current device in thread-local capture mode; capture_end() ends the capture and instantiates
struct PlanImpl {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int device = 0;
  int64_t launches = 0;  // library kernels per replay
};
cudaStream_t capture_begin();
int capture_end(cudaStream_t cs, int64_t launches, void** plan_out);
cudaEvent_t pool_event();
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start while its
// stream predecessor still runs; it calls pdl_trigger() early (lets ITS successor launch) and
// pdl_wait() before touching anything the predecessor writes (griddepcontrol.wait returns once
// the predecessor grid has completed and its memory is visible; a no-op without the attribute).
// Work that reads only inputs nobody in flight writes (e.g. U in the back substitution) goes
// before the wait, overlapping the predecessor's tail and the launch latency.  MDLS_PDL=0: off.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("MDLS_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#define MDLS_LAUNCH(FAM, ST, ...)          \
  do {                                     \
    ::mdls::trace_begin((ST), (FAM));      \
    __VA_ARGS__;                           \
    ::mdls::trace_end((ST), (FAM));        \
  } while (0)

struct Mat {
  double* p;
  int64_t ld, ps;
};
struct CMat {
  const double* p;
  int64_t ld, ps;
};

constexpr int64_t kMaxSplit = 8;

// per-device host state (kernel attributes, SM count, cluster support) is kept in
// arrays indexed by the CUDA device ordinal: one process may drive several GPUs
constexpr int kMaxDev = 64;
inline int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDev) ? d : 0;
}
// streaming multiprocessors of the current device (148 on B200)
inline int num_sms() {
  static int n[kMaxDev] = {0};
  const int d = cur_dev();
  if (n[d] <= 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    n[d] = v > 0 ? v : 148;
  }
  return n[d];
}
// largest thread-block cluster (16 non-portable, else 8) the current device can place with one
// whole-SM CTA per cluster rank (probed once per device, ledger.cu)
int max_cluster_size();

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// asynchronous global -> shared copies (LDGSTS): 8-byte granules, so any double-aligned operand
// (sub-matrix views with odd row offsets or odd leading dimensions included) can be staged; a
// false predicate copies nothing and zero-fills the destination
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(pred ? 8 : 0) : "memory");
}
// shared-memory address and mbarrier helpers (the leaf's DSMEM pushes, the back substitution's bulk copies)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "MDLS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MDLS_WAIT_%=;\n}\n" :: "r"(bar), "r"(parity) : "memory");
}
// back-substitution dataflow counters (solver.cuh::backsub): rows[j] = rows of tile j updated so far
// (nb per chain step), xrdy[i] = entries of x_i written; null rows = launch-ordered (PDL wait) mode
struct BsFlow {
  int* rows;
  int* xrdy;
  int64_t N;
};
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_geq(const int* p, int target) {
  while (ld_acquire_gpu(p) < target) __nanosleep(20);
}
// one-dimensional bulk copy global -> shared (TMA engine, UBLKCP): 16-byte aligned, size a multiple of 16;
// completes `bytes` on the mbarrier `bar` (armed by mbar_arm)
__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int grid_for(int64_t n, int threads) {
  int64_t g = cdiv(n, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 8 * num_sms()));
}


inline CMat cm(const Mat& a) { return CMat{a.p, a.ld, a.ps}; }
inline Mat sub(const Mat& a, int64_t i, int64_t j) { return Mat{a.p + i + j * a.ld, a.ld, a.ps}; }
inline CMat sub(const CMat& a, int64_t i, int64_t j) { return CMat{a.p + i + j * a.ld, a.ld, a.ps}; }

// md GEMM tile variants: <BM, BN, BK, TM, TN>; V = 0 large, 1 medium, 2 skinny-m
// (few output rows, e.g. W^T C), 3 skinny-n (few output columns, e.g. Q^T b)
template <int BM_, int BN_, int BK_, int TM_, int TN_, int MINB_ = 1>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, TM = TM_, TN = TN_, MINB = MINB_;  // MINB: CTAs per SM
  static constexpr int NT = (BM / TM) * (BN / TN);
};
template <int M, int V>
struct GemmTile;
// plain double (1d): the dd shapes (one FMA per pair instead of 12 FP64 operations)
template <> struct GemmTile<1, 0> : Tile<64, 64, 16, 4, 4> {};
template <> struct GemmTile<1, 1> : Tile<32, 32, 16, 2, 2> {};
template <> struct GemmTile<1, 2> : Tile<16, 64, 16, 1, 4> {};
template <> struct GemmTile<1, 3> : Tile<64, 16, 16, 4, 1> {};
// dd large tile 64 x 32, 4 x 2 outputs per thread, 80 registers, three CTAs per SM: alone the 64 x 64 / 4 x 4
// tile is faster (1024 x 1024 x 128: 0.133 vs 0.142 ms), but beside the leaf chain the solve is (4.37 -> 4.21 ms)
template <> struct GemmTile<2, 0> : Tile<64, 32, 16, 4, 2, 3> {};
template <> struct GemmTile<2, 1> : Tile<32, 32, 16, 2, 2> {};
template <> struct GemmTile<2, 2> : Tile<16, 64, 16, 1, 4> {};
template <> struct GemmTile<2, 3> : Tile<64, 16, 16, 4, 1> {};
template <> struct GemmTile<4, 0> : Tile<32, 32, 16, 2, 2> {};
template <> struct GemmTile<4, 1> : Tile<16, 16, 16, 1, 1> {};
template <> struct GemmTile<4, 2> : Tile<16, 32, 16, 1, 2> {};
template <> struct GemmTile<4, 3> : Tile<32, 16, 16, 2, 1> {};
template <> struct GemmTile<8, 0> : Tile<32, 16, 16, 2, 1> {};
template <> struct GemmTile<8, 1> : Tile<16, 16, 16, 1, 1> {};
template <> struct GemmTile<8, 2> : Tile<8, 32, 16, 1, 1> {};
template <> struct GemmTile<8, 3> : Tile<32, 8, 16, 1, 1> {};
constexpr int64_t kMaxSplitK = 64;

// CTA cap of the md GEMMs issued by this host thread (0: none).  A capped product runs its
// tiles in a grid-stride loop on at most that many CTAs, so a long low-priority product (the
// forward Q accumulation) leaves CTA slots free for the latency-critical updates of the
// factorisation chain.  Set with the RAII GemmCap.
inline thread_local int64_t g_gemm_cta_cap = 0;
struct GemmCap {
  int64_t prev;
  explicit GemmCap(int64_t cap) : prev(g_gemm_cta_cap) { g_gemm_cta_cap = cap; }
  ~GemmCap() { g_gemm_cta_cap = prev; }
};

struct GemmArgs {
  int64_t m, n, k;
  const double* A;
  int64_t lda, psa;
  const double* B;
  int64_t ldb, psb;
  double* C;
  int64_t ldc, psc;
  int mode;
  int64_t kc;     // k chunk per split
  double* part;   // split partials (nullptr: no split)
  int64_t S;      // number of splits
  // stream-K (sk_w > 0): CTA p computes the k-iterations [p*sk_w, (p+1)*sk_w) of the tile-major iteration
  // space (tiles x sk_I k-tiles); a tile split over CTAs is finished by the CTA holding its last k-tile,
  // which merges the others' partials (sk_part, one slot per CTA) in k order after their flags
  int64_t sk_w = 0, sk_I = 0;
  int* sk_flags = nullptr;
  double* sk_part = nullptr;
};


}  // namespace mdls
