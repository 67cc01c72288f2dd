// md GEMM instantiations for qd (4 limbs).
#include "kern_gemm.cuh"
namespace mdls {
MDLS_INSTANTIATE_GEMM(4, true, false)
MDLS_INSTANTIATE_GEMM(4, false, true)
MDLS_INSTANTIATE_GEMM(4, false, false)
MDLS_INSTANTIATE_GEMM(4, true, true)
}  // namespace mdls
