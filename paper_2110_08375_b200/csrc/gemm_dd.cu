// md GEMM instantiations for dd (2 limbs).
#include "kern_gemm.cuh"
namespace mdls {
MDLS_INSTANTIATE_GEMM(2, true, false)
MDLS_INSTANTIATE_GEMM(2, false, true)
MDLS_INSTANTIATE_GEMM(2, false, false)
MDLS_INSTANTIATE_GEMM(2, true, true)
}  // namespace mdls
