// md GEMM instantiations for od (8 limbs).
#include "kern_gemm.cuh"
namespace mdls {
MDLS_INSTANTIATE_GEMM(8, true, false)
MDLS_INSTANTIATE_GEMM(8, false, true)
MDLS_INSTANTIATE_GEMM(8, false, false)
MDLS_INSTANTIATE_GEMM(8, true, true)
}  // namespace mdls
