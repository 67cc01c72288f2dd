// md GEMM instantiations for plain double (1 limb, "1d").
#include "kern_gemm.cuh"
namespace mdls {
MDLS_INSTANTIATE_GEMM(1, true, false)
MDLS_INSTANTIATE_GEMM(1, false, true)
MDLS_INSTANTIATE_GEMM(1, false, false)
MDLS_INSTANTIATE_GEMM(1, true, true)
}  // namespace mdls
