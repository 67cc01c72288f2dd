// tile inversion / back substitution instantiations for od (8 limbs).
#include "kern_bs.cuh"
namespace mdls {
MDLS_INSTANTIATE_BS(8)
}  // namespace mdls
