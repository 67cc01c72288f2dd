// tile inversion / back substitution instantiations for dd (2 limbs).
#include "kern_bs.cuh"
namespace mdls {
MDLS_INSTANTIATE_BS(2)
}  // namespace mdls
