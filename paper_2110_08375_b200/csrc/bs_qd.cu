// tile inversion / back substitution instantiations for qd (4 limbs).
#include "kern_bs.cuh"
namespace mdls {
MDLS_INSTANTIATE_BS(4)
}  // namespace mdls
