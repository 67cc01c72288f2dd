// tile inversion / back substitution instantiations for plain double (1 limb, "1d").
#include "kern_bs.cuh"
namespace mdls {
MDLS_INSTANTIATE_BS(1)
}  // namespace mdls
