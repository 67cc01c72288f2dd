// leaf (sub-panel) factorisation instantiation for plain double (1 limb, "1d").
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF(1)
}  // namespace mdls
