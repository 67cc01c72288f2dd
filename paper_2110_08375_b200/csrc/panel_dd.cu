// leaf (sub-panel) factorisation instantiation for dd (2 limbs).
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF(2)
}  // namespace mdls
