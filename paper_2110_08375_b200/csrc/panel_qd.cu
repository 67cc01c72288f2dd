// leaf (sub-panel) factorisation instantiation for qd (4 limbs).
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF(4)
}  // namespace mdls
