// leaf (sub-panel) factorisation instantiation for od (8 limbs).
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF(8)
}  // namespace mdls
