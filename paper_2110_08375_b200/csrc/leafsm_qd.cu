// shared-memory leaf (rows per CTA beyond the register leaf) for qd (4 limbs).
#define MDLS_LEAF_SMEM_TU
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF_SMEM(4)
}  // namespace mdls
