// shared-memory leaf (rows per CTA beyond the register leaf) for dd (2 limbs).
#define MDLS_LEAF_SMEM_TU
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF_SMEM_WIDE(2)
MDLS_INSTANTIATE_LEAF_SMEM(2)
}  // namespace mdls
