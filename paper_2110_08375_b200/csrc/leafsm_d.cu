// shared-memory leaf (rows per CTA beyond the register leaf) for plain double (1 limb, "1d").
#define MDLS_LEAF_SMEM_TU
#include "kern_leaf.cuh"
namespace mdls {
MDLS_INSTANTIATE_LEAF_SMEM_WIDE(1)
MDLS_INSTANTIATE_LEAF_SMEM(1)
}  // namespace mdls
