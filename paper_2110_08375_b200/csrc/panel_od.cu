// panel-factorisation instantiation for od (8 limbs).
#include "kern_panel.cuh"
namespace mdls {
MDLS_INSTANTIATE_PANEL(8)
}  // namespace mdls
