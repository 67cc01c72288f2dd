// panel-factorisation instantiation for dd (2 limbs).
#include "kern_panel.cuh"
namespace mdls {
MDLS_INSTANTIATE_PANEL(2)
}  // namespace mdls
