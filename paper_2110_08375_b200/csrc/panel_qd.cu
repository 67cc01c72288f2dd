// panel-factorisation instantiation for qd (4 limbs).
#include "kern_panel.cuh"
namespace mdls {
MDLS_INSTANTIATE_PANEL(4)
}  // namespace mdls
