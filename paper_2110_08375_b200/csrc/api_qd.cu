// C-ABI entry points for the qd precision (4 limbs); see include/mdls.h.
#define MDLS_P qd
#define MDLS_M 4
#include "api.cuh"
