// C-ABI entry points for the dd precision (2 limbs); see include/mdls.h.
#define MDLS_P dd
#define MDLS_M 2
#include "api.cuh"
