// C-ABI entry points for the od precision (8 limbs); see include/mdls.h.
#define MDLS_P od
#define MDLS_M 8
#include "api.cuh"
