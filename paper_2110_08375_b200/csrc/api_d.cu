// C-ABI entry points for plain double (1 limb: "1d", the paper's double precision reference rows); see include/mdls.h.
#define MDLS_P d
#define MDLS_M 1
#include "api.cuh"
