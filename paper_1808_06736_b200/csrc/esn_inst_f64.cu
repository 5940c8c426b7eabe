// Precision instantiation: complex128 / float64.
#define ESN_T double
#include "esn_inst.cuh"
