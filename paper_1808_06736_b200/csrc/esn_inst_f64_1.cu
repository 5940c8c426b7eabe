// Instantiation: complex128/float64, 1D.
#define ESN_T double
#define ESN_D 1
#include "esn_inst.cuh"
