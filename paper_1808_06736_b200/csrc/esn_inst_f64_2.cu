// Instantiation: complex128/float64, 2D.
#define ESN_T double
#define ESN_D 2
#include "esn_inst.cuh"
