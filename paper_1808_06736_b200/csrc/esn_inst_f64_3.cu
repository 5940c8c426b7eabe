// Instantiation: complex128/float64, 3D.
#define ESN_T double
#define ESN_D 3
#include "esn_inst.cuh"
