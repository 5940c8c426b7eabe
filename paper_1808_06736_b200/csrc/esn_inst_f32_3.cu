// Instantiation: complex64/float32, 3D.
#define ESN_T float
#define ESN_D 3
#include "esn_inst.cuh"
