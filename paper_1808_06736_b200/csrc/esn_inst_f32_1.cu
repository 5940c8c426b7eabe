// Instantiation: complex64/float32, 1D.
#define ESN_T float
#define ESN_D 1
#include "esn_inst.cuh"
