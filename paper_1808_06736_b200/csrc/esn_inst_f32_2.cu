// Instantiation: complex64/float32, 2D.
#define ESN_T float
#define ESN_D 2
#include "esn_inst.cuh"
