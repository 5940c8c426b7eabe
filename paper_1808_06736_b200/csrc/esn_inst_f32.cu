// Precision instantiation: complex64 / float32.
#define ESN_T float
#include "esn_inst.cuh"
