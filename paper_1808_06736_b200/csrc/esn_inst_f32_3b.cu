// Instantiation: complex64/float32, 3D, kernel widths 9..16.
#define ESN_T float
#define ESN_D 3
#define ESN_PART 1
#include "esn_inst.cuh"
