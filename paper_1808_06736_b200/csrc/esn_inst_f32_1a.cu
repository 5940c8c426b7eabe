// Instantiation: complex64/float32, 1D, kernel widths 2..8.
#define ESN_T float
#define ESN_D 1
#define ESN_PART 0
#include "esn_inst.cuh"
