// Instantiation: complex64/float32, 2D, kernel widths 2..8.
#define ESN_T float
#define ESN_D 2
#define ESN_PART 0
#include "esn_inst.cuh"
