// Instantiation: complex128/float64, 2D, kernel widths 9..16.
#define ESN_T double
#define ESN_D 2
#define ESN_PART 1
#include "esn_inst.cuh"
