// Instantiation: complex128/float64, 3D, kernel widths 2..8.
#define ESN_T double
#define ESN_D 3
#define ESN_PART 0
#include "esn_inst.cuh"
