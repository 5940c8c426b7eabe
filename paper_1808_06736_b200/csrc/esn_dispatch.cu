// esn_dispatch.cu -- dimension dispatch over the per-(dtype, dim) kernel
// instantiations (esn_inst_<dtype>_<dim>.cu compile in parallel).
#include "esn_internal.h"

namespace esn {

template <typename T, int D>
static int launch_spread_d(const SpreadArgs<T> &a, int method, const int *key, const int *kstart,
                           T *cperm, cudaStream_t st) {
    return a.g.w <= kWidthSplit ? launch_spread_dp<T, D, 0>(a, method, key, kstart, cperm, st)
                                : launch_spread_dp<T, D, 1>(a, method, key, kstart, cperm, st);
}

template <typename T, int D>
static int launch_interp_d(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st) {
    return a.g.w <= kWidthSplit ? launch_interp_dp<T, D, 0>(a, cout, grid, st)
                                : launch_interp_dp<T, D, 1>(a, cout, grid, st);
}

template <typename T>
int launch_spread(const SpreadArgs<T> &a, int method, int nbins, const int *key, const int *kstart,
                  T *cperm, cudaStream_t st) {
    (void)nbins;
    switch (a.g.dim) {
        case 1:
            return launch_spread_d<T, 1>(a, method, key, kstart, cperm, st);
        case 2:
            return launch_spread_d<T, 2>(a, method, key, kstart, cperm, st);
        case 3:
            return launch_spread_d<T, 3>(a, method, key, kstart, cperm, st);
    }
    return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
}

template <typename T>
int launch_interp(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st) {
    switch (a.g.dim) {
        case 1:
            return launch_interp_d<T, 1>(a, cout, grid, st);
        case 2:
            return launch_interp_d<T, 2>(a, cout, grid, st);
        case 3:
            return launch_interp_d<T, 3>(a, cout, grid, st);
    }
    return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
}

template int launch_spread<double>(const SpreadArgs<double> &, int, int, const int *, const int *, double *,
                                   cudaStream_t);
template int launch_spread<float>(const SpreadArgs<float> &, int, int, const int *, const int *, float *,
                                  cudaStream_t);
template int launch_interp<double>(const SpreadArgs<double> &, double *, const double *, cudaStream_t);
template int launch_interp<float>(const SpreadArgs<float> &, float *, const float *, cudaStream_t);

}  // namespace esn
