// esn_extra.cu -- small device utilities behind the public Python API:
//  * esn_fold_coords: fold + grid-scale in original order (grid.py:152-168,
//    spreadinterp.py:90-101) -- the integer/float index work of setpts
//    exposed for parity checks;
//  * esn_direct: O(M N) direct exponential sums on the GPU in float64, the
//    product-side counterpart of oracle.py:52-151 (direct_type1/2/3);
//  * esn_plan_sort_view / esn_plan_bins: read-only views of a plan's bin sort.
#include <cuda_runtime.h>

#include "esn_internal.h"

namespace esn {

__global__ void k_fold(int64_t M, int coord_f32, const void *x, double n, double scale, double *g) {
    const double two_pi = 6.283185307179586;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        double v = coord_f32 ? (double)((const float *)x)[i] : ((const double *)x)[i];
        double r = fmod(v, two_pi);
        if (r < 0.0) r += two_pi;
        if (r >= two_pi) r = 0.0;
        double gg = r;
        if (n > 0.0) {
            gg = r * scale;
            if (gg >= n) gg -= n;
        }
        g[i] = isfinite(v) ? gg : 0.0;
    }
}

// One CTA per 1..4 targets; each thread strides over the points with a
// float64 sincos; block tree reduction in ascending lane order.
__global__ void __launch_bounds__(256) k_direct(int dim, int64_t M, const double *x, const double *y,
                                                const double *z, const double2 *c, int64_t nk, const double *s,
                                                const double *t, const double *u, double isign, double2 *out) {
    __shared__ double2 red[256];
    for (int64_t k = blockIdx.x; k < nk; k += gridDim.x) {
        const double sk = s[k], tk = dim > 1 ? t[k] : 0.0, uk = dim > 2 ? u[k] : 0.0;
        double are = 0.0, aim = 0.0;
        for (int64_t j = threadIdx.x; j < M; j += blockDim.x) {
            double ph = sk * x[j];
            if (dim > 1) ph = ph + tk * y[j];
            if (dim > 2) ph = ph + uk * z[j];
            double sn, cs;
            sincos(isign * ph, &sn, &cs);
            const double2 cj = c[j];
            are += cj.x * cs - cj.y * sn;
            aim += cj.x * sn + cj.y * cs;
        }
        red[threadIdx.x] = make_double2(are, aim);
        __syncthreads();
        for (int o = blockDim.x / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) {
                red[threadIdx.x].x += red[threadIdx.x + o].x;
                red[threadIdx.x].y += red[threadIdx.x + o].y;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) out[k] = red[0];
        __syncthreads();
    }
}

}  // namespace esn

using namespace esn;

extern "C" {

int esn_fold_coords(int64_t M, int coord_dtype, const void *x, int64_t n, void *g, void *stream) {
    if (M < 0 || n < 0) return fail(ESN_SIZE_ERROR, "bad fold arguments");
    if (M == 0) return ESN_SUCCESS;
    int64_t b = (M + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    k_fold<<<(int)b, 256, 0, (cudaStream_t)stream>>>(M, coord_dtype == ESN_F32, x, (double)n,
                                                      n > 0 ? (double)n / (2.0 * M_PI) : 1.0, (double *)g);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

int esn_direct(int dim, int64_t M, const void *x, const void *y, const void *z, const void *c, int64_t nk,
               const void *s, const void *t, const void *u, int isign, void *out, void *stream) {
    if (dim < 1 || dim > 3 || M < 0 || nk < 0) return fail(ESN_SIZE_ERROR, "bad direct-sum arguments");
    if (nk == 0) return ESN_SUCCESS;
    int64_t b = nk < 148 * 8 ? nk : 148 * 8;
    k_direct<<<(int)b, 256, 0, (cudaStream_t)stream>>>(dim, M, (const double *)x, (const double *)y,
                                                        (const double *)z, (const double2 *)c, nk,
                                                        (const double *)s, (const double *)t, (const double *)u,
                                                        (double)isign, (double2 *)out);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

}  // extern "C"
