// esn_extra.cu -- small device utilities behind the public Python API:
//  * esn_fold_coords: fold + grid-scale in original order (grid.py:152-168,
//    spreadinterp.py:90-101) -- the integer/float index work of setpts
//    exposed for parity checks;
//  * esn_direct: O(M N) direct exponential sums on the GPU in float64, the
//    product-side counterpart of oracle.py:52-151 (direct_type1/2/3);
//  * esn_plan_sort_view / esn_plan_bins: read-only views of a plan's bin sort.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// 2D type 1, float32, n2 = 1024 (c5): the y-direction FFT of only the N1
// needed columns, fused with the deconvolution (k_colfft1024_deconv), after
// a 1D cuFFT pass along x (batch ntransf * n2).  cuFFT's 2D plan spends
// ~250 us on its y pass for c5 and the separate deconvolution another 52 us
// (read + write of the modes); this kernel reads half the fine grid once
// and writes only the N1 x N2 modes (142 us).  Other shapes keep cuFFT 2D
// + k_deconv_rows (a radix-2 shared-memory variant for every power of two
// was measured slower than cuFFT: 338 us, ten smem passes).
namespace esn {

// n2 = 1024, float32: four-step column FFT (1024 = 32 x 32) in registers.
// Thread (c, j) of a CW = 8 column tile loads x[j + 32 m] (m < 32) of its
// column straight from the x-transformed grid, runs a 32-point FFT over m
// in registers, applies w_1024^{j k} and parks A[k][j] in shared memory;
// thread (c, k) then runs the 32-point FFT over j and writes the needed
// rows k + 32 j' with the deconvolution factors.  Two shared-memory passes
// instead of ten (radix-2 kernel above: smem-bound at ~340 us for c5).
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

constexpr int rev5(int i) {
    return ((i & 1) << 4) | ((i & 2) << 2) | (i & 4) | ((i & 8) >> 2) | ((i & 16) >> 4);
}

// in-place radix-2 DIT FFT of 32 register values given in BIT-REVERSED
// order (natural order out); twiddles w_32^k = tw[32 k] of the w_1024 table
__device__ __forceinline__ void fft32_reg(float2 (&b)[32], const float2 *tw) {
#pragma unroll
    for (int s = 1; s <= 5; ++s) {
#pragma unroll
        for (int bf = 0; bf < 16; ++bf) {  // (constant trip counts: fully unrolled, register-resident)
            const int half = 1 << (s - 1), pos = bf & (half - 1), i0 = ((bf >> (s - 1)) << s) + pos;
            const float2 u = b[i0];
            const float2 v = pos == 0 ? b[i0 + half] : cmulf(b[i0 + half], tw[(pos << (5 - s)) << 5]);
            b[i0] = make_float2(u.x + v.x, u.y + v.y);
            b[i0 + half] = make_float2(u.x - v.x, u.y - v.y);
        }
    }
}

__global__ void __launch_bounds__(256, 2) k_colfft1024_deconv(int ntransf, int n1, int N1, int N2,
                                                              const float *grid, const float *twid, const float *p1,
                                                              const float *p2, float *f) {
    constexpr int n2 = 1024, CW = 8, PK = 32 * CW + 8;  // pitch of one k row (+64 B: 2-wavefront reads)
    extern __shared__ __align__(16) unsigned char cf4_smem[];
    float2 *s_t = reinterpret_cast<float2 *>(cf4_smem);  // [32][PK]
    float2 *s_tw = s_t + 32 * PK;                        // [512]
    float *s_p2 = reinterpret_cast<float *>(s_tw + 512);  // [N2 <= 1024]
    const float2 *g = reinterpret_cast<const float2 *>(grid);
    float2 *out = reinterpret_cast<float2 *>(f);
    const int tid = threadIdx.x, c = tid & (CW - 1), q = tid >> 3;  // q = j (pass A) / k (pass B)
    for (int i = tid; i < 512; i += 256) s_tw[i] = reinterpret_cast<const float2 *>(twid)[i];
    for (int i = tid; i < N2; i += 256) s_p2[i] = p2[i];
    __syncthreads();
    auto w1024 = [&](int t) {  // w^t, t < 1024
        const float2 v = s_tw[t & 511];
        return t & 512 ? make_float2(-v.x, -v.y) : v;
    };
    const int64_t G = (int64_t)n1 * n2;
    const int ntile = (N1 + CW - 1) / CW;
    for (int item = blockIdx.x; item < ntile * ntransf; item += gridDim.x) {
        const int t = item / ntile, k1i = (item - t * ntile) * CW + c;
        const bool live = k1i < N1;
        int k1 = k1i - N1 / 2;
        if (k1 < 0) k1 += n1;
        const float2 *col = g + (int64_t)t * G + k1;
        float2 a[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) a[rev5(m)] = live ? col[(int64_t)(q + 32 * m) * n1] : make_float2(0.f, 0.f);
        fft32_reg(a, s_tw);
#pragma unroll
        for (int k = 0; k < 32; ++k) s_t[k * PK + q * CW + c] = cmulf(a[k], w1024(q * k));
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; ++j) a[rev5(j)] = s_t[q * PK + j * CW + c];
        fft32_reg(a, s_tw);
        // (back to the thread's own slots: the row selection below indexes
        // dynamically, which a register array cannot)
#pragma unroll
        for (int j = 0; j < 32; ++j) s_t[q * PK + j * CW + c] = a[j];
        if (live) {
            const float f1 = p1[k1i];
            float2 *o = out + (int64_t)t * N2 * N1 + k1i;
#pragma unroll 4
            for (int jj = 0; jj < 32; ++jj) {
                const int y = q + 32 * jj;  // fine row
                int k2i = -1;
                if (y < N2 - N2 / 2) k2i = y + N2 / 2;
                else if (y >= n2 - N2 / 2) k2i = y - n2 + N2 / 2;
                if (k2i >= 0) {
                    const float2 v = s_t[q * PK + jj * CW + c];
                    const float fac = f1 * s_p2[k2i];
                    o[(int64_t)k2i * N1] = make_float2(v.x * fac, v.y * fac);
                }
            }
        }
        __syncthreads();
    }
}

int launch_colfft1024_deconv(int ntransf, int n1, int N1, int N2, const float *grid, const float *twid,
                             const float *p1, const float *p2, float *f, cudaStream_t st) {
    const int64_t items = (int64_t)((N1 + 7) / 8) * ntransf;
    const int blocks = (int)std::min<int64_t>(items, (int64_t)device_sm_count() * 2);
    constexpr size_t smem = (size_t)32 * (32 * 8 + 8) * 8 + 512 * 8 + 1024 * 4;
    ESN_CUDA_TRY(cudaFuncSetAttribute(k_colfft1024_deconv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_colfft1024_deconv<<<blocks, 256, smem, st>>>(ntransf, n1, N1, N2, grid, twid, p1, p2, f);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

template <typename T>
int launch_colfft_deconv(int ntransf, int n1, int n2, int N1, int N2, const T *grid, const T *twid, const T *p1,
                         const T *p2, T *f, cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {
        if (n2 == 1024) return launch_colfft1024_deconv(ntransf, n1, N1, N2, grid, twid, p1, p2, f, st);
    }
    return fail(ESN_INTERNAL_ERROR, "fused column FFT: unsupported shape (n2 = %d, %zu-byte reals)", n2, sizeof(T));
}

bool colfft_eligible(int dtype, int dim, int n2) {
    static const bool off = [] {
        const char *e = getenv("ESN_COLFFT");
        return e && e[0] == '0';
    }();
    return !off && dim == 2 && dtype == ESN_F32 && n2 == 1024;
}

template int launch_colfft_deconv<double>(int, int, int, int, int, const double *, const double *, const double *,
                                          const double *, double *, cudaStream_t);
template int launch_colfft_deconv<float>(int, int, int, int, int, const float *, const float *, const float *,
                                         const float *, float *, cudaStream_t);

}  // namespace esn

namespace esn {

// complex64 -> complex128 (exact), for float64 type-1 host calls that take
// complex64 strengths (esn_opts.strength_dtype)
__global__ void k_upcast_c64(const float2 *in, double2 *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = in[i];
        out[i] = make_double2((double)v.x, (double)v.y);
    }
}

int launch_upcast_c64(const void *in, void *out, int64_t n, cudaStream_t st) {
    if (n <= 0) return ESN_SUCCESS;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)device_sm_count() * 16);
    k_upcast_c64<<<blocks, 256, 0, st>>>((const float2 *)in, (double2 *)out, n);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

}  // namespace esn
