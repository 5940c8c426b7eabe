// esn_internal.h -- shared declarations of the B200 NUFFT core (not part of
// the public ABI; see include/esnufft_b200.h).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "../../include/esnufft_b200.h"

namespace esn {

// ---- error plumbing: thread-local message + status int (errors.py:13-62)
void set_error(const char *msg);
int fail(int code, const char *fmt, ...);

// ---- host kernel math (esn_math.cpp)
int params_for_width(int w, double sigma, esn_kernel_params *out);
int select_params(double tol, double sigma, esn_kernel_params *out);
double class_tolerance(int w, double sigma);
int64_t next_smooth(int64_t n);
void gauss_legendre(int n, double *x, double *w);
void kernel_ft(const esn_kernel_params &p, double alpha, int64_t nk, const double *k, double *out);
int fseries_correction(const esn_kernel_params &p, int64_t n, int64_t nmodes, double *out);
int piecewise_poly(const esn_kernel_params &p, double *coeffs, double *residual);

constexpr int kMaxW = 16;
constexpr int kMaxCoef = kMaxW * (kMaxW + 4);

// ---- device-side argument blocks (passed by value; the Horner table rides
// in the kernel parameter bank, which every lane reads uniformly).
struct Geom {
    int dim;
    int w;
    int n[3];   // fine grid sizes (n_1, n_2, n_3), 1 beyond dim
    int bs[3];  // bin sizes in grid cells (footprint-origin bins)
    int nb[3];  // bins per dim
};

template <typename T>
struct KernelTab {
    T coef[kMaxCoef];  // w x (w+4), highest degree first
    T beta;
    int use_exact;
};

struct SetptsArgs {
    Geom g;
    int64_t M;
    int coord_f32;          // input coordinates are float (else double)
    int grid_units;         // coordinates already in grid units [0, n) (no fold)
    const void *x[3];
    double scale[3];        // n_d / (2 pi), computed on the host (grid.py:167)
    int *key;               // per original point: bin id
    int *rank;              // per original point: rank inside its bin
    int *bin_count;         // nbins (zeroed before)
    int *bin_start;         // nbins + 1
    int *perm;              // sorted position -> original index
    void *gs[3];            // sorted grid coordinates (plan dtype)
    unsigned long long *flags;  // [0..2] first non-finite per dim, [3..5] first |x|>3pi
    int check_bounds;
};

template <typename T>
struct SpreadArgs {
    Geom g;
    KernelTab<T> k;
    int64_t M;
    int ntransf;
    const T *gs[3];
    const int *perm;
    const int *bin_start;
    const int4 *subprob;     // (bin, start, count, 0)
    const int *nsub;         // device count of subproblems
    int *work;               // work-queue counter (zeroed before launch)
    const T *c;              // (ntransf, M) interleaved complex
    T *grid;                 // (ntransf, n3, n2, n1) interleaved complex
    int64_t gstride;         // complex cells per transform
    unsigned long long *flags;  // [6] first non-finite strength
};

// ---- launchers (esn_kernels.cu)
int launch_setpts(const SetptsArgs &a, int dtype, int nbins, int max_subprob, int4 *subprob,
                  int *nsub, int *scan_aux, cudaStream_t st);
template <typename T>
int launch_spread(const SpreadArgs<T> &a, int method, int nbins, cudaStream_t st);
template <typename T>
int launch_interp(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st);
template <typename T>
int launch_deconv(int dim, int ntransf, const int *n, const int64_t *N, const T *grid, const T *p1,
                  const T *p2, const T *p3, T *f, cudaStream_t st);
template <typename T>
int launch_amplify(int dim, int ntransf, const int *n, const int64_t *N, const T *f, const T *p1,
                   const T *p2, const T *p3, T *grid, unsigned long long *flag, cudaStream_t st);

size_t tile_smem_bytes(int dim, int w, const int *bs, int dtype);
int device_sm_count();

}  // namespace esn

#define ESN_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return ::esn::fail(ESN_INTERNAL_ERROR, "CUDA error %s at %s:%d (%s)",       \
                               cudaGetErrorString(_e), __FILE__, __LINE__, #expr);      \
    } while (0)
