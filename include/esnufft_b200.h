/*
 * esnufft_b200.h -- C ABI of the B200-native ES-kernel NUFFT core
 * (libesnufft_b200.so, sm_100a).
 *
 * This is the drop-in boundary for the reference package `esnufft`
 * (/root/reference/pkg/src/esnufft).  The reference has no C FFI: its
 * boundary is the Python entry points, and its C-style convention lives in
 * the status-code bindings `esnufftpy`
 * (pkg/bindings/src/esnufftpy/__init__.py:1-24, 112-122): caller-allocated
 * C-contiguous outputs, an int status (0 or an ErrorCode), argument misuse
 * rejected with SIZE_ERROR before any core work, no handles retained.
 * Every entry point below states the reference interface it replaces.
 *
 * Conventions
 *  - complex arrays are interleaved (re, im) of the plan dtype
 *    (ESN_F64: double, i.e. complex128; ESN_F32: float, i.e. complex64);
 *  - mode arrays are C order (N_d, ..., N_1) with dimension 1 fastest and
 *    centered ascending indices k = -floor(N/2) .. ceil(N/2)-1
 *    (grid.py:61-111); batched arrays carry a leading ntransf axis;
 *  - "device" pointers are CUDA device addresses (e.g. torch
 *    .data_ptr()), "host" pointers are ordinary host memory;
 *  - calls on a plan are stream ordered on the plan's stream and return
 *    after enqueue; esn_plan_check() synchronises and reports data errors;
 *  - thread safety: distinct plans may be used from distinct threads; the
 *    cuFFT plan cache is mutex guarded (mirrors fft.py:87-111).
 */
#ifndef ESNUFFT_B200_H
#define ESNUFFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status table, identical to esnufft.errors.ErrorCode (errors.py:13-20). */
enum {
    ESN_SUCCESS = 0,
    ESN_BAD_TOLERANCE = 1,
    ESN_BOUNDS_VIOLATION = 2,
    ESN_SIZE_ERROR = 3,
    ESN_RESOURCE_ERROR = 4,
    ESN_DATA_ERROR = 5,
    ESN_INTERNAL_ERROR = 6
};

/* Arithmetic type of a plan (the reference is complex128 only,
 * spreadinterp.py:198 / transforms.py:146). */
enum { ESN_F64 = 0, ESN_F32 = 1 };
/* OR into esn_plan_setpts' coord_dtype: coordinates are already grid units
 * in [0, n) (the input convention of bin_sort, grid.py:202-211). */
enum { ESN_COORD_GRID_UNITS = 0x10 };

/* Spreader selection (esn_opts.method). */
enum {
    ESN_METHOD_AUTO = 0,
    ESN_METHOD_GLOBAL = 1, /* point-parallel, direct global atomics        */
    ESN_METHOD_TILE = 2    /* per-bin register-resident row tiles + halo flush */
};

/* Library version (major*10000 + minor*100 + patch). */
int esn_version(void);
/* Thread-local text of the last non-zero status. */
const char *esn_last_error(void);

/* ------------------------------------------------------------------ */
/* Host kernel math -- replaces kernel.py / grid.py helpers.           */
/* ------------------------------------------------------------------ */

/* KernelParams (kernel.py:51-84). */
typedef struct {
    int w;         /* width in fine-grid points, 2..16          */
    double beta;   /* ES shape, 2.30 w at sigma = 2              */
    double sigma;  /* 2.0 or 1.25                                */
    double gamma;  /* safety factor                              */
    int p_quad;    /* positive Gauss-Legendre nodes >= 1.5w + 2  */
} esn_kernel_params;

/* select_params(tolerance, sigma) -- kernel.py:110-131. */
int esn_select_params(double tol, double sigma, esn_kernel_params *out);
/* params_for_width(w, sigma) -- kernel.py:98-107. */
int esn_params_for_width(int w, double sigma, esn_kernel_params *out);
/* class_tolerance(w, sigma) -- kernel.py:134-143. */
double esn_class_tolerance(int w, double sigma);
/* next_smooth(n) -- grid.py:34-58. */
int esn_next_smooth(int64_t n, int64_t *out);
/* fine_grid_sizes(num_modes, sigma, w) -- grid.py:141-149. */
int esn_fine_grid_sizes(int dim, const int64_t *nmodes, double sigma, int w,
                        int64_t *sizes);
/* gauss_legendre(n) -- kernel.py:167-203 (host arrays of length n). */
int esn_gauss_legendre(int n, double *nodes, double *weights);
/* kernel_ft(params, alpha, ks) -- kernel.py:213-231 (host arrays). */
int esn_kernel_ft(const esn_kernel_params *p, double alpha, int64_t nk,
                  const double *k, double *out);
/* fseries_correction(params, n, N) -- kernel.py:234-288 (host array N). */
int esn_fseries_correction(const esn_kernel_params *p, int64_t n,
                           int64_t nmodes, double *out);
/* build_piecewise_poly(params).coeffs -- kernel.py:322-367; coeffs is a
 * host array w x (w+4), highest degree first; residual may be NULL. */
int esn_piecewise_poly(const esn_kernel_params *p, double *coeffs,
                       double *residual);

/* ------------------------------------------------------------------ */
/* Options -- TransformOptions (transforms.py:44-80) plus GPU knobs.   */
/* ------------------------------------------------------------------ */
typedef struct {
    double sigma;              /* 2.0 (default) or 1.25                     */
    int check_bounds;          /* reject |x| > 3 pi (grid.py:152-164)       */
    int use_exact_kernel;      /* exp/sqrt instead of Horner                */
    int64_t max_grid_values;   /* ResourceError cap (transforms.py:129-133) */
    int dtype;                 /* ESN_F64 / ESN_F32                         */
    int method;                /* ESN_METHOD_*                              */
    int bin_size[3];           /* 0 = auto                                  */
    int max_subprob;           /* 0 = auto                                  */
    int timing;                /* record per-stage CUDA events              */
    void *stream;              /* cudaStream_t, NULL = legacy default       */
    const esn_kernel_params *params; /* override select_params (may be NULL) */
    const double *coeffs;      /* override Horner table w x (w+4) (NULL)    */
    int strength_dtype;        /* host calls, type 1, float64 plans: ESN_F32 =
                                  complex64 input strengths, upcast exactly on
                                  the device (half the H2D bytes); 0 = the
                                  plan dtype                                  */
    int coord_dtype;           /* host calls: ESN_F32 = the x / y / z arrays
                                  hold float32 (read as float*); 0 = float64 */
} esn_opts;

void esn_default_opts(esn_opts *o);

/* ------------------------------------------------------------------ */
/* Plan API -- the transforms.py:136-218 pipelines as a reusable plan   */
/* (sort / phi-hat / cuFFT plan amortised across executes).  */
/* ------------------------------------------------------------------ */
typedef struct esn_plan_s *esn_plan;

/* type 1 (exec_type1, transforms.py:136) or 2 (exec_type2, :176).
 * nmodes = (N_1, .., N_dim).  isign = +1 / -1. */
int esn_plan_create(int type, int dim, const int64_t *nmodes, int isign,
                    int ntransf, double tol, const esn_opts *opts,
                    esn_plan *out);
/* Spread/interp-only plan on an explicit fine grid n = (n_1..n_dim):
 * replaces spreadinterp.spread / interp (spreadinterp.py:187, 259). */
int esn_spreader_create(int dim, const int64_t *nfine, int ntransf,
                        const esn_opts *opts, esn_plan *out);
/* Fold, grid-scale and bin-sort M points (device arrays of coord_dtype);
 * replaces build_point_set + ensure_sorted (spreadinterp.py:79-114).
 * Stream contract: a type-2 plan sorts on private side streams (the count
 * pass on one at the plan stream's priority, the scans and the record
 * scatter on a high-priority one) that first wait for the work already
 * queued on opts.stream; the coordinate arrays are read by those streams
 * until the next call on this plan
 * (execute / interp / spread / check / setpts), which orders opts.stream
 * after the sort.  Do not modify or free x / y / z before that call (or a
 * stream synchronisation).  Each setpts first joins any earlier pending
 * sort of the plan. */
int esn_plan_setpts(esn_plan p, int64_t M, int coord_dtype, const void *x,
                    const void *y, const void *z);
/* Run the transform (device arrays).  type 1: c (ntransf, M) -> f
 * (ntransf, N_d..N_1); type 2: f -> c. */
int esn_plan_execute(esn_plan p, void *c, void *f);
/* Spread c -> grid / interp grid -> c on the plan's fine grid (device
 * arrays; grid is (ntransf, n_d..n_1)); spread zeroes grid itself. */
int esn_plan_spread(esn_plan p, const void *c, void *grid);
int esn_plan_interp(esn_plan p, const void *grid, void *c);
/* Second half of a type-1 transform on a caller fine grid (e.g. the sum of
 * per-GPU spreads after an NCCL reduce): cuFFT in place on grid, then the
 * deconvolution into f (N_d..N_1).  esn_plan_spread(p, c, grid) followed by
 * esn_plan_finish_type1(p, grid, f) equals esn_plan_execute(p, c, f). */
int esn_plan_finish_type1(esn_plan p, void *grid, void *f);
/* Spread c ADDING into grid (device array (ntransf, n_d..n_1), not zeroed
 * here): the spreader's tile flushes are REDs (atomic adds), so several
 * plans -- on this GPU or on peer GPUs that map the same grid through
 * esn_peer_open -- may add into one grid concurrently.  This is the
 * point-split multi-GPU type 1 with the reduction fused into the spreader:
 * every rank flushes straight into the root's fine grid over NVLink
 * instead of spreading into a private grid that NCCL then reduces
 * (the reference has no counterpart: its spread() writes a
 * private array, spreadinterp.py:187-256).  SIZE_ERROR for the batched 2D
 * owner-computes spreader (plain stores, not concurrent-safe). */
int esn_plan_spread_add(esn_plan p, const void *c, void *grid);
/* Peer-mappable device memory (cudaMalloc + CUDA IPC): esn_peer_alloc
 * returns the pointer and a 64-byte handle that another PROCESS (one per
 * GPU) turns into a pointer valid on its own device with esn_peer_open
 * (peer access over NVLink enabled lazily).  esn_peer_close unmaps an
 * opened pointer, esn_peer_free releases an allocated one. */
int esn_peer_alloc(int64_t bytes, void **ptr, unsigned char handle[64]);
int esn_peer_open(const unsigned char handle[64], void **ptr);
int esn_peer_close(void *ptr);
int esn_peer_free(void *ptr);
/* Synchronise the plan stream and report data errors found on device:
 * returns ESN_DATA_ERROR / ESN_BOUNDS_VIOLATION with the offending point
 * index in info[0] and the (1-based) dimension in info[1] (0 = strength).*/
int esn_plan_check(esn_plan p, int64_t *info);
/* Stage seconds of the last setpts+execute, reference keys
 * (transforms.py:83-85); requires opts.timing. */
int esn_plan_stage_times(esn_plan p, double *sort_s, double *spread_s,
                         double *fft_s, double *correct_s);
/* Device seconds of the last spread kernel (type 1 / spreader) or interp
 * kernel (type 2) alone -- the roofline numerator's denominator. */
int esn_plan_hot_kernel_seconds(esn_plan p, double *seconds);
/* Fine grid sizes (n_1..n_3) and kernel parameters of a plan. */
int esn_plan_info(esn_plan p, int64_t *nfine, esn_kernel_params *kp);
/* Bin geometry of a plan: total bins, bin size and bins per dimension. */
int esn_plan_bins(esn_plan p, int *nbins, int *bin_size, int *bins_per_dim);
/* Work items (subproblems) of the last sort, the spread / interp kernels'
 * unit of dynamic scheduling (the tasks count of spreadinterp.py:165-184).
 * Waits for the plan stream. */
int esn_plan_tasks(esn_plan p, int64_t *ntasks);
/* Copy the plan's bin sort into caller device buffers (any may be NULL):
 * perm (M int32, sorted slot -> original index), keys (M int32, bin of each
 * original point), bin_start (nbins + 1 int32).  Replaces the
 * BinSortPermutation of grid.py:171-182. */
int esn_plan_sort_view(esn_plan p, void *perm, void *keys, void *bin_start);
/* Target chunks of a type-2 plan's sort order (set by esn_plan_setpts): with
 * nchunk > 1 the points are ordered by (chunk of original indices, bin,
 * sub-cell) so that one chunk's scattered outputs stay L2-resident while
 * it is interpolated; results are identical to the plain bin order.
 * esn_plan_sort_view is unavailable (SIZE_ERROR) on such a plan. */
int esn_plan_target_chunks(esn_plan p, int *nchunk);
/* Device scratch bytes held by the plan. */
int64_t esn_plan_device_bytes(esn_plan p);
int esn_plan_destroy(esn_plan p);

/* fft_exec(FftPlanKey, data) -- fft.py:114-124: in-place unnormalised
 * n-D FFT of ntransf device grids (n_1..n_dim), sign +1 applies
 * e^{+2 pi i l k / n} (the reference "FORWARD"). */
/* ---- type-3 device pieces (float64 / complex128 device buffers; replace
 * the numpy steps of transforms.py:267-351 around the composed spread and
 * type 2).  x0 / s0: per-dimension source / target shifts, gamma: rescale
 * factors, n: the type-3 fine grid (plan_type3_geometry, :245-264). */
/* c_out = conj?(c_in) * e^{i sum_d s0_d (x_d - x0_d)};  xr_d = (x_d - x0_d) / gamma_d */
int esn_type3_prephase(int dim, int64_t M, const double *x, const double *y, const double *z, const double *x0,
                       const double *s0, const double *gamma, int conj, const void *c_in, void *c_out, double *xr,
                       double *yr, double *zr, void *stream);
/* inner type-2 targets t_d = (2 pi / n_d) gamma_d (s_d - s0_d) */
int esn_type3_targets(int dim, int64_t K, const double *s1, const double *s2, const double *s3, const double *s0,
                      const double *gamma, const int64_t *n, double *t1, double *t2, double *t3, void *stream);
/* out *= prod_d (2 pi / n_d) / psi-hat_d(gamma_d (s_d - s0_d)) * e^{i sum_d x0_d s_d}, then conj? (in place) */
int esn_type3_correct(int dim, int64_t K, const double *s1, const double *s2, const double *s3, const double *x0,
                      const double *s0, const double *gamma, const int64_t *n, const esn_kernel_params *kp, int conj,
                      void *out, void *stream);
/* centring permutation of an (n_d..n_1) complex128 grid (numpy fftshift), out != in */
int esn_fftshift(int dim, const int64_t *n, const void *in, void *out, void *stream);

int esn_fft(int dim, int dtype, int ntransf, const int64_t *nfine,
            void *data, int sign, void *stream);

/* Explicit FFT plans: replace fft.py:79-84 (_build_plan), :87-96 (get_plan)
 * and :99-106 (clear_plan_cache).  One cuFFT handle and work area per plan;
 * executions of one plan are serialised (one stream at a time).  sign = +1
 * is the reference FORWARD (e^{+2 pi i lk/n}), -1 BACKWARD; in place,
 * unnormalised, (ntransf, n_d..n_1) C order. */
typedef struct esn_fft_plan_s *esn_fft_plan;
int esn_fft_plan_create(int dim, int dtype, int ntransf, const int64_t *nfine, esn_fft_plan *out);
int esn_fft_plan_exec(esn_fft_plan plan, void *data, int sign, void *stream);
int64_t esn_fft_plan_work_bytes(esn_fft_plan plan);
int esn_fft_plan_destroy(esn_fft_plan plan);
/* drop the handles esn_fft caches per (shape, dtype, batch, device, stream) */
int esn_fft_cache_clear(void);

/* fold_coords + grid scaling (grid.py:152-168, spreadinterp.py:90-101) on
 * device: g[i] = (x[i] mod 2 pi) * n / 2 pi in [0, n), float64 output,
 * original order (n = 0: the folded radians in [0, 2 pi)).  Non-finite
 * inputs give 0. */
int esn_fold_coords(int64_t M, int coord_dtype, const void *x, int64_t n,
                    void *g, void *stream);
/* Direct O(M nk) sums f_k = sum_j c_j exp(isign i s_k . x_j) in float64 on
 * device (oracle.py:52-88, direct_type3); t/u and y/z unused below dim. */
int esn_direct(int dim, int64_t M, const void *x, const void *y, const void *z,
               const void *c, int64_t nk, const void *s, const void *t,
               const void *u, int isign, void *out, void *stream);

/* ------------------------------------------------------------------ */
/* One-shot routines on HOST buffers, mirroring the esnufftpy status  */
/* bindings (bindings/src/esnufftpy/__init__.py:173-215).  Complex     */
/* buffers are interleaved complex128 (or complex64 when opts->dtype is */
/* ESN_F32 -- coordinates stay float64).  Host<->device copies happen  */
/* inside.  opts may be NULL.                                          */
/* ------------------------------------------------------------------ */
int esn_nufft1d1(int64_t M, const double *x, const void *c, int isign,
                 double tol, int64_t N1, void *f, const esn_opts *opts);
int esn_nufft2d1(int64_t M, const double *x, const double *y, const void *c,
                 int isign, double tol, int64_t N1, int64_t N2, void *f,
                 const esn_opts *opts);
int esn_nufft3d1(int64_t M, const double *x, const double *y, const double *z,
                 const void *c, int isign, double tol, int64_t N1, int64_t N2,
                 int64_t N3, void *f, const esn_opts *opts);
int esn_nufft1d2(int64_t M, const double *x, void *c, int isign, double tol,
                 int64_t N1, const void *f, const esn_opts *opts);
int esn_nufft2d2(int64_t M, const double *x, const double *y, void *c,
                 int isign, double tol, int64_t N1, int64_t N2, const void *f,
                 const esn_opts *opts);
int esn_nufft3d2(int64_t M, const double *x, const double *y, const double *z,
                 void *c, int isign, double tol, int64_t N1, int64_t N2,
                 int64_t N3, const void *f, const esn_opts *opts);
/* Batched host-buffer type 1/2 (ntransf strength / mode vectors sharing
 * one point set); x,y,z may be NULL beyond dim. */
/* Type 3 on host buffers (esnufftpy nufft{1,2,3}d3): f[k] = sum_j c[j]
 * exp(isign i s_k . x_j) for K targets (s, t, u); float64 / complex128. */
int esn_nufft1d3(int64_t M, const double *x, const void *c, int isign, double tol, int64_t K, const double *s,
                 void *f, const esn_opts *opts);
int esn_nufft2d3(int64_t M, const double *x, const double *y, const void *c, int isign, double tol, int64_t K,
                 const double *s, const double *t, void *f, const esn_opts *opts);
int esn_nufft3d3(int64_t M, const double *x, const double *y, const double *z, const void *c, int isign, double tol,
                 int64_t K, const double *s, const double *t, const double *u, void *f, const esn_opts *opts);
int esn_nufft_host(int type, int dim, int64_t M, const double *x,
                   const double *y, const double *z, int ntransf, void *c,
                   int isign, double tol, const int64_t *nmodes, void *f,
                   const esn_opts *opts);

#ifdef __cplusplus
}
#endif
#endif /* ESNUFFT_B200_H */
