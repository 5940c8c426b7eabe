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

// Sorted point record: float64 grid coordinates + original index, one
// aligned 32-byte record per point for every plan dtype.  setpts writes it
// with a single 256-bit store (STG.E.ENL2.256: a full L2 sector, so the
// scattered writes need no read-modify-write) and the spreader /
// interpolator read it coalesced with one 256-bit load.  float32 plans thus
// keep float64 coordinates until the kernel row is formed.
struct alignas(32) Rec {
    double g[3];
    int j;
    int pad;
};

struct SetptsArgs {
    Geom g;
    int sbl[3];             // log2 of the sub-bin size per dim (fine sort key)
    int spb;                // sub-bins per bin
    int nkeys;              // nchunk * nbins * spb
    int nbins_geo;          // geometric bins
    int64_t chunk_len;      // > 0: points per target chunk (key major part)
    double inv_chunk;       // 1 / chunk_len
    double inv_bs[3];       // 1 / bs (fast division, corrected exactly)
    int bs_log2[3];         // log2 bs when bs is a power of two, else -1
    int64_t M;
    int rev;                // record scatter walks the input back to front
    int coord_f32;          // input coordinates are float (else double)
    int grid_units;         // coordinates already in grid units [0, n) (no fold)
    const void *x[3];
    double scale[3];        // n_d / (2 pi), computed on the host (grid.py:167)
    int *key_count;         // nkeys (zeroed before)
    int *cursor;            // nkeys: exclusive scan of key_count (key start)
    int *key;               // M: sorted position of each point (written when store_pos)
    int store_pos;          // keep positions in key[] (batched strength permutation)
    int *bin_start;         // nbins + 1
    int *block_sums;        // scan scratch
    Rec *rec;               // M sorted records
    int64_t ibase;          // index offset of this point chunk (error reports)
    unsigned long long *flags;  // [0..2] first non-finite per dim, [3..5] first |x|>3pi
    int check_bounds;
    int hints;              // L2 cache hints in the record scatter (ESN_SCATTER_HINTS=0: off)
};

template <typename T>
struct SpreadArgs {
    Geom g;
    KernelTab<T> k;
    int64_t M;
    int ntransf;
    const Rec *rec;          // sorted point records
    const int *bin_start;
    const int4 *subprob;     // (bin, start, count, 0)
    const int *kstart;       // start of every fine sort key (bin-major, sub-cell minor)
    int spb;                 // sub-cells per bin
    int sbl[3];              // log2 sub-cell size per dim
    const int *nsub;         // device count of subproblems
    const int *subofs;       // first subproblem of every bin (type 1; nullptr: unused)
    int roll;                // 3D row spreader: z-rolling segments (small bins on average)
    const int *imb;          // batched 2D owner-computes plans: device flag set by setpts when the bin
                             // counts are badly imbalanced (clustered points) -> RED-flush spreader; or null
    int *work;               // work-queue counter (zeroed before launch)
    const T *c;              // (ntransf, M) interleaved complex
    T *grid;                 // (ntransf, n3, n2, n1) interleaved complex
    int64_t gstride;         // complex cells per transform
    int64_t ibase;           // index offset of this point chunk (error reports)
    unsigned long long *flags;  // [6] first non-finite strength
    int accumulate;          // add into the grid (owner-computes spreaders; else they overwrite it)
};

// ---- compile-time geometry of the spreaders (shared with the host planner)
template <typename T, int DIM, int W>
struct RowsCfg {
    static constexpr int BX = (sizeof(T) == 8) ? (W <= 8 ? 16 : 8) : (W <= 10 ? 32 : 16);
    static constexpr int X = BX + W - 1;
    static constexpr int RY = DIM == 3 ? 16 : 64;
    static constexpr int RZ = DIM == 3 ? 16 : 1;
    static constexpr int NT = RY * RZ;
    static constexpr int BY = RY - W + 1;
    static constexpr int BZ = DIM == 3 ? RZ - W + 1 : 1;
    static constexpr int CH = NT;  // staged points per chunk (one per thread)
    static constexpr int MINB = DIM == 3 ? 2 : 1;  // two CTAs per SM (<= 128 registers)
};

// Tile of the 3D row spreader (k_spread_rows3): RY x RZ rows of X cells in
// registers, one row per thread, warps of LY (y) x LZ (z) rows.  For w <= 7
// the tile is THIN in z (LZ = RZ = 8): every point's z footprint lies inside
// every warp's block, so a warp visit covers w / 8 of its z rows and only
// the y overlap varies (c3, w = 7: 61 % of the lanes covered, against 35 %
// for 8 x 4 blocks of a 16 x 16 tile); wider kernels keep the square tile.
#ifndef ESN_THIN_RY
#define ESN_THIN_RY 32
#endif
#ifndef ESN_THIN16_MAXW
#define ESN_THIN16_MAXW 10
#endif
template <typename T, int W>
struct Rows3Geo {
    static constexpr bool THIN = W <= 7;
    static constexpr bool THIN16 = !THIN && W <= ESN_THIN16_MAXW;  // z extent 16, warps 2 y x 16 z
    static constexpr int BX = RowsCfg<T, 3, W>::BX;
    static constexpr int X = BX + W - 1;
    static constexpr int LY = THIN ? 4 : (THIN16 ? 2 : 8), LZ = THIN ? 8 : (THIN16 ? 16 : 4);
    static constexpr int RY = THIN ? ESN_THIN_RY : 16, RZ = THIN ? 8 : 16;
    static constexpr int WY = RY / LY, WZ = RZ / LZ;  // warp blocks
    static constexpr int BY = RY - W + 1, BZ = RZ - W + 1;
    static constexpr int NT = RY * RZ;
    static_assert((NT == 256 || NT == 512) && WY * WZ * 32 == NT, "8 or 16 warps of 32 rows");
};

template <typename T, int W>
struct Batch2Cfg {
    static constexpr int BX = 16;
    static constexpr int X = BX + W - 1;
    static constexpr int BY = 16;
    static constexpr int RY = BY + W - 1;  // rows (one warp each)
    static constexpr int NT = RY * 32;
    static constexpr int CH = 64;
};

// ---- launchers (esn_kernels.cu)
// aux (optional): a second stream and two events of the caller; the
// subproblem tables (they need only the scanned bin starts) are then built
// beside the record scatter instead of after it
struct SetptsAux {
    cudaStream_t st = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    // optional: the count pass on its own stream (already ordered after its
    // inputs by the caller); `counted` joins it into the sort stream
    cudaStream_t count_st = nullptr;
    cudaEvent_t counted = nullptr;
};
int launch_setpts(const SetptsArgs &a, int nbins, int max_subprob, int4 *subprob, int *nsub, int *subofs,
                  cudaStream_t st, const SetptsAux *aux = nullptr);
constexpr int kScanTile = 4096;  // keys per scan block
// records in original order, no sort (small 1D type-1 plans, global-atomic spreader)
int launch_setpts_unsorted(const SetptsArgs &a, cudaStream_t st);
// device flag: 1 when the fullest bin holds > 2048 points and > 8x the mean (clustered points)
int launch_bin_imbalance(const int *bin_start, int nbins, int64_t M, int *flag, cudaStream_t st);
int launch_sort_view(int dtype, const void *rec, const int *bin_start, int nbins, int64_t M, int *perm,
                     int *keys, cudaStream_t st);
// Bin geometry the chosen spreader needs: (bx, by, bz); returns 0 if the
// method has no fixed geometry (global atomics).
int spreader_bins(int method, int dtype, int dim, int w, int ntransf, int *bs);
template <typename T>
int launch_spread(const SpreadArgs<T> &a, int method, int nbins, const int *key,
                  const int *kstart, T *cperm, cudaStream_t st);
// does the batched 2D path (needs a permuted-strength scratch) apply?
bool batched_spread(int dtype, int dim, int w, int ntransf, int method);
// does the batched 2D owner-computes spreader (writes every fine cell, no
// memset needed) apply?  Needs cell-resolution keys over 16 x 16 bins.
bool batched_owner(int dtype, int dim, int w, int ntransf, int method, const int *sbl, const int *bs);
bool batched_roll_off();
template <typename T>
int launch_interp(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st);
// per-(dtype, dim, width part) instantiations, one translation unit each
// so the heavy template sets compile in parallel: part 0 = widths 2..8,
// part 1 = widths 9..16 (kWidthSplit)
constexpr int kWidthSplit = 8;
template <typename T, int D, int P>
int launch_spread_dp(const SpreadArgs<T> &a, int method, const int *key, const int *kstart,
                     T *cperm, cudaStream_t st);
template <typename T, int D, int P>
int launch_interp_dp(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st);
template <typename T>
int launch_deconv(int dim, int ntransf, const int *n, const int64_t *N, const T *grid, const T *p1,
                  const T *p2, const T *p3, T *f, cudaStream_t st);
template <typename T>
int launch_amplify(int dim, int ntransf, const int *n, const int64_t *N, const T *f, const T *p1,
                   const T *p2, const T *p3, T *grid, unsigned long long *flag, cudaStream_t st);

int device_sm_count();
// index of the calling thread's current CUDA device, clamped to [0, 64)
int current_device();
// a launcher setting cached per device: kernel attributes (the dynamic
// shared-memory limit) and occupancy-derived grid sizes are per-device
// properties, so a process driving several GPUs keeps one slot for each
template <typename V>
struct PerDev {
    V v[64] = {};
    V &operator()() { return v[current_device()]; }
};

// 2D type 1 with a power-of-two n2: pruned y-FFT fused with the
// deconvolution (after a 1D cuFFT x pass); twid = e^{isign 2 pi i k / n2},
// k < n2 / 2, in the plan dtype
bool colfft_eligible(int dtype, int dim, int n2);
// complex64 -> complex128 (host calls with complex64 strengths for a float64 plan)
int launch_upcast_c64(const void *in, void *out, int64_t n, cudaStream_t st);
template <typename T>
int launch_colfft_deconv(int ntransf, int n1, int n2, int N1, int N2, const T *grid, const T *twid, const T *p1,
                         const T *p2, T *f, cudaStream_t st);

}  // namespace esn

#define ESN_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return ::esn::fail(ESN_INTERNAL_ERROR, "CUDA error %s at %s:%d (%s)",       \
                               cudaGetErrorString(_e), __FILE__, __LINE__, #expr);      \
    } while (0)
