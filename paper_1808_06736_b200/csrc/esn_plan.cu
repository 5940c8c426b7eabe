// esn_plan.cu -- plan runtime and the C ABI of libesnufft_b200.so.
//
// A plan owns everything a repeated transform can reuse: kernel parameters
// and the Horner table (kernel.py:322-367), the phi-hat correction vectors
// (kernel.py:234-288) on device, the bin geometry, the sorted point set, the
// fine grid and a cached cuFFT plan.  The pipelines are those of
// transforms.py:136-218 with the isign = -1 conjugations replaced by the
// opposite cuFFT direction (the kernel is real, so conj(F+(conj b)) = F-(b)).
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <chrono>
#include <tuple>
#include <vector>

#include "esn_internal.h"

namespace esn {
const char *last_error();
}
using namespace esn;

#define ESN_VERSION 100  // 0.1.0 series, mirrors esnufft.__version__ (__init__.py:21)

static inline size_t real_size(int dtype) { return dtype == ESN_F64 ? 8 : 4; }

// ---------------------------------------------------------------------------
// cuFFT handles.  A cuFFT handle owns one work area, so two FFTs may run
// concurrently only on different handles: every esn_plan owns its handle
// (created on first use, destroyed with the plan; captured graphs of the
// plan bake in the plan's own work area), and the plan-less esn_fft keeps a
// cache keyed by (shape, dtype, batch, device, STREAM) -- work on one stream
// is serialised by the stream itself.  The fft.py:87-111 analog.
namespace {
struct FftKey {
    int dim, n1, n2, n3, dtype, batch, device;
    uintptr_t stream;
    bool operator<(const FftKey &o) const {
        return std::tie(dim, n1, n2, n3, dtype, batch, device, stream) <
               std::tie(o.dim, o.n1, o.n2, o.n3, o.dtype, o.batch, o.device, o.stream);
    }
};
std::mutex g_fft_mu;
std::map<FftKey, cufftHandle> g_fft_cache;

int make_fft_plan(int dim, const int *n, int dtype, int batch, cufftHandle *out) {
    int dims[3];
    for (int d = 0; d < dim; ++d) dims[d] = n[dim - 1 - d];  // slowest first
    int64_t dist = 1;
    for (int d = 0; d < dim; ++d) dist *= n[d];
    cufftHandle h;
    cufftResult r = cufftPlanMany(&h, dim, dims, nullptr, 1, (int)dist, nullptr, 1, (int)dist,
                                  dtype == ESN_F64 ? CUFFT_Z2Z : CUFFT_C2C, batch);
    if (r != CUFFT_SUCCESS) return fail(ESN_INTERNAL_ERROR, "cufftPlanMany failed (%d)", (int)r);
    *out = h;
    return ESN_SUCCESS;
}

int exec_fft(cufftHandle h, int dtype, void *data, int sign, cudaStream_t st) {
    if (cufftSetStream(h, st) != CUFFT_SUCCESS) return fail(ESN_INTERNAL_ERROR, "cufftSetStream failed");
    // reference FORWARD = e^{+2 pi i lk/n} = CUFFT_INVERSE (fft.py:3-6, 52-59)
    const int dir = sign > 0 ? CUFFT_INVERSE : CUFFT_FORWARD;
    cufftResult r = dtype == ESN_F64
                        ? cufftExecZ2Z(h, (cufftDoubleComplex *)data, (cufftDoubleComplex *)data, dir)
                        : cufftExecC2C(h, (cufftComplex *)data, (cufftComplex *)data, dir);
    if (r != CUFFT_SUCCESS) return fail(ESN_INTERNAL_ERROR, "cufftExec failed (%d)", (int)r);
    return ESN_SUCCESS;
}

// plan-less FFT (esn_fft): one handle per (shape, stream)
int run_fft_cached(int dim, const int *n, int dtype, int batch, void *data, int sign, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    FftKey key{dim, n[0], dim > 1 ? n[1] : 1, dim > 2 ? n[2] : 1, dtype, batch, dev, (uintptr_t)st};
    std::lock_guard<std::mutex> lk(g_fft_mu);
    cufftHandle h;
    auto it = g_fft_cache.find(key);
    if (it != g_fft_cache.end()) {
        h = it->second;
    } else {
        if (int rc = make_fft_plan(dim, n, dtype, batch, &h)) return rc;
        g_fft_cache[key] = h;
    }
    return exec_fft(h, dtype, data, sign, st);
}
}  // namespace

// ---------------------------------------------------------------------------
struct esn_plan_s {
    int type = 0, dim = 0, dtype = ESN_F64, isign = 1, ntransf = 1;
    int64_t N[3] = {1, 1, 1};
    int n[3] = {1, 1, 1};
    esn_kernel_params kp{};
    std::vector<double> coeffs;
    esn_opts opts{};
    cudaStream_t st = nullptr;
    Geom geom{};
    int nbins = 1, maxsub = 8192, method = ESN_METHOD_TILE;
    int64_t G = 1;
    // device state
    void *pk[3] = {nullptr, nullptr, nullptr};
    Rec *rec = nullptr;  // sorted point records
    int *pkey = nullptr;  // per-point sorted position (batched plans: strength permutation)
    void *twid = nullptr;                   // column-FFT twiddles (2D type 1, power-of-two n2)
    void *cperm = nullptr;                  // batched strengths in sorted order
    int64_t cperm_bytes = 0;
    int *cursor = nullptr, *key_count = nullptr, *block_sums = nullptr;
    int *bin_start = nullptr, *subofs = nullptr, *nsub = nullptr, *work = nullptr;
    int sbl[3] = {0, 0, 0}, spb = 1, nkeys = 1;
    // type-2 target chunks: the sort key is (chunk of original indices, bin,
    // sub-cell), so the interpolator's scattered output writes of one chunk
    // land in an L2-sized window and merge into whole sectors there
    int nchunk = 1, nbk = 1;          // chunks; sort bins = nchunk * nbins
    int64_t chunk_len = 0;            // points per chunk (0: unchunked)
    int keycap = 0, bincap = 0;       // allocated key / sort-bin capacity
    int64_t keycap_req = (int64_t)8 << 20;  // key-space limit the current sbl was chosen for
    int4 *subprob = nullptr;
    unsigned long long *flags = nullptr;
    int *imb = nullptr;  // batched owner-computes plans: bins badly imbalanced (set by setpts on the device)
    void *grid = nullptr;
    int64_t M = -1, Mcap = 0, subcap = 0;
    int64_t device_bytes = 0;
    cudaEvent_t ev[8] = {};
    bool have_events = false;
    bool points_set = false;
    bool borrowed = false;    // pk[] and grid belong to another plan (pipeline helper)
    bool keep_flags = false;  // setpts keeps accumulating error flags (chunked runs)
    int64_t ibase = 0;        // original index of this plan's point 0 (chunked runs)
    // type-2 plans sort on a side stream (st2), so the next execute's
    // amplify + FFT (independent of the points) overlap the sort; consumers
    // of the sorted points join e_sorted on st first (join_sort)
    cudaStream_t st2 = nullptr;
    cudaEvent_t e_in = nullptr, e_sorted = nullptr;
    // aux stream of setpts (subproblem tables beside the record scatter);
    // type-2 side sorts also run their count pass on aux.count_st at the plan
    // stream's priority (see esn_plan_setpts)
    SetptsAux aux;
    bool sort_pending = false;
    // CUDA-graph replay of launch-bound calls (small M): the stream work of
    // setpts / execute is captured once per signature on a private stream
    // and replayed as one graph launch (slot 0: setpts, 1: execute)
    cudaStream_t gs = nullptr;
    cudaEvent_t g_in = nullptr, g_out = nullptr;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    uint64_t gsig[2] = {0, 0};
    int64_t gen = 0;        // bumped whenever a device buffer is (re)allocated
    bool capturing = false;
    bool graphs_off = false;  // a capture failed once: run directly from then on
    float last_ms[4] = {0, 0, 0, 0};  // sort, spread, fft, correct
    // this plan's own cuFFT handle (no work area shared with other plans)
    cufftHandle fft_h = 0;
    bool fft_made = false;
};

// the plan's FFT shape: 2D type 1 with the fused column FFT runs cuFFT along
// x only (batch ntransf * n2); everything else the full d-dimensional FFT
static int ensure_fft_plan(esn_plan p) {
    if (p->fft_made) return ESN_SUCCESS;
    int rc;
    if (p->twid && p->type == 1) {
        const int n1 = p->n[0];
        rc = make_fft_plan(1, &n1, p->dtype, p->ntransf * p->n[1], &p->fft_h);
    } else {
        rc = make_fft_plan(p->dim, p->n, p->dtype, p->ntransf, &p->fft_h);
    }
    if (rc) return rc;
    p->fft_made = true;
    return ESN_SUCCESS;
}

static int plan_fft(esn_plan p, void *data, cudaStream_t st) {
    if (int rc = ensure_fft_plan(p)) return rc;
    return exec_fft(p->fft_h, p->dtype, data, p->isign, st);
}

// timing events: inside a graph capture they become EXTERNAL event-record
// nodes (plain captured records cannot be timed)
static cudaError_t rec_ev(esn_plan p, cudaEvent_t e, cudaStream_t st) {
    return p->capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
}

template <typename P>
static int dmalloc(esn_plan p, P **ptr, size_t bytes) {
    ++p->gen;  // captured graphs hold device pointers
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc((void **)ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ESN_RESOURCE_ERROR, "device allocation of %zu bytes failed (%s)", bytes, cudaGetErrorString(e));
    }
    p->device_bytes += (int64_t)bytes;
    return ESN_SUCCESS;
}

static void dfree(void *ptr) {
    if (ptr) cudaFree(ptr);
}

// (re)allocate the key-space arrays when the key space / sort-bin count grew
static int ensure_key_space(esn_plan p) {
    int rc;
    if (p->nkeys > p->keycap) {
        dfree(p->key_count);
        dfree(p->cursor);
        dfree(p->block_sums);
        p->key_count = p->cursor = p->block_sums = nullptr;
        if ((rc = dmalloc(p, &p->key_count, sizeof(int) * p->nkeys))) return rc;
        // (+64 ints: the batched spreader stages key-start rows with 16-byte
        // copies that may run past the last key)
        if ((rc = dmalloc(p, &p->cursor, sizeof(int) * ((size_t)p->nkeys + 64)))) return rc;
        if ((rc = dmalloc(p, &p->block_sums, sizeof(int) * ((p->nkeys + kScanTile - 1) / kScanTile + 1)))) return rc;
        p->keycap = p->nkeys;
    }
    if (p->nbk > p->bincap) {
        dfree(p->bin_start);
        dfree(p->subofs);
        p->bin_start = p->subofs = nullptr;
        if ((rc = dmalloc(p, &p->bin_start, sizeof(int) * (p->nbk + 1)))) return rc;
        if ((rc = dmalloc(p, &p->subofs, sizeof(int) * (p->nbk + 1)))) return rc;
        p->bincap = p->nbk;
    }
    return ESN_SUCCESS;
}

template <int W>
static void rows_bins(int dtype, int dim, int ntransf, int *bs) {
    if (dim == 3) {
        // bins of the spreader that will run: k_spread_rows3 (Rows3Geo) or,
        // with ESN_SPREAD3=rows, the earlier k_spread_rows (RowsCfg)
        static const bool old_rows = [] {
            const char *e = getenv("ESN_SPREAD3");
            return e && std::string(e) == "rows";
        }();
        if (old_rows && dtype == ESN_F64) {
            bs[0] = RowsCfg<double, 3, W>::BX; bs[1] = RowsCfg<double, 3, W>::BY; bs[2] = RowsCfg<double, 3, W>::BZ;
        } else if (old_rows) {
            bs[0] = RowsCfg<float, 3, W>::BX; bs[1] = RowsCfg<float, 3, W>::BY; bs[2] = RowsCfg<float, 3, W>::BZ;
        } else if (dtype == ESN_F64) {
            bs[0] = Rows3Geo<double, W>::BX; bs[1] = Rows3Geo<double, W>::BY; bs[2] = Rows3Geo<double, W>::BZ;
        } else {
            bs[0] = Rows3Geo<float, W>::BX; bs[1] = Rows3Geo<float, W>::BY; bs[2] = Rows3Geo<float, W>::BZ;
        }
    } else if (esn::batched_spread(dtype, dim, W, ntransf, ESN_METHOD_TILE)) {
        bs[0] = Batch2Cfg<float, W>::BX; bs[1] = Batch2Cfg<float, W>::BY; bs[2] = 1;
    } else if (dtype == ESN_F64) {
        bs[0] = RowsCfg<double, 2, W>::BX; bs[1] = RowsCfg<double, 2, W>::BY; bs[2] = 1;
    } else {
        bs[0] = RowsCfg<float, 2, W>::BX; bs[1] = RowsCfg<float, 2, W>::BY; bs[2] = 1;
    }
}

int esn::spreader_bins(int method, int dtype, int dim, int w, int ntransf, int *bs) {
    bs[0] = bs[1] = bs[2] = 1;
    if (method == ESN_METHOD_GLOBAL || dim == 1) return 0;
    switch (w) {
#define ESN_BW(WW) case WW: rows_bins<WW>(dtype, dim, ntransf, bs); return 1;
        ESN_BW(2) ESN_BW(3) ESN_BW(4) ESN_BW(5) ESN_BW(6) ESN_BW(7) ESN_BW(8) ESN_BW(9)
        ESN_BW(10) ESN_BW(11) ESN_BW(12) ESN_BW(13) ESN_BW(14) ESN_BW(15) ESN_BW(16)
#undef ESN_BW
    }
    return 0;
}

static void set_key_space(esn_plan p, int nchunk, int64_t maxkeys = (int64_t)8 << 20);

static void choose_bins(esn_plan p) {
    const int dim = p->dim, w = p->kp.w;
    int bs[3] = {1, 1, 1};
    if (p->type == 2 && dim > 1) {
        // interpolation-only plan: bins sized for the shared-memory patch
        const size_t cb = p->dtype == ESN_F64 ? 16 : 8;
        if (dim == 2) {
            bs[0] = 32;
            bs[1] = 32;
            static const char *be = getenv("ESN_T2_BIN");  // "WxH": 2D interpolation bin (cells)
            if (be) {
                int bw = 0, bh = 0;
                if (sscanf(be, "%dx%d", &bw, &bh) == 2 && bw > 0 && bh > 0) {
                    bs[0] = bw;
                    bs[1] = bh;
                }
            }
        } else {
            bs[0] = 16;
            bs[1] = 8;
            bs[2] = 8;
        }
        auto patch = [&]() {
            size_t c = cb;
            for (int d = 0; d < dim; ++d) c *= (size_t)(bs[d] + w - 1);
            return c;
        };
        while (patch() > 96 * 1024) {
            int big = 0;
            for (int d = 1; d < dim; ++d)
                if (bs[d] > bs[big]) big = d;
            if (bs[big] <= 2) break;
            bs[big] /= 2;
        }
    } else if (!esn::spreader_bins(p->method, p->dtype, dim, w, p->ntransf, bs)) {
        // global-atomic spreader / 1D: bins only order the points for locality
        if (dim == 1) {
            bs[0] = 1024;
        } else if (dim == 2) {
            bs[0] = 32; bs[1] = 32;
        } else {
            bs[0] = 16; bs[1] = 8; bs[2] = 8;
        }
        for (int d = 0; d < 3; ++d)
            if (p->opts.bin_size[d] > 0) bs[d] = p->opts.bin_size[d];
    }
    p->nbins = 1;
    for (int d = 0; d < 3; ++d) {
        p->geom.bs[d] = d < dim ? bs[d] : 1;
        p->geom.n[d] = p->n[d];
        p->geom.nb[d] = d < dim ? (p->n[d] + bs[d] - 1) / bs[d] : 1;
        p->nbins *= p->geom.nb[d];
    }
    p->geom.dim = dim;
    p->geom.w = w;
    set_key_space(p, 1);
}

// fine sort key: sub-cells of 2^sbl cells inside each bin, coarsened
// (fastest dims first) until the key space (nchunk * nbins * sub-cells) is
// <= 8M entries
static void set_key_space(esn_plan p, int nchunk, int64_t maxkeys) {
    const int dim = p->dim;
    p->nchunk = nchunk;
    p->nbk = p->nbins * nchunk;
    for (int d = 0; d < 3; ++d) p->sbl[d] = 0;
    // sub-cells per bin along d: ceil(bs / 2^sbl)
    auto sub = [&](int d) { return ((p->geom.bs[d] - 1) >> p->sbl[d]) + 1; };
    auto keys = [&]() {
        int64_t k = p->nbk;
        for (int d = 0; d < dim; ++d) k *= sub(d);
        return k;
    };
    if (dim == 3 && p->type != 2 && p->method != ESN_METHOD_GLOBAL) {
        // 3D row spreader (k_spread_rows3): the key inside a bin is the x cell
        // of the footprint origin only, so contiguous chunks are x-ordered
        p->sbl[1] = p->sbl[2] = 30;
        p->spb = sub(0);
        p->nkeys = (int)keys();
        return;
    }
    for (int guard = 0; guard < 64 && keys() > maxkeys; ++guard) {
        bool grew = false;
        for (int d = 0; d < dim && keys() > maxkeys; ++d) {
            const int s2 = 1 << (p->sbl[d] + 1);
            if (p->geom.bs[d] % s2 == 0) {
                p->sbl[d]++;
                grew = true;
            }
        }
        if (!grew) break;
    }
    p->spb = 1;
    for (int d = 0; d < dim; ++d) p->spb *= sub(d);
    p->nkeys = (int)keys();
}

static int plan_common_init(esn_plan p, const esn_opts *o) {
    if (o)
        p->opts = *o;
    else
        esn_default_opts(&p->opts);
    p->dtype = p->opts.dtype == ESN_F32 ? ESN_F32 : ESN_F64;
    p->st = (cudaStream_t)p->opts.stream;
    p->coeffs.assign((size_t)p->kp.w * (p->kp.w + 4), 0.0);
    if (p->opts.coeffs) {
        std::memcpy(p->coeffs.data(), p->opts.coeffs, p->coeffs.size() * sizeof(double));
    } else {
        int rc = piecewise_poly(p->kp, p->coeffs.data(), nullptr);
        if (rc) return rc;
    }
    p->opts.params = nullptr;
    p->opts.coeffs = nullptr;
    p->G = 1;
    for (int d = 0; d < 3; ++d) p->G *= p->n[d];
    if (p->G * 1 > p->opts.max_grid_values)  // transforms.py:129-133
        return fail(ESN_RESOURCE_ERROR,
                    "fine grids need %lld complex values, over the cap of %lld; this regime is better "
                    "served by direct summation",
                    (long long)p->G, (long long)p->opts.max_grid_values);
    p->method = p->opts.method;
    if (p->method == ESN_METHOD_AUTO) p->method = (p->dim == 1) ? ESN_METHOD_GLOBAL : ESN_METHOD_TILE;
    choose_bins(p);
    p->maxsub = p->opts.max_subprob > 0 ? p->opts.max_subprob : 8192;
    int rc;
    if ((rc = ensure_key_space(p))) return rc;
    if ((rc = dmalloc(p, &p->nsub, sizeof(int) * 2))) return rc;
    if ((rc = dmalloc(p, &p->work, sizeof(int) * 2))) return rc;
    if ((rc = dmalloc(p, &p->flags, sizeof(unsigned long long) * 8))) return rc;
    if ((rc = dmalloc(p, &p->grid, real_size(p->dtype) * 2 * (size_t)p->G * p->ntransf))) return rc;
    ESN_CUDA_TRY(cudaMemsetAsync(p->flags, 0xff, sizeof(unsigned long long) * 8, p->st));
    // (ESN_B2_SWITCH=0: batched owner-computes plans never hand over to the RED-flush spreader)
    static const bool b2switch = [] {
        const char *e = getenv("ESN_B2_SWITCH");
        return !(e && e[0] == '0');
    }();
    if (b2switch && esn::batched_spread(p->dtype, p->dim, p->kp.w, p->ntransf, p->method)) {
        if ((rc = dmalloc(p, &p->imb, sizeof(int)))) return rc;
        ESN_CUDA_TRY(cudaMemsetAsync(p->imb, 0, sizeof(int), p->st));
    }
    if (p->opts.timing) {
        for (int i = 0; i < 8; ++i) ESN_CUDA_TRY(cudaEventCreate(&p->ev[i]));
        p->have_events = true;
    }
    return ESN_SUCCESS;
}

static int upload_corrections(esn_plan p) {
    for (int d = 0; d < p->dim; ++d) {
        std::vector<double> v((size_t)p->N[d]);
        int rc = fseries_correction(p->kp, p->n[d], p->N[d], v.data());
        if (rc) return rc;
        if ((rc = dmalloc(p, &p->pk[d], real_size(p->dtype) * v.size()))) return rc;
        if (p->dtype == ESN_F64) {
            ESN_CUDA_TRY(cudaMemcpy(p->pk[d], v.data(), v.size() * 8, cudaMemcpyHostToDevice));
        } else {
            std::vector<float> f(v.begin(), v.end());
            ESN_CUDA_TRY(cudaMemcpy(p->pk[d], f.data(), f.size() * 4, cudaMemcpyHostToDevice));
        }
    }
    return ESN_SUCCESS;
}

extern "C" {

int esn_version(void) { return ESN_VERSION; }
const char *esn_last_error(void) { return esn::last_error(); }

int esn_select_params(double tol, double sigma, esn_kernel_params *out) {
    if (!out) return fail(ESN_SIZE_ERROR, "null output");
    return select_params(tol, sigma, out);
}
int esn_params_for_width(int w, double sigma, esn_kernel_params *out) {
    if (!out) return fail(ESN_SIZE_ERROR, "null output");
    return params_for_width(w, sigma, out);
}
double esn_class_tolerance(int w, double sigma) { return class_tolerance(w, sigma); }
int esn_next_smooth(int64_t n, int64_t *out) {
    if (n < 1) return fail(ESN_SIZE_ERROR, "next_smooth needs n >= 1, got %lld", (long long)n);
    if (n > ((int64_t)1 << 60)) return fail(ESN_SIZE_ERROR, "next_smooth overflow for n=%lld", (long long)n);
    *out = next_smooth(n);
    return ESN_SUCCESS;
}
int esn_fine_grid_sizes(int dim, const int64_t *nmodes, double sigma, int w, int64_t *sizes) {
    for (int d = 0; d < dim; ++d) {
        if (nmodes[d] < 1) return fail(ESN_SIZE_ERROR, "mode counts must be >= 1");
        int64_t fl = std::max((int64_t)std::ceil(sigma * (double)nmodes[d]), (int64_t)(2 * w));
        sizes[d] = next_smooth(fl);
    }
    return ESN_SUCCESS;
}
int esn_gauss_legendre(int n, double *nodes, double *weights) {
    if (n < 1) return fail(ESN_SIZE_ERROR, "gauss_legendre needs n >= 1, got %d", n);
    gauss_legendre(n, nodes, weights);
    return ESN_SUCCESS;
}
int esn_kernel_ft(const esn_kernel_params *p, double alpha, int64_t nk, const double *k, double *out) {
    if (!(alpha > 0)) return fail(ESN_SIZE_ERROR, "alpha must be positive, got %g", alpha);
    kernel_ft(*p, alpha, nk, k, out);
    return ESN_SUCCESS;
}
int esn_fseries_correction(const esn_kernel_params *p, int64_t n, int64_t nmodes, double *out) {
    return fseries_correction(*p, n, nmodes, out);
}
int esn_piecewise_poly(const esn_kernel_params *p, double *coeffs, double *residual) {
    return piecewise_poly(*p, coeffs, residual);
}

void esn_default_opts(esn_opts *o) {
    std::memset(o, 0, sizeof(*o));
    o->sigma = 2.0;
    o->max_grid_values = (int64_t)1 << 31;  // transforms.py:41
    o->dtype = ESN_F64;
    o->method = ESN_METHOD_AUTO;
}

int esn_plan_destroy(esn_plan p) {
    if (!p) return ESN_SUCCESS;
    if (p->st2) cudaStreamSynchronize(p->st2);
    if (p->st) cudaStreamSynchronize(p->st);
    else cudaDeviceSynchronize();
    if (p->st2) {
        cudaEventDestroy(p->e_in);
        cudaEventDestroy(p->e_sorted);
        cudaStreamDestroy(p->st2);
    }
    if (p->aux.count_st) {
        cudaStreamSynchronize(p->aux.count_st);
        cudaEventDestroy(p->aux.counted);
        cudaStreamDestroy(p->aux.count_st);
    }
    if (p->aux.st) {
        cudaStreamSynchronize(p->aux.st);
        cudaEventDestroy(p->aux.fork);
        cudaEventDestroy(p->aux.join);
        cudaStreamDestroy(p->aux.st);
    }
    if (p->gs) {
        cudaStreamSynchronize(p->gs);
        for (auto &g : p->gexec)
            if (g) cudaGraphExecDestroy(g);
        cudaEventDestroy(p->g_in);
        cudaEventDestroy(p->g_out);
        cudaStreamDestroy(p->gs);
    }
    if (!p->borrowed) {
        for (int d = 0; d < 3; ++d) dfree(p->pk[d]);
        dfree(p->grid);
    }
    dfree(p->rec);
    dfree(p->pkey);
    dfree(p->twid);
    dfree(p->cperm);
    dfree(p->cursor);
    dfree(p->key_count);
    dfree(p->block_sums);
    dfree(p->bin_start);
    dfree(p->subofs);
    dfree(p->nsub);
    dfree(p->work);
    dfree(p->subprob);
    dfree(p->flags);
    dfree(p->imb);
    if (p->have_events)
        for (int i = 0; i < 8; ++i) cudaEventDestroy(p->ev[i]);
    if (p->fft_made) cufftDestroy(p->fft_h);
    delete p;
    return ESN_SUCCESS;
}

int esn_plan_create(int type, int dim, const int64_t *nmodes, int isign, int ntransf, double tol,
                    const esn_opts *opts, esn_plan *out) {
    if (!out) return fail(ESN_SIZE_ERROR, "null plan pointer");
    *out = nullptr;
    if (type != 1 && type != 2) return fail(ESN_SIZE_ERROR, "type must be 1 or 2, got %d", type);
    if (dim < 1 || dim > 3) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3, got %d", dim);
    if (isign != 1 && isign != -1) return fail(ESN_SIZE_ERROR, "isign must be +1 or -1, got %d", isign);
    if (ntransf < 1) return fail(ESN_SIZE_ERROR, "ntransf must be >= 1, got %d", ntransf);
    for (int d = 0; d < dim; ++d)
        if (nmodes[d] < 1) return fail(ESN_SIZE_ERROR, "mode counts must be >= 1");
    esn_opts o;
    if (opts) o = *opts; else esn_default_opts(&o);
    esn_plan p = new esn_plan_s();
    p->type = type;
    p->dim = dim;
    p->isign = isign;
    p->ntransf = ntransf;
    int rc;
    if (o.params) {
        p->kp = *o.params;
        if ((rc = params_for_width(p->kp.w, p->kp.sigma, &p->kp)) != ESN_SUCCESS) { delete p; return rc; }
        p->kp = *o.params;
    } else if ((rc = select_params(tol, o.sigma, &p->kp)) != ESN_SUCCESS) {
        delete p;
        return rc;
    }
    for (int d = 0; d < dim; ++d) {
        p->N[d] = nmodes[d];
        int64_t fl = std::max((int64_t)std::ceil(o.sigma * (double)nmodes[d]), (int64_t)(2 * p->kp.w));
        int64_t nn = next_smooth(fl);
        if (nn > INT_MAX) { delete p; return fail(ESN_RESOURCE_ERROR, "fine grid axis %lld too large", (long long)nn); }
        p->n[d] = (int)nn;
    }
    if ((rc = plan_common_init(p, &o)) || (rc = upload_corrections(p))) {
        esn_plan_destroy(p);
        return rc;
    }
    if (type == 1 && esn::colfft_eligible(p->dtype, dim, p->n[1])) {
        const int n2 = p->n[1];
        std::vector<double> tw((size_t)n2);  // n2 / 2 complex
        for (int k = 0; k < n2 / 2; ++k) {
            const double a = 2.0 * M_PI * k / n2;
            tw[2 * k] = std::cos(a);
            tw[2 * k + 1] = isign * std::sin(a);
        }
        const size_t rs = real_size(p->dtype);
        if ((rc = dmalloc(p, &p->twid, rs * n2))) {
            esn_plan_destroy(p);
            return rc;
        }
        cudaError_t e;
        if (p->dtype == ESN_F64) {
            e = cudaMemcpy(p->twid, tw.data(), sizeof(double) * n2, cudaMemcpyHostToDevice);
        } else {
            std::vector<float> twf(tw.begin(), tw.end());
            e = cudaMemcpy(p->twid, twf.data(), sizeof(float) * n2, cudaMemcpyHostToDevice);
        }
        if (e != cudaSuccess) {
            esn_plan_destroy(p);
            return fail(ESN_INTERNAL_ERROR, "twiddle upload failed");
        }
    }
    static const bool overlap = [] {
        const char *e = getenv("ESN_SORT_OVERLAP");
        return !(e && std::string(e) == "0");
    }();
    if (type == 2 && overlap) {
        // the sort is the critical path of a type-2 step (the amplify + FFT
        // beside it have slack): highest priority, so its small scan kernels
        // do not queue behind the FFT's CTAs (ESN_SORT_PRIO=0: the plan
        // stream's priority)
        int prio = 0;
        cudaStreamGetPriority(p->st, &prio);
        static const bool high = [] {
            const char *e = getenv("ESN_SORT_PRIO");
            return !(e && e[0] == '0');
        }();
        if (high) {
            int least = 0, greatest = 0;
            if (cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess) prio = greatest;
            else cudaGetLastError();
        }
        if (cudaStreamCreateWithPriority(&p->st2, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->e_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->e_sorted, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            esn_plan_destroy(p);
            return fail(ESN_INTERNAL_ERROR, "side stream creation failed");
        }
    }
    // the count pass of a side-stream sort at the PLAN stream's priority: it
    // is bound by L2 atomics, not by SM time, and at the sort's high priority
    // its resident CTAs starved the amplify + FFT beside it, whose tail then
    // ran after the scatter (ESN_SORT_COUNT_LO=0: count on the sort stream)
    static const bool countlo = [] {
        const char *e = getenv("ESN_SORT_COUNT_LO");
        return !(e && e[0] == '0');
    }();
    if (p->st2 && countlo) {
        int prio = 0;
        cudaStreamGetPriority(p->st, &prio);
        if (cudaStreamCreateWithPriority(&p->aux.count_st, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->aux.counted, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            esn_plan_destroy(p);
            return fail(ESN_INTERNAL_ERROR, "count stream creation failed");
        }
    }
    static const bool auxtab = [] {
        const char *e = getenv("ESN_SORT_AUX");
        return !(e && e[0] == '0');
    }();
    if (auxtab) {
        int least = 0, greatest = 0;
        if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) cudaGetLastError();
        if (cudaStreamCreateWithPriority(&p->aux.st, cudaStreamNonBlocking, greatest) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->aux.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->aux.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            esn_plan_destroy(p);
            return fail(ESN_INTERNAL_ERROR, "aux stream creation failed");
        }
    }
    *out = p;
    return ESN_SUCCESS;
}

// make the plan stream wait for an in-flight side-stream sort
static int join_sort(esn_plan p) {
    if (p->sort_pending) {
        ESN_CUDA_TRY(cudaStreamWaitEvent(p->st, p->e_sorted, 0));
        p->sort_pending = false;
    }
    return ESN_SUCCESS;
}

// Launch-bound problems (M <= ESN_GRAPH_MAX_M, default 2^19) replay each
// setpts / execute as one CUDA graph: ~15-20 launches and memsets per call
// otherwise cost more host time than the GPU work (c1: 62 us of kernels in
// a 112 us step).  The body enqueues on p->st; for a capture p->st is
// swapped for the private stream gs (captures cannot run on the legacy
// stream), and replays are ordered against the caller's stream by events.
static uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

static bool graph_eligible(esn_plan p) {
    static const int64_t lim = [] {
        const char *e = getenv("ESN_GRAPH_MAX_M");
        return e ? atoll(e) : (int64_t)1 << 19;
    }();
    return !p->graphs_off && !p->borrowed && p->M >= 0 && p->M <= lim;
}

extern "C++" {
template <class F>
static int run_graphed(esn_plan p, int slot, uint64_t sig, F &&body) {
    if (!p->gs) {
        if (cudaStreamCreateWithFlags(&p->gs, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->g_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->g_out, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            p->graphs_off = true;
            return body();
        }
    }
    sig = mix(mix(sig, (uint64_t)p->gen), (uint64_t)(uintptr_t)p->st);
    if (!p->gexec[slot] || p->gsig[slot] != sig) {
        if (p->gexec[slot]) {
            cudaGraphExecDestroy(p->gexec[slot]);
            p->gexec[slot] = nullptr;
        }
        const int64_t gen0 = p->gen;
        cudaStream_t user = p->st;
        // the capture stream starts after the caller's queued work, like a replay
        ESN_CUDA_TRY(cudaEventRecord(p->g_in, user));
        ESN_CUDA_TRY(cudaStreamWaitEvent(p->gs, p->g_in, 0));
        if (cudaStreamBeginCapture(p->gs, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
            cudaGetLastError();
            p->graphs_off = true;
            return body();
        }
        p->st = p->gs;
        p->capturing = true;
        const int rc = body();
        cudaGraph_t graph = nullptr;
        const cudaError_t e = cudaStreamEndCapture(p->gs, &graph);
        p->st = user;
        p->capturing = false;
        cudaGraphExec_t exec = nullptr;
        const bool ok = rc == ESN_SUCCESS && e == cudaSuccess && graph &&
                        cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {
            cudaGetLastError();
            if (rc != ESN_SUCCESS) return rc;  // (argument / resource errors surface as before)
            p->graphs_off = true;              // capture unsupported here: run directly
            return body();
        }
        p->gexec[slot] = exec;
        // allocations inside the body (first call) invalidate other slots' pointers
        p->gsig[slot] = p->gen == gen0 ? sig : 0;
        if (p->gen != gen0) p->gsig[1 - slot] = 0;
    }
    ESN_CUDA_TRY(cudaEventRecord(p->g_in, p->st));
    ESN_CUDA_TRY(cudaStreamWaitEvent(p->gs, p->g_in, 0));
    ESN_CUDA_TRY(cudaGraphLaunch(p->gexec[slot], p->gs));
    ESN_CUDA_TRY(cudaEventRecord(p->g_out, p->gs));
    ESN_CUDA_TRY(cudaStreamWaitEvent(p->st, p->g_out, 0));
    return ESN_SUCCESS;
}
}  // extern "C++"

int esn_spreader_create(int dim, const int64_t *nfine, int ntransf, const esn_opts *opts, esn_plan *out) {
    if (!out) return fail(ESN_SIZE_ERROR, "null plan pointer");
    *out = nullptr;
    if (dim < 1 || dim > 3) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3, got %d", dim);
    esn_opts o;
    if (opts) o = *opts; else esn_default_opts(&o);
    if (!o.params) return fail(ESN_SIZE_ERROR, "spreader plans need explicit kernel params");
    esn_plan p = new esn_plan_s();
    p->type = 0;
    p->dim = dim;
    p->ntransf = ntransf < 1 ? 1 : ntransf;
    p->kp = *o.params;
    int rc;
    esn_kernel_params chk;
    if ((rc = params_for_width(p->kp.w, p->kp.sigma, &chk))) { delete p; return rc; }
    for (int d = 0; d < dim; ++d) {
        if (nfine[d] < 1 || nfine[d] > INT_MAX) { delete p; return fail(ESN_SIZE_ERROR, "bad fine grid size"); }
        p->n[d] = (int)nfine[d];
    }
    if ((rc = plan_common_init(p, &o))) {
        esn_plan_destroy(p);
        return rc;
    }
    *out = p;
    return ESN_SUCCESS;
}

int esn_plan_setpts(esn_plan p, int64_t M, int coord_dtype, const void *x, const void *y, const void *z) {
    if (!p) return fail(ESN_SIZE_ERROR, "null plan");
    // an earlier side-stream sort may still be writing the records / key
    // arrays this call reallocates or rewrites (and a graphed setpts would
    // not wait for it): order the plan stream after it first
    if (int jr = join_sort(p)) return jr;
    if (M < 0 || M > INT_MAX) return fail(ESN_SIZE_ERROR, "point count %lld outside [0, 2^31)", (long long)M);
    const void *xs[3] = {x, y, z};
    for (int d = 0; d < p->dim; ++d)
        if (M > 0 && !xs[d]) return fail(ESN_SIZE_ERROR, "coordinate array %d missing", d + 1);
    int rc;
    const bool store_pos = esn::batched_spread(p->dtype, p->dim, p->kp.w, p->ntransf, p->method);
    if (M > p->Mcap) {
        dfree(p->rec);
        dfree(p->pkey);
        p->rec = nullptr;
        p->pkey = nullptr;
        if ((rc = dmalloc(p, &p->rec, sizeof(Rec) * M))) return rc;
        if (store_pos && (rc = dmalloc(p, &p->pkey, sizeof(int) * M))) return rc;
        p->Mcap = M;
    }
    if (p->type == 2) {
        // target chunks sized so one chunk's outputs (all transforms) stay
        // well inside L2 while it is being interpolated
        static const char *env = getenv("ESN_OUT_CHUNK_MB");
        static const double l2mb = [] {
            int dev = 0, l2 = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
            return l2 > 0 ? 0.75 * l2 / 1048576.0 : 64.0;
        }();
        const double mb = env ? atof(env) : l2mb;
        const double out_bytes = (double)M * real_size(p->dtype) * 2;
        int h = mb > 0 ? (int)std::ceil(out_bytes / (mb * 1048576.0)) : 1;
        h = std::max(1, std::min({h, 64, std::max(1, (8 << 20) / p->nbins)}));
        // the interpolator only needs bins; sub-cells beyond ~2 keys per
        // point cost key-space work (memset + scans) for nothing, and past
        // 4 Mi keys the finer order no longer pays for the larger scans
        // (c2 sweep with the overlapped sort: 8 Mi 0.872, 4 Mi 0.837,
        // 2 Mi 0.839, 1 Mi 0.842 ms/step)
        static const char *kenv = getenv("ESN_T2_KEYS");
        int64_t maxkeys = std::min<int64_t>((int64_t)4 << 20, std::max<int64_t>(2 * M, 1 << 16));
        if (kenv) maxkeys = std::max<int64_t>(1, atoll(kenv));
        if (h != p->nchunk || maxkeys != p->keycap_req) {
            set_key_space(p, h, maxkeys);
            p->keycap_req = maxkeys;
            if ((rc = ensure_key_space(p))) return rc;
        }
        p->chunk_len = h > 1 ? (M + h - 1) / h : 0;
    }
    const int64_t subneed = p->nbk + M / p->maxsub + 1;
    if (subneed > p->subcap) {
        dfree(p->subprob);
        p->subprob = nullptr;
        if ((rc = dmalloc(p, &p->subprob, sizeof(int4) * subneed))) return rc;
        p->subcap = subneed;
    }
    p->M = M;
    const bool graphed = graph_eligible(p);
    const bool side = p->st2 && !graphed;  // (small, graphed sorts stay on the plan stream)
    auto enqueue = [&]() -> int {
    int rc;
    // side stream: ordered after everything queued on the plan stream so far
    // (the previous execute may still read the records this sort rewrites)
    cudaStream_t ss = p->st;
    // hs: the stream of the sort's head (clears, count pass) -- the sort
    // stream itself, or the count stream, which the rest of the sort joins
    // through aux.counted (launch_setpts)
    cudaStream_t hs = ss;
    SetptsAux aux = p->aux;
    if (!(side && aux.st)) aux.count_st = nullptr;  // (the count stream rides on the aux block)
    if (side) {
        ss = p->st2;
        hs = aux.count_st ? aux.count_st : ss;
        // the count stream follows the previous sort (same plan, st2)
        if (aux.count_st) ESN_CUDA_TRY(cudaStreamWaitEvent(hs, p->e_sorted, 0));
        // the fill cursors are touched by the sort only: clear them before
        // joining the plan stream, i.e. beside the previous execute instead
        // of after it (c2: 16 MB, ~9 us off the step)
        ESN_CUDA_TRY(cudaMemsetAsync(p->key_count, 0, sizeof(int) * p->nkeys, hs));
        ESN_CUDA_TRY(cudaEventRecord(p->e_in, p->st));
        ESN_CUDA_TRY(cudaStreamWaitEvent(hs, p->e_in, 0));
        if (hs != ss) ESN_CUDA_TRY(cudaStreamWaitEvent(ss, p->e_in, 0));
    }
    if (p->have_events) ESN_CUDA_TRY(rec_ev(p, p->ev[0], hs));
    if (!side) ESN_CUDA_TRY(cudaMemsetAsync(p->key_count, 0, sizeof(int) * p->nkeys, ss));
    // point flags [0..5] only when overlapped: flag 6 (data) belongs to the
    // concurrent execute on the plan stream
    if (!p->keep_flags)
        ESN_CUDA_TRY(cudaMemsetAsync(p->flags, 0xff, sizeof(unsigned long long) * (side ? 6 : 8), hs));
    SetptsArgs a{};
    a.ibase = p->ibase;
    a.g = p->geom;
    a.M = M;
    a.coord_f32 = (coord_dtype & 0xf) == ESN_F32;
    a.grid_units = (coord_dtype & ESN_COORD_GRID_UNITS) != 0;
    for (int d = 0; d < 3; ++d) {
        a.x[d] = d < p->dim ? xs[d] : nullptr;
        a.scale[d] = (double)p->n[d] / (2.0 * M_PI);  // sizes[d] / TWO_PI (spreadinterp.py:99)
    }
    for (int d = 0; d < 3; ++d) {
        a.sbl[d] = p->sbl[d];
        a.inv_bs[d] = 1.0 / (double)p->geom.bs[d];
        const int b = p->geom.bs[d];
        a.bs_log2[d] = (b > 0 && (b & (b - 1)) == 0) ? __builtin_ctz((unsigned)b) : -1;
    }
    a.spb = p->spb;
    a.nkeys = p->nkeys;
    a.nbins_geo = p->nbins;
    a.chunk_len = p->chunk_len;
    a.inv_chunk = p->chunk_len > 0 ? 1.0 / (double)p->chunk_len : 0.0;
    a.key_count = p->key_count;
    a.block_sums = p->block_sums;
    a.bin_start = p->bin_start;
    a.cursor = p->cursor;
    a.key = p->pkey;
    a.store_pos = store_pos ? 1 : 0;
    a.rec = p->rec;
    a.flags = p->flags;
    a.check_bounds = p->opts.check_bounds;
    static const int hints = [] {
        const char *e = getenv("ESN_SCATTER_HINTS");
        return e && e[0] == '0' ? 0 : 1;
    }();
    a.hints = hints;
    static const int rev = [] {
        const char *e = getenv("ESN_SCATTER_REV");
        return e && e[0] == '0' ? 0 : 1;
    }();
    a.rev = rev;
    // small 1D type-1 plans spread point-parallel with global atomics: the
    // records need no order (ESN_SORT1D=1 forces the sort)
    static const bool sort1d = [] {
        const char *e = getenv("ESN_SORT1D");
        return e && e[0] == '1';
    }();
    const bool unsorted = p->type == 1 && p->dim == 1 && M <= ((int64_t)1 << 20) && !sort1d &&
                          p->method == ESN_METHOD_GLOBAL;
    if (unsorted) {
        if ((rc = launch_setpts_unsorted(a, ss))) return rc;
    } else if ((rc = launch_setpts(a, p->nbk, p->maxsub, p->subprob, p->nsub, p->subofs, ss,
                                   (p->aux.st && !graphed) ? &aux : nullptr))) {
        return rc;
    }
    // batched owner-computes plans: let the device decide whether the
    // points are too clustered for one warp per item (see esn_inst.cuh)
    if (p->imb && !unsorted && M > 0 &&
        esn::batched_owner(p->dtype, p->dim, p->kp.w, p->ntransf, p->method, p->sbl, p->geom.bs)) {
        if ((rc = esn::launch_bin_imbalance(p->bin_start, p->nbins, M, p->imb, ss))) return rc;
    }
    if (p->have_events) ESN_CUDA_TRY(rec_ev(p, p->ev[1], ss));
    if (side) ESN_CUDA_TRY(cudaEventRecord(p->e_sorted, p->st2));
    return ESN_SUCCESS;
    };
    if (graphed) {
        uint64_t sig = 0x5e7;
        for (uint64_t v : {(uint64_t)M, (uint64_t)coord_dtype, (uint64_t)(uintptr_t)x, (uint64_t)(uintptr_t)y,
                           (uint64_t)(uintptr_t)z, (uint64_t)p->keep_flags, (uint64_t)p->ibase,
                           (uint64_t)p->have_events, (uint64_t)p->nkeys, (uint64_t)p->nbk, (uint64_t)p->chunk_len,
                           (uint64_t)p->ntransf})
            sig = mix(sig, v);
        rc = run_graphed(p, 0, sig, enqueue);
    } else {
        rc = enqueue();
    }
    if (rc) return rc;
    p->sort_pending = side;
    p->points_set = true;
    return ESN_SUCCESS;
}

}  // extern "C"

template <typename T>
static SpreadArgs<T> make_spread_args(esn_plan p, const void *c, void *grid) {
    SpreadArgs<T> a{};
    a.g = p->geom;
    const int w = p->kp.w;
    for (int i = 0; i < w * (w + 4); ++i) a.k.coef[i] = (T)p->coeffs[i];
    a.k.beta = (T)p->kp.beta;
    a.k.use_exact = p->opts.use_exact_kernel;
    a.M = p->M;
    a.ntransf = p->ntransf;
    a.rec = p->rec;
    a.bin_start = p->bin_start;
    a.subprob = p->subprob;
    a.kstart = p->cursor;
    a.spb = p->spb;
    for (int d = 0; d < 3; ++d) a.sbl[d] = p->sbl[d];
    a.nsub = p->nsub;
    a.subofs = p->type == 2 ? nullptr : p->subofs;
    // z-rolling pays where bins hold a few hundred points (c3: ~490; its
    // host-pipeline chunks ~100); c3f's ~2000-point bins gain nothing from it
    static const int roll_env = [] {
        const char *e = getenv("ESN_ROLL3");
        return e ? atoi(e) : -1;
    }();
    a.roll = roll_env >= 0 ? roll_env : (p->nbins > 0 && p->M <= (int64_t)512 * p->nbins);
    a.work = p->work;
    a.c = (const T *)c;
    a.grid = (T *)grid;
    a.gstride = p->G;
    a.ibase = p->ibase;
    a.flags = p->flags;
    // (only plans on the owner-computes path switch; elsewhere the RED-flush kernel always runs)
    a.imb = (p->imb && p->type == 1 &&
             esn::batched_owner(p->dtype, p->dim, p->kp.w, p->ntransf, p->method, p->sbl, p->geom.bs))
                ? p->imb
                : nullptr;
    return a;
}

bool esn::batched_spread(int dtype, int dim, int w, int ntransf, int method) {
    return method != ESN_METHOD_GLOBAL && dim == 2 && dtype == ESN_F32 && ntransf > 1 && w <= 10;
}

// ESN_B2=own: the per-item owner-computes kernel (k_spread_b2own) instead of
// the y-rolling one (k_spread_b2roll)
bool esn::batched_roll_off() {
    static const bool off = [] {
        const char *e = getenv("ESN_B2");
        return e && std::string(e) == "own";
    }();
    return off;
}

bool esn::batched_owner(int dtype, int dim, int w, int ntransf, int method, const int *sbl, const int *bs) {
    static const bool off = [] {
        const char *e = getenv("ESN_B2");
        return e && std::string(e) == "tile";
    }();
    return !off && batched_spread(dtype, dim, w, ntransf, method) && sbl[0] == 0 && sbl[1] == 0 &&
           bs[0] == Batch2Cfg<float, 2>::BX && bs[1] == Batch2Cfg<float, 2>::BY;
}

// scratch of the batched spreader: permuted strengths + per-point rows
// table (<= 96 B per point)
static int ensure_spread_scratch(esn_plan p, int method) {
    if (esn::batched_spread(p->dtype, p->dim, p->kp.w, p->ntransf, method)) {
        const int64_t need = (int64_t)((p->ntransf + 31) / 32) * 32 * p->M * (int64_t)real_size(p->dtype) * 2 +
                             96 * p->M + 256;
        if (need > p->cperm_bytes) {
            dfree(p->cperm);
            p->cperm = nullptr;
            int rc = dmalloc(p, &p->cperm, (size_t)need);
            if (rc) return rc;
            p->cperm_bytes = need;
        }
    }
    return ESN_SUCCESS;
}

static int do_spread(esn_plan p, const void *c, void *grid, bool zero = true) {
    if (int jr = join_sort(p)) return jr;
    // the bin-structured spreaders need their own bin geometry and the
    // geometric sort; a type-2 plan (interpolation bins, possibly a
    // target-chunked order) spreads its adjoint with the order-agnostic
    // spreader
    const int method = p->type == 2 ? ESN_METHOD_GLOBAL : p->method;
    if (int rc = ensure_spread_scratch(p, method)) return rc;
    // the owner-computes batched spreader writes every fine cell itself
    const bool owner = esn::batched_owner(p->dtype, p->dim, p->kp.w, p->ntransf, method, p->sbl, p->geom.bs);
    if (zero && !owner)
        ESN_CUDA_TRY(cudaMemsetAsync(grid, 0, real_size(p->dtype) * 2 * (size_t)p->G * p->ntransf, p->st));
    ESN_CUDA_TRY(cudaMemsetAsync(p->work, 0, sizeof(int) * 2, p->st));  // (two work queues)
    if (p->have_events) ESN_CUDA_TRY(rec_ev(p, p->ev[6], p->st));
    int rc;
    if (p->dtype == ESN_F64) {
        SpreadArgs<double> a = make_spread_args<double>(p, c, grid);
        a.accumulate = zero ? 0 : 1;
        rc = launch_spread<double>(a, method, p->nbins, p->pkey, p->cursor, (double *)p->cperm, p->st);
    } else {
        SpreadArgs<float> a = make_spread_args<float>(p, c, grid);
        a.accumulate = zero ? 0 : 1;
        rc = launch_spread<float>(a, method, p->nbins, p->pkey, p->cursor, (float *)p->cperm, p->st);
    }
    if (!rc && p->have_events) ESN_CUDA_TRY(rec_ev(p, p->ev[7], p->st));
    return rc;
}

static int do_interp(esn_plan p, const void *grid, void *c) {
    if (int jr = join_sort(p)) return jr;
    ESN_CUDA_TRY(cudaMemsetAsync(p->work, 0, sizeof(int), p->st));
    if (p->have_events) ESN_CUDA_TRY(rec_ev(p, p->ev[6], p->st));
    int rc = p->dtype == ESN_F64
                 ? launch_interp<double>(make_spread_args<double>(p, nullptr, nullptr), (double *)c,
                                         (const double *)grid, p->st)
                 : launch_interp<float>(make_spread_args<float>(p, nullptr, nullptr), (float *)c,
                                        (const float *)grid, p->st);
    if (!rc && p->have_events) ESN_CUDA_TRY(rec_ev(p, p->ev[7], p->st));
    return rc;
}

extern "C" {

int esn_plan_spread(esn_plan p, const void *c, void *grid) {
    if (!p || !p->points_set) return fail(ESN_SIZE_ERROR, "plan has no points (call esn_plan_setpts first)");
    ESN_CUDA_TRY(cudaMemsetAsync(p->flags + 6, 0xff, sizeof(unsigned long long), p->st));
    return do_spread(p, c, grid);
}

// type-1 tail: fine-grid FFT + deconvolution into the modes.  2D plans with
// a power-of-two n2 run cuFFT along x only and the fused pruned y-FFT +
// deconvolution kernel; others cuFFT (full) + k_deconv*.  `ev_mid` (may be
// null) is recorded between the two halves.
static int fft_deconv_type1(esn_plan p, void *grid, void *f, cudaStream_t st, cudaEvent_t ev_mid) {
    int rc;
    if (p->twid) {
        const int n1 = p->n[0];
        if ((rc = plan_fft(p, grid, st))) return rc;
        if (ev_mid) ESN_CUDA_TRY(rec_ev(p, ev_mid, st));
        if (p->dtype == ESN_F64)
            return launch_colfft_deconv<double>(p->ntransf, p->n[0], p->n[1], (int)p->N[0], (int)p->N[1],
                                                (const double *)grid, (const double *)p->twid,
                                                (const double *)p->pk[0], (const double *)p->pk[1], (double *)f, st);
        return launch_colfft_deconv<float>(p->ntransf, p->n[0], p->n[1], (int)p->N[0], (int)p->N[1],
                                           (const float *)grid, (const float *)p->twid, (const float *)p->pk[0],
                                           (const float *)p->pk[1], (float *)f, st);
    }
    if ((rc = plan_fft(p, grid, st))) return rc;
    if (ev_mid) ESN_CUDA_TRY(rec_ev(p, ev_mid, st));
    if (p->dtype == ESN_F64)
        return launch_deconv<double>(p->dim, p->ntransf, p->n, p->N, (const double *)grid, (const double *)p->pk[0],
                                     (const double *)p->pk[1], (const double *)p->pk[2], (double *)f, st);
    return launch_deconv<float>(p->dim, p->ntransf, p->n, p->N, (const float *)grid, (const float *)p->pk[0],
                                (const float *)p->pk[1], (const float *)p->pk[2], (float *)f, st);
}


int esn_plan_finish_type1(esn_plan p, void *grid, void *f) {
    if (!p || p->type != 1) return fail(ESN_SIZE_ERROR, "finish_type1 needs a type-1 plan");
    if (!grid || !f) return fail(ESN_SIZE_ERROR, "null grid or mode array");
    return fft_deconv_type1(p, grid, f, p->st, nullptr);
}

int esn_plan_spread_add(esn_plan p, const void *c, void *grid) {
    if (!p || !p->points_set) return fail(ESN_SIZE_ERROR, "plan has no points (call esn_plan_setpts first)");
    if (!grid) return fail(ESN_SIZE_ERROR, "null grid");
    const int method = p->type == 2 ? ESN_METHOD_GLOBAL : p->method;
    if (esn::batched_owner(p->dtype, p->dim, p->kp.w, p->ntransf, method, p->sbl, p->geom.bs))
        return fail(ESN_SIZE_ERROR, "spread_add: the batched owner-computes spreader stores without atomics");
    ESN_CUDA_TRY(cudaMemsetAsync(p->flags + 6, 0xff, sizeof(unsigned long long), p->st));
    return do_spread(p, c, grid, false);
}

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "the ABI carries 64-byte handles");

int esn_peer_alloc(int64_t bytes, void **ptr, unsigned char handle[64]) {
    if (!ptr || !handle || bytes <= 0) return fail(ESN_SIZE_ERROR, "peer_alloc: bad arguments");
    void *d = nullptr;
    cudaError_t e = cudaMalloc(&d, (size_t)bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ESN_RESOURCE_ERROR, "peer allocation of %lld bytes failed (%s)", (long long)bytes,
                    cudaGetErrorString(e));
    }
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, d);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d);
        return fail(ESN_RESOURCE_ERROR, "cudaIpcGetMemHandle failed (%s)", cudaGetErrorString(e));
    }
    std::memcpy(handle, &h, 64);
    *ptr = d;
    return ESN_SUCCESS;
}

int esn_peer_open(const unsigned char handle[64], void **ptr) {
    if (!ptr || !handle) return fail(ESN_SIZE_ERROR, "peer_open: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void *d = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ESN_RESOURCE_ERROR, "cudaIpcOpenMemHandle failed (%s)", cudaGetErrorString(e));
    }
    *ptr = d;
    return ESN_SUCCESS;
}

int esn_peer_close(void *ptr) {
    if (!ptr) return ESN_SUCCESS;
    ESN_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return ESN_SUCCESS;
}

int esn_peer_free(void *ptr) {
    if (!ptr) return ESN_SUCCESS;
    ESN_CUDA_TRY(cudaFree(ptr));
    return ESN_SUCCESS;
}

int esn_plan_interp(esn_plan p, const void *grid, void *c) {
    if (!p || !p->points_set) return fail(ESN_SIZE_ERROR, "plan has no points (call esn_plan_setpts first)");
    return do_interp(p, grid, c);
}

static int execute_body(esn_plan p, void *c, void *f);

int esn_plan_execute(esn_plan p, void *c, void *f) {
    if (!p || !p->points_set) return fail(ESN_SIZE_ERROR, "plan has no points (call esn_plan_setpts first)");
    if (p->type != 1 && p->type != 2) return fail(ESN_SIZE_ERROR, "spreader plans have no execute");
    if (!graph_eligible(p)) return execute_body(p, c, f);
    // everything that allocates happens before a capture
    int rc;
    if ((rc = ensure_spread_scratch(p, p->type == 2 ? ESN_METHOD_GLOBAL : p->method))) return rc;
    if ((rc = ensure_fft_plan(p))) return rc;
    uint64_t sig = 0xe8ec;
    for (uint64_t v : {(uint64_t)(uintptr_t)c, (uint64_t)(uintptr_t)f, (uint64_t)p->M, (uint64_t)p->have_events,
                       (uint64_t)p->ntransf, (uint64_t)p->keep_flags})
        sig = mix(sig, v);
    return run_graphed(p, 1, sig, [&]() { return execute_body(p, c, f); });
}

static int execute_body(esn_plan p, void *c, void *f) {
    int rc;
    const bool ev = p->have_events;
    // (keep_flags: a caller accumulating the data flag over several executes)
    if (!p->keep_flags) ESN_CUDA_TRY(cudaMemsetAsync(p->flags + 6, 0xff, sizeof(unsigned long long), p->st));
    if (p->type == 1) {
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[2], p->st));
        if ((rc = do_spread(p, c, p->grid))) return rc;
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[3], p->st));
        if ((rc = fft_deconv_type1(p, p->grid, f, p->st, ev ? p->ev[4] : nullptr))) return rc;
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[5], p->st));
    } else {
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[2], p->st));
        if (p->dtype == ESN_F64)
            rc = launch_amplify<double>(p->dim, p->ntransf, p->n, p->N, (const double *)f, (const double *)p->pk[0],
                                        (const double *)p->pk[1], (const double *)p->pk[2], (double *)p->grid,
                                        p->flags + 6, p->st);
        else
            rc = launch_amplify<float>(p->dim, p->ntransf, p->n, p->N, (const float *)f, (const float *)p->pk[0],
                                       (const float *)p->pk[1], (const float *)p->pk[2], (float *)p->grid,
                                       p->flags + 6, p->st);
        if (rc) return rc;
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[3], p->st));
        if ((rc = plan_fft(p, p->grid, p->st))) return rc;
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[4], p->st));
        if ((rc = do_interp(p, p->grid, c))) return rc;
        if (ev) ESN_CUDA_TRY(rec_ev(p, p->ev[5], p->st));
    }
    return ESN_SUCCESS;
}

int esn_plan_check(esn_plan p, int64_t *info) {
    if (!p) return fail(ESN_SIZE_ERROR, "null plan");
    if (int jr = join_sort(p)) return jr;
    ESN_CUDA_TRY(cudaStreamSynchronize(p->st));
    unsigned long long h[8];
    ESN_CUDA_TRY(cudaMemcpy(h, p->flags, sizeof(h), cudaMemcpyDeviceToHost));
    const unsigned long long none = ~0ull;
    int64_t dummy[2];
    if (!info) info = dummy;
    info[0] = -1;
    info[1] = -1;
    auto strength = [&]() -> int {
        if (h[6] != none) {
            info[0] = (int64_t)h[6];
            info[1] = 0;
            return fail(ESN_DATA_ERROR, "non-finite %s at index %lld", p->type == 2 ? "mode coefficient" : "strength",
                        (long long)h[6]);
        }
        return ESN_SUCCESS;
    };
    if (p->type == 2) {
        int rc = strength();
        if (rc) return rc;
    }
    for (int d = 0; d < p->dim; ++d) {
        if (h[d] != none) {
            info[0] = (int64_t)h[d];
            info[1] = d + 1;
            return fail(ESN_DATA_ERROR, "non-finite coordinate at index %lld in dimension %d", (long long)h[d], d + 1);
        }
        if (p->opts.check_bounds && h[3 + d] != none) {
            info[0] = (int64_t)h[3 + d];
            info[1] = d + 1;
            return fail(ESN_BOUNDS_VIOLATION, "coordinate at index %lld outside [-3 pi, 3 pi]", (long long)h[3 + d]);
        }
    }
    if (p->type != 2) return strength();
    return ESN_SUCCESS;
}

int esn_plan_stage_times(esn_plan p, double *sort_s, double *spread_s, double *fft_s, double *correct_s) {
    if (!p || !p->have_events) return fail(ESN_SIZE_ERROR, "plan was created without opts.timing");
    if (int jr = join_sort(p)) return jr;
    ESN_CUDA_TRY(cudaStreamSynchronize(p->st));
    float ms[4] = {0, 0, 0, 0};
    if (p->points_set) cudaEventElapsedTime(&ms[0], p->ev[0], p->ev[1]);
    cudaEventElapsedTime(&ms[1], p->ev[2], p->ev[3]);
    cudaEventElapsedTime(&ms[2], p->ev[3], p->ev[4]);
    cudaEventElapsedTime(&ms[3], p->ev[4], p->ev[5]);
    cudaGetLastError();
    // stage keys follow transforms.py:83-85; for type 2 the first timed
    // segment is the amplify ("correct") and the last the interp ("spread").
    double s = ms[0] * 1e-3, a = ms[1] * 1e-3, b = ms[2] * 1e-3, c = ms[3] * 1e-3;
    if (sort_s) *sort_s = s;
    if (p->type == 2) {
        if (spread_s) *spread_s = c;
        if (correct_s) *correct_s = a;
    } else {
        if (spread_s) *spread_s = a;
        if (correct_s) *correct_s = c;
    }
    if (fft_s) *fft_s = b;
    return ESN_SUCCESS;
}

int esn_plan_hot_kernel_seconds(esn_plan p, double *seconds) {
    if (!p || !p->have_events) return fail(ESN_SIZE_ERROR, "plan was created without opts.timing");
    if (int jr = join_sort(p)) return jr;
    ESN_CUDA_TRY(cudaStreamSynchronize(p->st));
    float ms = 0.f;
    ESN_CUDA_TRY(cudaEventElapsedTime(&ms, p->ev[6], p->ev[7]));
    *seconds = ms * 1e-3;
    return ESN_SUCCESS;
}

int esn_plan_info(esn_plan p, int64_t *nfine, esn_kernel_params *kp) {
    if (!p) return fail(ESN_SIZE_ERROR, "null plan");
    if (nfine)
        for (int d = 0; d < 3; ++d) nfine[d] = p->n[d];
    if (kp) *kp = p->kp;
    return ESN_SUCCESS;
}

int esn_plan_bins(esn_plan p, int *nbins, int *bin_size, int *bins_per_dim) {
    if (!p) return fail(ESN_SIZE_ERROR, "null plan");
    if (nbins) *nbins = p->nbins;
    for (int d = 0; d < 3; ++d) {
        if (bin_size) bin_size[d] = p->geom.bs[d];
        if (bins_per_dim) bins_per_dim[d] = p->geom.nb[d];
    }
    return ESN_SUCCESS;
}

// spreadinterp.py:165-184 (_run_tasks stats): the work items of the last
// sort -- subproblems, the spread / interp kernels' unit of dynamic
// scheduling -- read back after the plan stream drains
int esn_plan_tasks(esn_plan p, int64_t *ntasks) {
    if (!p || !p->points_set) return fail(ESN_SIZE_ERROR, "plan has no points");
    if (int jr = join_sort(p)) return jr;
    int v = 0;
    if (p->nsub) {
        ESN_CUDA_TRY(cudaMemcpyAsync(&v, p->nsub, sizeof(int), cudaMemcpyDeviceToHost, p->st));
        ESN_CUDA_TRY(cudaStreamSynchronize(p->st));
    }
    if (ntasks) *ntasks = v;
    return ESN_SUCCESS;
}

int esn_plan_sort_view(esn_plan p, void *perm, void *keys, void *bin_start) {
    if (!p || !p->points_set) return fail(ESN_SIZE_ERROR, "plan has no points");
    if (p->nchunk > 1) return fail(ESN_SIZE_ERROR, "sort view needs a spreader plan (this plan's order is target-chunked)");
    if (int jr = join_sort(p)) return jr;
    int rc = launch_sort_view(p->dtype, p->rec, p->bin_start, p->nbins, p->M, (int *)perm, (int *)keys, p->st);
    if (rc) return rc;
    if (bin_start)
        ESN_CUDA_TRY(cudaMemcpyAsync(bin_start, p->bin_start, sizeof(int) * (p->nbins + 1),
                                     cudaMemcpyDeviceToDevice, p->st));
    return ESN_SUCCESS;
}

int esn_plan_target_chunks(esn_plan p, int *nchunk) {
    if (!p) return fail(ESN_SIZE_ERROR, "null plan");
    if (nchunk) *nchunk = p->nchunk;
    return ESN_SUCCESS;
}

int64_t esn_plan_device_bytes(esn_plan p) { return p ? p->device_bytes : 0; }

// Explicit cuFFT plans (fft.py:79-111 _build_plan / get_plan / clear_plan_cache):
// one handle and work area per plan; executions of one plan are serialised
// by its mutex (SetStream + Exec), so callers that run one plan from two
// streams at once must use two plans.
struct esn_fft_plan_s {
    int dim = 1, dtype = ESN_F64, batch = 1, device = 0;
    int n[3] = {1, 1, 1};
    cufftHandle h = 0;
    size_t work = 0;
    std::mutex mu;
};

int esn_fft_plan_create(int dim, int dtype, int ntransf, const int64_t *nfine, esn_fft_plan *out) {
    if (!out) return fail(ESN_SIZE_ERROR, "null plan pointer");
    *out = nullptr;
    if (dim < 1 || dim > 3) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
    auto *p = new (std::nothrow) esn_fft_plan_s;
    if (!p) return fail(ESN_RESOURCE_ERROR, "out of host memory");
    p->dim = dim;
    p->dtype = dtype == ESN_F32 ? ESN_F32 : ESN_F64;
    p->batch = ntransf < 1 ? 1 : ntransf;
    cudaGetDevice(&p->device);
    for (int d = 0; d < dim; ++d) {
        if (nfine[d] < 1 || nfine[d] > INT_MAX) {
            delete p;
            return fail(ESN_SIZE_ERROR, "invalid transform shape");
        }
        p->n[d] = (int)nfine[d];
    }
    if (int rc = make_fft_plan(dim, p->n, p->dtype, p->batch, &p->h)) {
        delete p;
        return rc;
    }
    cufftGetSize(p->h, &p->work);
    *out = p;
    return ESN_SUCCESS;
}

int esn_fft_plan_exec(esn_fft_plan p, void *data, int sign, void *stream) {
    if (!p) return fail(ESN_SIZE_ERROR, "null plan");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != p->device) return fail(ESN_SIZE_ERROR, "FFT plan made on device %d, current device %d", p->device, dev);
    std::lock_guard<std::mutex> lk(p->mu);
    return exec_fft(p->h, p->dtype, data, sign, (cudaStream_t)stream);
}

int64_t esn_fft_plan_work_bytes(esn_fft_plan p) { return p ? (int64_t)p->work : 0; }

int esn_fft_plan_destroy(esn_fft_plan p) {
    if (!p) return ESN_SUCCESS;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        if (p->h) cufftDestroy(p->h);
    }
    delete p;
    return ESN_SUCCESS;
}

// drops the plan-less esn_fft handles (fft.py:101-106 clear_plan_cache(None))
int esn_fft_cache_clear(void) {
    std::lock_guard<std::mutex> lk(g_fft_mu);
    for (auto &kv : g_fft_cache) cufftDestroy(kv.second);
    g_fft_cache.clear();
    return ESN_SUCCESS;
}

int esn_fft(int dim, int dtype, int ntransf, const int64_t *nfine, void *data, int sign, void *stream) {
    if (dim < 1 || dim > 3) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
    int n[3] = {1, 1, 1};
    for (int d = 0; d < dim; ++d) {
        if (nfine[d] < 1 || nfine[d] > INT_MAX) return fail(ESN_SIZE_ERROR, "invalid transform shape");
        n[d] = (int)nfine[d];
    }
    return run_fft_cached(dim, n, dtype == ESN_F32 ? ESN_F32 : ESN_F64, ntransf < 1 ? 1 : ntransf, data, sign,
                          (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Host-buffer one-shot routines (esnufftpy analog).  A small cache keeps the
// plan, two pipeline helper plans and device staging buffers for repeated
// calls of the same shape.  With pinned host buffers and enough points the
// transfer is pipelined: points are processed in chunks on two streams so
// host->device copies of chunk i+1, the kernels of chunk i and the
// device->host copy of chunk i-1 overlap (PCIe is full duplex); the fine
// grid is shared (type 1: chunks spread into it; type 2: chunks interpolate
// from it once amplify + FFT are done).

// A plan that shares `main`'s kernel tables, corrections and fine grid but
// owns its own point scratch and stream.
static int clone_point_plan(esn_plan main, cudaStream_t st, esn_plan *out) {
    esn_plan p = new esn_plan_s();
    p->type = main->type;
    p->dim = main->dim;
    p->dtype = main->dtype;
    p->isign = main->isign;
    p->ntransf = main->ntransf;
    for (int d = 0; d < 3; ++d) {
        p->N[d] = main->N[d];
        p->n[d] = main->n[d];
        p->pk[d] = main->pk[d];
        p->sbl[d] = main->sbl[d];
    }
    p->kp = main->kp;
    p->coeffs = main->coeffs;
    p->opts = main->opts;
    p->opts.timing = 0;
    p->opts.stream = st;
    p->st = st;
    p->geom = main->geom;
    p->nbins = main->nbins;
    p->maxsub = main->maxsub;
    p->method = main->method;
    p->G = main->G;
    p->spb = main->spb;
    p->nkeys = main->nkeys;
    p->grid = main->grid;
    p->borrowed = true;
    int rc;
    p->nchunk = main->nchunk;
    p->nbk = main->nbk;
    if ((rc = ensure_key_space(p)) || (rc = dmalloc(p, &p->nsub, sizeof(int) * 2)) ||
        (rc = dmalloc(p, &p->work, sizeof(int) * 2)) ||
        (rc = dmalloc(p, &p->flags, sizeof(unsigned long long) * 8))) {
        esn_plan_destroy(p);
        return rc;
    }
    *out = p;
    return ESN_SUCCESS;
}

namespace {
struct HostSlot {
    int type, dim, isign, ntransf, dtype;
    int device;  // the slot's plan, streams and buffers live on this device
    int64_t N[3];
    double tol, sigma;
    int method;
    esn_plan plan = nullptr;
    static constexpr int NH = 8;  // pipeline helpers / streams (capacity)
    esn_plan helper[NH] = {};
    cudaStream_t hst[NH] = {};
    cudaEvent_t ev_grid = nullptr, ev_done[NH] = {};
    // transfer streams: every H2D goes through `up` (back to back, in chunk
    // order), every D2H through `down`; per-chunk events link them to the
    // compute streams so neither copy engine waits behind kernels
    static constexpr int KC = 64;  // chunk capacity
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t ev_in = nullptr, ev_up[KC] = {}, ev_comp[KC] = {}, ev_down = nullptr;
    void *dx[3] = {nullptr, nullptr, nullptr};
    void *dc = nullptr, *df = nullptr;
    int64_t Mcap = 0;
    cudaStream_t st = nullptr;
};
std::mutex g_host_mu;
std::vector<HostSlot> g_slots;

void free_slot(HostSlot &s) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != s.device) cudaSetDevice(s.device);
    for (int h = 0; h < HostSlot::NH; ++h) {
        if (s.helper[h]) esn_plan_destroy(s.helper[h]);
        if (s.hst[h]) cudaStreamDestroy(s.hst[h]);
        if (s.ev_done[h]) cudaEventDestroy(s.ev_done[h]);
    }
    if (s.ev_grid) cudaEventDestroy(s.ev_grid);
    for (int k = 0; k < HostSlot::KC; ++k) {
        if (s.ev_up[k]) cudaEventDestroy(s.ev_up[k]);
        if (s.ev_comp[k]) cudaEventDestroy(s.ev_comp[k]);
    }
    if (s.ev_in) cudaEventDestroy(s.ev_in);
    if (s.ev_down) cudaEventDestroy(s.ev_down);
    if (s.up) cudaStreamDestroy(s.up);
    if (s.down) cudaStreamDestroy(s.down);
    if (s.plan) esn_plan_destroy(s.plan);
    for (int d = 0; d < 3; ++d) dfree(s.dx[d]);
    dfree(s.dc);
    dfree(s.df);
    if (s.st) cudaStreamDestroy(s.st);
    if (cur != s.device) cudaSetDevice(cur);
}

bool is_pinned(const void *ptr) {
    if (!ptr) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
}  // namespace

// strided (ntransf rows) H2D / D2H of point range [lo, hi) of a (T, M) array
static int copy_rows(void *dst, const void *src, int64_t M_dst, int64_t M_src, int64_t lo_dst, int64_t lo_src,
                     int64_t cnt, int T, size_t cb, cudaMemcpyKind kind, cudaStream_t st) {
    if (cnt <= 0) return ESN_SUCCESS;
    if (T == 1) {
        if (cudaMemcpyAsync((char *)dst + lo_dst * cb, (const char *)src + lo_src * cb, cnt * cb, kind, st) !=
            cudaSuccess)
            return fail(ESN_INTERNAL_ERROR, "copy failed (%s)", cudaGetErrorString(cudaGetLastError()));
        return ESN_SUCCESS;
    }
    if (cudaMemcpy2DAsync((char *)dst + lo_dst * cb, M_dst * cb, (const char *)src + lo_src * cb, M_src * cb,
                          cnt * cb, T, kind, st) != cudaSuccess)
        return fail(ESN_INTERNAL_ERROR, "strided copy failed (%s)", cudaGetErrorString(cudaGetLastError()));
    return ESN_SUCCESS;
}

static int pipelined(HostSlot *slot, int type, int dim, int64_t M, const double *const *xs, int T, void *c, void *f,
                     int64_t nm, size_t cb, bool c64in, int cdt) {
    const size_t xsz = cdt == ESN_F32 ? 4 : 8;  // coordinate element size (esn_opts.coord_dtype)
    const auto t_start = std::chrono::steady_clock::now();
    esn_plan p = slot->plan;
    int rc;
    static const int NH = [] {  // helpers / compute streams in use
        const char *e = getenv("ESN_PIPE_STREAMS");
        const int v = e ? atoi(e) : 4;
        return std::max(1, std::min(v, HostSlot::NH));
    }();
    static const int KMAX = [] {
        const char *e = getenv("ESN_PIPE_CHUNKS");
        return std::max(1, std::min(e ? atoi(e) : 12, HostSlot::KC));
    }();
    for (int h = 0; h < NH; ++h) {
        if (!slot->hst[h]) {
            ESN_CUDA_TRY(cudaStreamCreateWithFlags(&slot->hst[h], cudaStreamNonBlocking));
            ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_done[h], cudaEventDisableTiming));
        }
        if (!slot->helper[h] && (rc = clone_point_plan(p, slot->hst[h], &slot->helper[h]))) return rc;
    }
    if (!slot->up) {
        ESN_CUDA_TRY(cudaStreamCreateWithFlags(&slot->up, cudaStreamNonBlocking));
        ESN_CUDA_TRY(cudaStreamCreateWithFlags(&slot->down, cudaStreamNonBlocking));
        ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_grid, cudaEventDisableTiming));
        ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_in, cudaEventDisableTiming));
        ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_down, cudaEventDisableTiming));
        for (int k = 0; k < HostSlot::KC; ++k) {
            ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_up[k], cudaEventDisableTiming));
            ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_comp[k], cudaEventDisableTiming));
        }
    }
    cudaStream_t st = p->st, up = slot->up, down = slot->down;
    static const bool trace = getenv("ESN_TRACE") != nullptr;
    static cudaEvent_t tev[4][HostSlot::KC + 1];  // start, up, comp, down
    static bool tev_init = false;
    if (trace && !tev_init) {
        for (auto &row : tev)
            for (auto &e : row) cudaEventCreate(&e);
        tev_init = true;
    }
    if (trace) cudaEventRecord(tev[0][0], st);
    // type 1: every chunk's spread pays a full halo flush of every bin it
    // touches, so few large chunks win (3D 1e7 points: K = 12 11.6 ms, K = 6
    // 9.64, K = 5 9.60, K = 4 9.76 ms; c4: K = 5 10.1 ms, K = 4 11.1 ms;
    // c5 flat at 13.7 ms)
    static const int KMAX1 = [] {
        const char *e = getenv("ESN_PIPE_CHUNKS");
        return std::max(1, std::min(e ? atoi(e) : 5, HostSlot::KC));
    }();
    const int K = (int)std::min<int64_t>(type == 1 ? KMAX1 : KMAX, (M + (1 << 19) - 1) >> 19);
    // chunk boundaries: short first chunks (compute and the download start
    // early) and geometrically shrinking last ones (short tail after the
    // final upload); equal chunks in between
    int64_t bound[HostSlot::KC + 1];
    {
        double w[HostSlot::KC], wsum = 0;
        for (int k = 0; k < K; ++k) w[k] = 1.0;
        // (type 1 keeps equal chunks: a short last chunk was measured slower,
        // its predecessors grow and their spreads stop hiding under the copies)
        if (K >= 6 && type == 2) {
            w[0] = 0.25; w[1] = 0.5;
            w[K - 3] = 0.5; w[K - 2] = 0.25; w[K - 1] = 0.125;
        }
        for (int k = 0; k < K; ++k) wsum += w[k];
        double acc = 0;
        bound[0] = 0;
        for (int k = 0; k < K; ++k) {
            acc += w[k];
            bound[k + 1] = k == K - 1 ? M : std::min<int64_t>(M, (int64_t)std::llround(M * (acc / wsum)));
        }
    }
    // main stream: error flags, then type 2: modes in + amplify + FFT;
    // type 1: zero the shared grid
    ESN_CUDA_TRY(cudaMemsetAsync(p->flags, 0xff, sizeof(unsigned long long) * 8, st));
    for (int h = 0; h < NH; ++h) {
        ESN_CUDA_TRY(cudaMemsetAsync(slot->helper[h]->flags, 0xff, sizeof(unsigned long long) * 8, slot->hst[h]));
        slot->helper[h]->keep_flags = true;
    }
    // the transfer streams start after everything queued before this call
    ESN_CUDA_TRY(cudaEventRecord(slot->ev_in, st));
    ESN_CUDA_TRY(cudaStreamWaitEvent(up, slot->ev_in, 0));
    ESN_CUDA_TRY(cudaStreamWaitEvent(down, slot->ev_in, 0));
    if (type == 2) {
        if (cudaMemcpyAsync(slot->df, f, cb * nm * T, cudaMemcpyHostToDevice, up) != cudaSuccess)
            return fail(ESN_INTERNAL_ERROR, "H2D copy failed");
        ESN_CUDA_TRY(cudaEventRecord(slot->ev_in, up));
        ESN_CUDA_TRY(cudaStreamWaitEvent(st, slot->ev_in, 0));
        if (p->dtype == ESN_F64)
            rc = launch_amplify<double>(p->dim, p->ntransf, p->n, p->N, (const double *)slot->df, (const double *)p->pk[0],
                                        (const double *)p->pk[1], (const double *)p->pk[2], (double *)p->grid,
                                        p->flags + 6, st);
        else
            rc = launch_amplify<float>(p->dim, p->ntransf, p->n, p->N, (const float *)slot->df, (const float *)p->pk[0],
                                       (const float *)p->pk[1], (const float *)p->pk[2], (float *)p->grid, p->flags + 6,
                                       st);
        if (rc) return rc;
        if ((rc = plan_fft(p, p->grid, st))) return rc;
    } else {
        ESN_CUDA_TRY(cudaMemsetAsync(p->grid, 0, real_size(p->dtype) * 2 * (size_t)p->G * p->ntransf, st));
    }
    ESN_CUDA_TRY(cudaEventRecord(slot->ev_grid, st));
    // all uploads back to back (chunk k lands in staging slot lo: disjoint
    // per chunk, so no reuse hazard)
    auto block = [&](int64_t lo) {  // (T, cnt) staging block of chunk at lo
        return (char *)slot->dc + (T > 1 ? (size_t)M * T * cb + (size_t)lo * T * cb : (size_t)lo * cb);
    };
    // complex64 input strengths land in the half of the staging buffer that
    // block() leaves free, and are upcast into block() on the compute stream
    auto stage64 = [&](int64_t lo) {
        return (char *)slot->dc + (T > 1 ? (size_t)lo * T * 8 : (size_t)M * cb + (size_t)lo * 8);
    };
    for (int k = 0; k < K; ++k) {
        const int64_t lo = bound[k], cnt = bound[k + 1] - lo;
        if (cnt <= 0) continue;
        for (int d = 0; d < dim; ++d)
            if (cudaMemcpyAsync((char *)slot->dx[d] + lo * xsz, (const char *)xs[d] + lo * xsz, xsz * cnt, cudaMemcpyHostToDevice,
                                up) != cudaSuccess)
                return fail(ESN_INTERNAL_ERROR, "H2D copy failed");
        if (type == 1 && (rc = c64in ? copy_rows(stage64(lo), c, cnt, M, 0, lo, cnt, T, 8, cudaMemcpyHostToDevice, up)
                                     : copy_rows(block(lo), c, cnt, M, 0, lo, cnt, T, cb, cudaMemcpyHostToDevice, up)))
            return rc;
        ESN_CUDA_TRY(cudaEventRecord(slot->ev_up[k], up));
        if (trace) cudaEventRecord(tev[1][k], up);
    }
    for (int k = 0; k < K; ++k) {
        const int h = k % NH;
        esn_plan q = slot->helper[h];
        cudaStream_t hs = slot->hst[h];
        const int64_t lo = bound[k], cnt = bound[k + 1] - lo;
        if (cnt <= 0) continue;
        // chunk views of the (T, M) strength / output arrays: the kernels
        // index c[t * cnt + j], so T > 1 stages through a (T, cnt) block in
        // the second half of the staging buffer (disjoint per chunk)
        char *blk = block(lo);
        ESN_CUDA_TRY(cudaStreamWaitEvent(hs, slot->ev_up[k], 0));
        q->ibase = lo;
        const void *cx[3] = {nullptr, nullptr, nullptr};
        for (int d = 0; d < dim; ++d) cx[d] = (const char *)slot->dx[d] + lo * xsz;
        if ((rc = esn_plan_setpts(q, cnt, cdt, cx[0], cx[1], cx[2]))) return rc;
        ESN_CUDA_TRY(cudaStreamWaitEvent(hs, slot->ev_grid, 0));
        if (type == 1) {
            if (c64in && (rc = launch_upcast_c64(stage64(lo), blk, cnt * T, hs))) return rc;
            if ((rc = do_spread(q, blk, p->grid, false))) return rc;
            if (trace) cudaEventRecord(tev[2][k], hs);
        } else {
            if ((rc = do_interp(q, p->grid, blk))) return rc;
            ESN_CUDA_TRY(cudaEventRecord(slot->ev_comp[k], hs));
            ESN_CUDA_TRY(cudaStreamWaitEvent(down, slot->ev_comp[k], 0));
            if ((rc = copy_rows(c, blk, M, cnt, lo, 0, cnt, T, cb, cudaMemcpyDeviceToHost, down))) return rc;
            if (trace) {
                cudaEventRecord(tev[2][k], hs);
                cudaEventRecord(tev[3][k], down);
            }
        }
        // (the helper's scratch is reused NH chunks later on the same stream)
        ESN_CUDA_TRY(cudaEventRecord(slot->ev_done[h], hs));
    }
    for (int h = 0; h < NH; ++h) ESN_CUDA_TRY(cudaStreamWaitEvent(st, slot->ev_done[h], 0));
    ESN_CUDA_TRY(cudaEventRecord(slot->ev_down, down));
    ESN_CUDA_TRY(cudaStreamWaitEvent(st, slot->ev_down, 0));
    if (type == 1) {
        if ((rc = fft_deconv_type1(p, p->grid, slot->df, st, nullptr))) return rc;
        if (cudaMemcpyAsync(f, slot->df, cb * nm * T, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            return fail(ESN_INTERNAL_ERROR, "D2H copy failed");
    }
    const auto t_enq = std::chrono::steady_clock::now();
    ESN_CUDA_TRY(cudaStreamSynchronize(st));
    if (trace) {
        fprintf(stderr, "[esn] pipelined K=%d NH=%d: enqueue %.3f ms, wait %.3f ms\n", K, NH,
                std::chrono::duration<double, std::milli>(t_enq - t_start).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enq).count());
        cudaDeviceSynchronize();
        for (int k = 0; k < K; ++k) {
            float a = 0, b = 0, d = 0;
            cudaEventElapsedTime(&a, tev[0][0], tev[1][k]);
            cudaEventElapsedTime(&b, tev[0][0], tev[2][k]);
            if (type == 2) cudaEventElapsedTime(&d, tev[0][0], tev[3][k]);
            fprintf(stderr, "[esn]   chunk %2d: up %.3f  comp %.3f  down %.3f ms\n", k, a, b, d);
        }
        if (type == 1) {  // FFT + deconvolution + download of the modes on the plan stream
            cudaEventRecord(tev[3][K], st);
            cudaEventSynchronize(tev[3][K]);
            float e = 0;
            cudaEventElapsedTime(&e, tev[0][0], tev[3][K]);
            fprintf(stderr, "[esn]   done (FFT, deconvolution, D2H): %.3f ms\n", e);
        }
        cudaGetLastError();  // (events a transfer-only probe never recorded)
    }
    const auto t_sync = std::chrono::steady_clock::now();
    // merge the error flags: helpers hold the coordinate (and type-1
    // strength) flags with global indices, the main plan the mode flags
    unsigned long long h[HostSlot::NH + 1][8];
    ESN_CUDA_TRY(cudaMemcpy(h[0], p->flags, sizeof(h[0]), cudaMemcpyDeviceToHost));
    for (int k = 0; k < NH; ++k)
        ESN_CUDA_TRY(cudaMemcpy(h[1 + k], slot->helper[k]->flags, sizeof(h[0]), cudaMemcpyDeviceToHost));
    unsigned long long merged[8];
    for (int i = 0; i < 8; ++i) {
        merged[i] = h[0][i];
        for (int k = 1; k <= NH; ++k) merged[i] = std::min(merged[i], h[k][i]);
    }
    ESN_CUDA_TRY(cudaMemcpy(p->flags, merged, sizeof(merged), cudaMemcpyHostToDevice));
    rc = esn_plan_check(p, nullptr);
    if (trace)
        fprintf(stderr, "[esn]   flag merge + check %.3f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_sync).count());
    return rc;
}

// Batched type 1 with points below the chunked-pipeline threshold (c5: 64
// transforms of 1e6 points): the strengths dominate the transfer (512 MB),
// so the pipeline runs over TRANSFORM groups instead of point chunks --
// coordinates up and one sort, then per group of 32 transforms: strengths up
// (transfer stream) -> batched spread + FFT + deconvolution on the plan
// stream -> modes down (second transfer stream), so group g's compute and
// download overlap group g + 1's upload.
static int transform_pipelined(HostSlot *slot, int dim, int64_t M, const double *const *xs, int T, void *c, void *f,
                               int64_t nm, size_t cb, bool c64in, int cdt) {
    const size_t xsz = cdt == ESN_F32 ? 4 : 8;
    esn_plan p = slot->plan;
    cudaStream_t st = p->st;
    if (!slot->up) {
        ESN_CUDA_TRY(cudaStreamCreateWithFlags(&slot->up, cudaStreamNonBlocking));
        ESN_CUDA_TRY(cudaStreamCreateWithFlags(&slot->down, cudaStreamNonBlocking));
        ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_grid, cudaEventDisableTiming));
        ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_in, cudaEventDisableTiming));
        ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_down, cudaEventDisableTiming));
        for (int k = 0; k < HostSlot::KC; ++k) {
            ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_up[k], cudaEventDisableTiming));
            ESN_CUDA_TRY(cudaEventCreateWithFlags(&slot->ev_comp[k], cudaEventDisableTiming));
        }
    }
    cudaStream_t up = slot->up, down = slot->down;
    // groups of 32 transforms (one lane group of the batched spreader); a
    // remainder below 2 joins the previous group (a batch keeps >= 2)
    int bounds[HostSlot::KC + 1], ng = 0;
    for (int t0 = 0; t0 < T && ng < HostSlot::KC - 1; t0 += 32) bounds[ng++] = t0;
    bounds[ng] = T;
    if (ng > 1 && bounds[ng] - bounds[ng - 1] < 2) bounds[--ng] = T;
    if (bounds[ng] != T) bounds[ng] = T;
    ESN_CUDA_TRY(cudaEventRecord(slot->ev_in, st));
    ESN_CUDA_TRY(cudaStreamWaitEvent(up, slot->ev_in, 0));
    ESN_CUDA_TRY(cudaStreamWaitEvent(down, slot->ev_in, 0));
    for (int d = 0; d < dim; ++d)
        if (cudaMemcpyAsync(slot->dx[d], xs[d], xsz * M, cudaMemcpyHostToDevice, up) != cudaSuccess)
            return fail(ESN_INTERNAL_ERROR, "H2D copy failed");
    ESN_CUDA_TRY(cudaEventRecord(slot->ev_grid, up));
    // (complex64 input strengths: staged in the second half of dc, upcast per group)
    const size_t cbi = c64in ? 8 : cb;
    char *const stage = (char *)slot->dc + (c64in ? (size_t)M * T * cb : 0);
    for (int g = 0; g < ng; ++g) {
        const size_t off = (size_t)bounds[g] * M * cbi, bytes = (size_t)(bounds[g + 1] - bounds[g]) * M * cbi;
        if (cudaMemcpyAsync(stage + off, (const char *)c + off, bytes, cudaMemcpyHostToDevice, up) != cudaSuccess)
            return fail(ESN_INTERNAL_ERROR, "H2D copy failed");
        ESN_CUDA_TRY(cudaEventRecord(slot->ev_up[g], up));
    }
    ESN_CUDA_TRY(cudaStreamWaitEvent(st, slot->ev_grid, 0));
    int rc = esn_plan_setpts(p, M, cdt, slot->dx[0], slot->dx[1], slot->dx[2]);  // (resets every flag)
    const int T0 = p->ntransf;
    p->keep_flags = true;  // the data flag accumulates over the groups
    struct Restore {       // (every exit path restores the plan)
        esn_plan p;
        int T0;
        ~Restore() {
            p->keep_flags = false;
            p->ntransf = T0;
        }
    } restore{p, T0};
    for (int g = 0; g < ng && !rc; ++g) {
        ESN_CUDA_TRY(cudaStreamWaitEvent(st, slot->ev_up[g], 0));
        if (c64in && (rc = launch_upcast_c64(stage + (size_t)bounds[g] * M * 8, (char *)slot->dc + (size_t)bounds[g] * M * cb,
                                              (int64_t)(bounds[g + 1] - bounds[g]) * M, st)))
            break;
        p->ntransf = bounds[g + 1] - bounds[g];  // (the plan's buffers are sized for all T)
        rc = esn_plan_execute(p, (char *)slot->dc + (size_t)bounds[g] * M * cb,
                              (char *)slot->df + (size_t)bounds[g] * nm * cb);
        if (rc) break;
        ESN_CUDA_TRY(cudaEventRecord(slot->ev_comp[g], st));
        ESN_CUDA_TRY(cudaStreamWaitEvent(down, slot->ev_comp[g], 0));
        const size_t off = (size_t)bounds[g] * nm * cb, bytes = (size_t)(bounds[g + 1] - bounds[g]) * nm * cb;
        if (cudaMemcpyAsync((char *)f + off, (const char *)slot->df + off, bytes, cudaMemcpyDeviceToHost, down) !=
            cudaSuccess)
            return fail(ESN_INTERNAL_ERROR, "D2H copy failed");
    }
    p->keep_flags = false;
    p->ntransf = T0;
    ESN_CUDA_TRY(cudaEventRecord(slot->ev_down, down));
    ESN_CUDA_TRY(cudaStreamWaitEvent(st, slot->ev_down, 0));
    if (rc) {
        cudaStreamSynchronize(st);
        return rc;
    }
    return esn_plan_check(p, nullptr);
}

int esn_nufft_host(int type, int dim, int64_t M, const double *x, const double *y, const double *z, int ntransf,
                   void *c, int isign, double tol, const int64_t *nmodes, void *f, const esn_opts *opts) {
    // argument misuse -> SIZE_ERROR before any core work (esnufftpy __init__.py:54-122)
    if (type != 1 && type != 2) return fail(ESN_SIZE_ERROR, "type must be 1 or 2");
    if (dim < 1 || dim > 3) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
    if (M < 0) return fail(ESN_SIZE_ERROR, "negative point count");
    if (isign != 1 && isign != -1) return fail(ESN_SIZE_ERROR, "isign must be +1 or -1");
    if (ntransf < 1) return fail(ESN_SIZE_ERROR, "ntransf must be >= 1");
    if (!nmodes || !c || !f) return fail(ESN_SIZE_ERROR, "null array argument");
    const double *xs[3] = {x, y, z};
    for (int d = 0; d < dim; ++d)
        if (M > 0 && !xs[d]) return fail(ESN_SIZE_ERROR, "coordinate array %d missing", d + 1);
    esn_opts o;
    if (opts) o = *opts; else esn_default_opts(&o);
    const int dtype = o.dtype == ESN_F32 ? ESN_F32 : ESN_F64;
    std::lock_guard<std::mutex> lk(g_host_mu);
    const bool cacheable = !o.params && !o.coeffs && !o.check_bounds && !o.use_exact_kernel && !o.stream;
    HostSlot *slot = nullptr;
    const int device = current_device();
    if (cacheable) {
        for (auto &s : g_slots) {
            bool same = s.device == device && s.type == type && s.dim == dim && s.isign == isign && s.ntransf == ntransf &&
                        s.dtype == dtype && s.tol == tol && s.sigma == o.sigma && s.method == o.method;
            for (int d = 0; d < dim && same; ++d) same = s.N[d] == nmodes[d];
            if (same) {
                slot = &s;
                break;
            }
        }
    }
    HostSlot tmp{};
    bool transient = false;
    if (!slot) {
        tmp.type = type; tmp.dim = dim; tmp.isign = isign; tmp.ntransf = ntransf; tmp.dtype = dtype;
        tmp.tol = tol; tmp.sigma = o.sigma; tmp.method = o.method; tmp.device = device;
        for (int d = 0; d < 3; ++d) tmp.N[d] = d < dim ? nmodes[d] : 1;
        if (!o.stream) {
            ESN_CUDA_TRY(cudaStreamCreateWithFlags(&tmp.st, cudaStreamNonBlocking));
            o.stream = tmp.st;
        }
        int rc = esn_plan_create(type, dim, nmodes, isign, ntransf, tol, &o, &tmp.plan);
        if (rc) {
            if (tmp.st) cudaStreamDestroy(tmp.st);
            return rc;
        }
        if (cacheable) {
            if (g_slots.size() >= 4) {
                free_slot(g_slots.front());
                g_slots.erase(g_slots.begin());
            }
            g_slots.push_back(tmp);
            slot = &g_slots.back();
        } else {
            transient = true;
            slot = &tmp;
        }
    }
    esn_plan p = slot->plan;
    cudaStream_t st = p->st;
    const size_t cb = real_size(dtype) * 2;
    int64_t nm = 1;
    for (int d = 0; d < dim; ++d) nm *= nmodes[d];
    int rc = ESN_SUCCESS;
    if (M > slot->Mcap || !slot->dc) {
        for (int d = 0; d < 3; ++d) { dfree(slot->dx[d]); slot->dx[d] = nullptr; }
        dfree(slot->dc);
        slot->dc = nullptr;
        for (int d = 0; d < dim && !rc; ++d) rc = dmalloc(p, &slot->dx[d], sizeof(double) * (M > 0 ? M : 1));
        // strengths / outputs plus a (T, chunk) staging block per chunk
        if (!rc) rc = dmalloc(p, &slot->dc, cb * (M > 0 ? M : 1) * ntransf * 2);
        slot->Mcap = M;
    }
    if (!rc && !slot->df) rc = dmalloc(p, &slot->df, cb * nm * ntransf);
    const bool c64in = type == 1 && dtype == ESN_F64 && o.strength_dtype == ESN_F32;
    const int cdt = o.coord_dtype == ESN_F32 ? ESN_F32 : ESN_F64;  // (host coordinates as float32)
    const size_t xsz = cdt == ESN_F32 ? 4 : 8;
    if (o.strength_dtype && o.strength_dtype != dtype && !c64in)
        return fail(ESN_SIZE_ERROR, "strength_dtype: only complex64 strengths for a float64 type-1 transform");
    bool pipe = !rc && cacheable && M >= (int64_t)(2 << 20) && is_pinned(c) && is_pinned(f);
    for (int d = 0; d < dim && pipe; ++d) pipe = is_pinned(xs[d]);
    static const char *nopipe = getenv("ESN_NO_PIPELINE");
    if (nopipe && nopipe[0] == '1') pipe = false;
    if (pipe) {
        rc = pipelined(slot, type, dim, M, xs, ntransf, c, f, nm, cb, c64in, cdt);
        if (transient) free_slot(*slot);
        return rc;
    }
    bool tpipe = !rc && cacheable && type == 1 && ntransf > 32 && M > 0 && is_pinned(c) && is_pinned(f);
    for (int d = 0; d < dim && tpipe; ++d) tpipe = is_pinned(xs[d]);
    if (nopipe && nopipe[0] == '1') tpipe = false;
    if (tpipe) {
        rc = transform_pipelined(slot, dim, M, xs, ntransf, c, f, nm, cb, c64in, cdt);
        if (transient) free_slot(*slot);
        return rc;
    }
    if (!rc) {
        for (int d = 0; d < dim && M > 0; ++d)
            if (cudaMemcpyAsync(slot->dx[d], xs[d], xsz * M, cudaMemcpyHostToDevice, st) != cudaSuccess)
                rc = fail(ESN_INTERNAL_ERROR, "H2D copy failed");
        if (!rc && type == 1 && M > 0) {
            // (complex64 strengths: staged in the second half of dc, upcast into the first)
            char *dst = (char *)slot->dc + (c64in ? cb * M * ntransf : 0);
            if (cudaMemcpyAsync(dst, c, (c64in ? 8 : cb) * M * ntransf, cudaMemcpyHostToDevice, st) != cudaSuccess)
                rc = fail(ESN_INTERNAL_ERROR, "H2D copy failed");
            if (!rc && c64in) rc = launch_upcast_c64(dst, slot->dc, M * ntransf, st);
        }
        if (!rc && type == 2)
            if (cudaMemcpyAsync(slot->df, f, cb * nm * ntransf, cudaMemcpyHostToDevice, st) != cudaSuccess)
                rc = fail(ESN_INTERNAL_ERROR, "H2D copy failed");
    }
    if (!rc) rc = esn_plan_setpts(p, M, cdt, slot->dx[0], slot->dx[1], slot->dx[2]);
    if (!rc) rc = esn_plan_execute(p, slot->dc, slot->df);
    if (!rc) {
        if (type == 1) {
            if (cudaMemcpyAsync(f, slot->df, cb * nm * ntransf, cudaMemcpyDeviceToHost, st) != cudaSuccess)
                rc = fail(ESN_INTERNAL_ERROR, "D2H copy failed");
        } else if (M > 0) {
            if (cudaMemcpyAsync(c, slot->dc, cb * M * ntransf, cudaMemcpyDeviceToHost, st) != cudaSuccess)
                rc = fail(ESN_INTERNAL_ERROR, "D2H copy failed");
        }
    }
    if (!rc) rc = esn_plan_check(p, nullptr);
    if (transient) free_slot(*slot);
    return rc;
}

int esn_nufft1d1(int64_t M, const double *x, const void *c, int isign, double tol, int64_t N1, void *f,
                 const esn_opts *opts) {
    int64_t nm[1] = {N1};
    return esn_nufft_host(1, 1, M, x, nullptr, nullptr, 1, (void *)c, isign, tol, nm, f, opts);
}
int esn_nufft2d1(int64_t M, const double *x, const double *y, const void *c, int isign, double tol, int64_t N1,
                 int64_t N2, void *f, const esn_opts *opts) {
    int64_t nm[2] = {N1, N2};
    return esn_nufft_host(1, 2, M, x, y, nullptr, 1, (void *)c, isign, tol, nm, f, opts);
}
int esn_nufft3d1(int64_t M, const double *x, const double *y, const double *z, const void *c, int isign, double tol,
                 int64_t N1, int64_t N2, int64_t N3, void *f, const esn_opts *opts) {
    int64_t nm[3] = {N1, N2, N3};
    return esn_nufft_host(1, 3, M, x, y, z, 1, (void *)c, isign, tol, nm, f, opts);
}
int esn_nufft1d2(int64_t M, const double *x, void *c, int isign, double tol, int64_t N1, const void *f,
                 const esn_opts *opts) {
    int64_t nm[1] = {N1};
    return esn_nufft_host(2, 1, M, x, nullptr, nullptr, 1, c, isign, tol, nm, (void *)f, opts);
}
int esn_nufft2d2(int64_t M, const double *x, const double *y, void *c, int isign, double tol, int64_t N1, int64_t N2,
                 const void *f, const esn_opts *opts) {
    int64_t nm[2] = {N1, N2};
    return esn_nufft_host(2, 2, M, x, y, nullptr, 1, c, isign, tol, nm, (void *)f, opts);
}
int esn_nufft3d2(int64_t M, const double *x, const double *y, const double *z, void *c, int isign, double tol,
                 int64_t N1, int64_t N2, int64_t N3, const void *f, const esn_opts *opts) {
    int64_t nm[3] = {N1, N2, N3};
    return esn_nufft_host(2, 3, M, x, y, z, 1, c, isign, tol, nm, (void *)f, opts);
}

}  // extern "C"
