// esn_setpts.cu -- point preparation on sm_100a: fold + grid scale + bin key
// (fused with the finite / bounds checks), bin counting sort (warp-aggregated
// atomic histogram -> single-CTA exclusive scan -> scatter of the permutation
// and of the sorted grid coordinates), and the subproblem table.
//
// Replaces build_point_set / fold_coords / bin_sort / ensure_sorted /
// partition_subproblems (spreadinterp.py:79-150, grid.py:152-254).  The
// reference sorts by 16x4x4 boxes of floor(g) with a stable CPU counting
// sort; here bins are boxes of the footprint origin i0 = floor(g - w/2 + 1)
// (spreadinterp.py:117-120) so a bin maps to a tight (bs + w - 1)^d tile, and
// the within-bin order is whatever the atomics hand out (the reference only
// guarantees bin membership, SPEC.md "bin_sort ... stability is NOT
// guaranteed multithreaded").
#include <cuda_runtime.h>

#include <climits>
#include <cstring>
#include <mutex>

#include "esn_internal.h"

namespace esn {

static thread_local char g_errbuf[1024];

void set_error(const char *msg) {
    std::strncpy(g_errbuf, msg, sizeof(g_errbuf) - 1);
    g_errbuf[sizeof(g_errbuf) - 1] = 0;
}

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_errbuf, sizeof(g_errbuf), fmt, ap);
    va_end(ap);
    return code;
}

const char *last_error() { return g_errbuf; }

int device_sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 0 || dev >= 64) dev = 0;
    if (cached[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached[dev] = v;
    }
    return cached[dev];
}

// grid.py:152-168 + spreadinterp.py:99-100 in float64: np.mod(x, 2 pi)
// (fmod plus 2 pi when the signs differ), exact 2 pi wraps to 0, scale by
// n / 2 pi (host-computed), pull back g >= n.  Bit-identical to numpy.
__device__ __forceinline__ double fold_scale(double x, double n, double scale) {
    const double two_pi = 6.283185307179586;
    double r = fmod(x, two_pi);
    if (r < 0.0) r += two_pi;
    if (r >= two_pi) r = 0.0;
    double g = r * scale;
    if (g >= n) g -= n;
    return g;
}

template <typename T>
__device__ __forceinline__ T to_plan(double g, int n) {
    T v = (T)g;
    if (v >= (T)n) v -= (T)n;  // float rounding can land exactly on n
    return v;
}

template <typename T>
__device__ __forceinline__ int point_key(const SetptsArgs &a, int64_t i, const double *xin, double *gout, bool check) {
    int key = 0, mul = 1;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (d >= a.g.dim) break;
        const double x = xin[d];
        double g = 0.0;
        if (!isfinite(x)) {
            if (check) atomicMin(&a.flags[d], (unsigned long long)i);
        } else {
            if (check && a.check_bounds && fabs(x) > 3.0 * 3.141592653589793)
                atomicMin(&a.flags[3 + d], (unsigned long long)i);
            if (a.grid_units) {
                g = x;  // caller already folded (bin_sort on grid coordinates, grid.py:202)
                if (g >= (double)a.g.n[d]) g -= (double)a.g.n[d];
                if (g < 0.0) g = 0.0;
            } else {
                g = fold_scale(x, (double)a.g.n[d], a.scale[d]);
            }
        }
        gout[d] = g;
        int i0 = (int)floor(g - 0.5 * a.g.w + 1.0);  // spreadinterp.py:117-120
        if (i0 < 0) i0 += a.g.n[d];
        key += (i0 / a.g.bs[d]) * mul;
        mul *= a.g.nb[d];
    }
    return key;
}

constexpr int kILP = 4;  // points in flight per thread (independent loads / atomics)

template <typename XT>
__device__ __forceinline__ void load_coords(const SetptsArgs &a, int64_t base, double (*x)[3]) {
    // all loads first (independent, read-only), compute afterwards
#pragma unroll
    for (int u = 0; u < kILP; ++u) {
        const int64_t i = base + (int64_t)u * blockDim.x;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            x[u][d] = 0.0;
            if (d < a.g.dim && i < a.M) x[u][d] = (double)__ldg(reinterpret_cast<const XT *>(a.x[d]) + i);
        }
    }
}

// Pass 1: bin histogram (fire-and-forget REDs, no return value needed) and
// the finite / bounds flags.
template <typename XT, typename T>
__global__ void __launch_bounds__(256) k_setpts_count(SetptsArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kILP;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * kILP + threadIdx.x; base < a.M; base += stride) {
        double x[kILP][3];
        load_coords<XT>(a, base, x);
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            if (i >= a.M) continue;
            double g[3];
            atomicAdd(&a.bin_count[point_key<T>(a, i, x[u], g, true)], 1);
        }
    }
}

// Pass 2: claim a slot in the point's bin (atomic on the bin cursor) and
// write its full record {g, j} there with one 256-bit store.
template <typename XT, typename T>
__global__ void __launch_bounds__(256) k_setpts_scatter(SetptsArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kILP;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * kILP + threadIdx.x; base < a.M; base += stride) {
        double x[kILP][3];
        load_coords<XT>(a, base, x);
        int pos[kILP];
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            double g[3];
            pos[u] = i < a.M ? atomicAdd(&a.cursor[point_key<T>(a, i, x[u], g, false)], 1) : -1;
            x[u][0] = g[0];
            x[u][1] = a.g.dim > 1 ? g[1] : 0.0;
            x[u][2] = a.g.dim > 2 ? g[2] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
            if (pos[u] < 0) continue;
            const unsigned long long j = (unsigned long long)(unsigned)(base + (int64_t)u * blockDim.x);
            asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(a.rec + pos[u]),
                         "l"(__double_as_longlong(x[u][0])), "l"(__double_as_longlong(x[u][1])),
                         "l"(__double_as_longlong(x[u][2])), "l"(j)
                         : "memory");
        }
    }
}

// Single-CTA exclusive scan of the bin counts and of the per-bin subproblem
// counts ceil(count / max_subprob); also publishes the subproblem total.
__global__ void __launch_bounds__(1024) k_scan_bins(const int *count, int *start, int *cursor, int *subofs,
                                                    int nbins, int maxsub, int *nsub_total) {
    __shared__ int wsum[2][32];
    __shared__ int carry[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry[0] = carry[1] = 0;
    __syncthreads();
    for (int base = 0; base < nbins; base += 1024) {
        const int i = base + tid;
        const int c = i < nbins ? count[i] : 0;
        const int s = i < nbins ? (c + maxsub - 1) / maxsub : 0;
        int xc = c, xs = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int yc = __shfl_up_sync(0xffffffffu, xc, o);
            int ys = __shfl_up_sync(0xffffffffu, xs, o);
            if (lane >= o) {
                xc += yc;
                xs += ys;
            }
        }
        if (lane == 31) {
            wsum[0][warp] = xc;
            wsum[1][warp] = xs;
        }
        __syncthreads();
        if (warp == 0) {
            int vc = wsum[0][lane], vs = wsum[1][lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int yc = __shfl_up_sync(0xffffffffu, vc, o);
                int ys = __shfl_up_sync(0xffffffffu, vs, o);
                if (lane >= o) {
                    vc += yc;
                    vs += ys;
                }
            }
            wsum[0][lane] = vc;
            wsum[1][lane] = vs;
        }
        __syncthreads();
        const int offc = carry[0] + (warp ? wsum[0][warp - 1] : 0);
        const int offs = carry[1] + (warp ? wsum[1][warp - 1] : 0);
        if (i < nbins) {
            start[i] = offc + xc - c;
            cursor[i] = offc + xc - c;
            subofs[i] = offs + xs - s;
        }
        __syncthreads();
        if (tid == 0) {
            carry[0] += wsum[0][31];
            carry[1] += wsum[1][31];
        }
        __syncthreads();
    }
    if (tid == 0) {
        start[nbins] = carry[0];
        subofs[nbins] = carry[1];
        *nsub_total = carry[1];
    }
}

__global__ void k_fill_subprob(const int *count, const int *start, const int *subofs, int nbins, int maxsub,
                               int4 *table) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += gridDim.x * blockDim.x) {
        const int c = count[b];
        int o = subofs[b];
        for (int s = 0; s * maxsub < c; ++s)
            table[o + s] = make_int4(b, start[b] + s * maxsub, min(maxsub, c - s * maxsub), 0);
    }
}

template <typename XT, typename T>
static int setpts_impl(const SetptsArgs &a, int nbins, int maxsub, int4 *subprob, int *nsub, int *scan_aux,
                       cudaStream_t st) {
    const int threads = 256;
    int64_t blocks = (a.M + threads * kILP - 1) / (threads * kILP);
    const int64_t cap = (int64_t)device_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (a.M > 0) {
        k_setpts_count<XT, T><<<(int)blocks, threads, 0, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
    }
    k_scan_bins<<<1, 1024, 0, st>>>(a.bin_count, a.bin_start, a.cursor, scan_aux, nbins, maxsub, nsub);
    ESN_CUDA_TRY(cudaGetLastError());
    if (a.M > 0) {
        k_setpts_scatter<XT, T><<<(int)blocks, threads, 0, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
        int fb = (nbins + 255) / 256;
        k_fill_subprob<<<fb < 1 ? 1 : fb, 256, 0, st>>>(a.bin_count, a.bin_start, scan_aux, nbins, maxsub,
                                                         subprob);
        ESN_CUDA_TRY(cudaGetLastError());
    }
    return ESN_SUCCESS;
}

__global__ void k_sort_view(const Rec *rec, const int *bin_start, int nbins, int *perm, int *keys) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += gridDim.x * blockDim.x) {
        for (int k = bin_start[b]; k < bin_start[b + 1]; ++k) {
            const int j = rec[k].j;
            if (perm) perm[k] = j;
            if (keys) keys[j] = b;
        }
    }
}

int launch_sort_view(int dtype, const void *rec, const int *bin_start, int nbins, int64_t M, int *perm, int *keys,
                     cudaStream_t st) {
    if (M == 0) return ESN_SUCCESS;
    int fb = (nbins + 127) / 128;
    (void)dtype;
    k_sort_view<<<fb, 128, 0, st>>>((const Rec *)rec, bin_start, nbins, perm, keys);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

int launch_setpts(const SetptsArgs &a, int dtype, int nbins, int max_subprob, int4 *subprob, int *nsub,
                  int *scan_aux, cudaStream_t st) {
    if (dtype == ESN_F64) {
        return a.coord_f32 ? setpts_impl<float, double>(a, nbins, max_subprob, subprob, nsub, scan_aux, st)
                           : setpts_impl<double, double>(a, nbins, max_subprob, subprob, nsub, scan_aux, st);
    }
    return a.coord_f32 ? setpts_impl<float, float>(a, nbins, max_subprob, subprob, nsub, scan_aux, st)
                       : setpts_impl<double, float>(a, nbins, max_subprob, subprob, nsub, scan_aux, st);
}

}  // namespace esn
