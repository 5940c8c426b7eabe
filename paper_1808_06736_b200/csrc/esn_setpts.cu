// esn_setpts.cu -- point preparation on sm_100a: fold + grid scale + sort key
// (fused with the finite / bounds checks), counting sort over fine keys
// (RED histogram -> 3-phase exclusive scan -> atomic-cursor scatter of one
// 256-bit record per point), and the subproblem table of the spreader.
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

#include <algorithm>
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

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    return (dev < 0 || dev >= 64) ? 0 : dev;
}

int device_sm_count() {
    static int cached[64] = {0};
    const int dev = current_device();
    if (cached[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached[dev] = v;
    }
    return cached[dev];
}

// grid.py:152-168 + spreadinterp.py:99-100 in float64: np.mod(x, 2 pi)
// (fmod plus 2 pi when the signs differ), exact 2 pi wraps to 0, scale by
// n / 2 pi (host-computed), pull back g >= n.  Bit-identical to numpy; fmod
// is skipped when |x| < 2 pi, where it is the identity.
__device__ __forceinline__ double fold_scale(double x, double n, double scale) {
    const double two_pi = 6.283185307179586;
    double r = x;
    if (!(fabs(x) < two_pi)) r = fmod(x, two_pi);
    if (r < 0.0) r += two_pi;
    if (r >= two_pi) r = 0.0;
    double g = r * scale;
    if (g >= n) g -= n;
    return g;
}

// exact q = i / d for 0 <= i < 2^31 via a float64 reciprocal and one fix-up
__device__ __forceinline__ int fast_div(int i, int d, double inv) {
    int q = __double2int_rz((double)i * inv);
    if (q * d > i) --q;
    else if ((q + 1) * d <= i) ++q;
    return q;
}

// Grid coordinate of one coordinate value on the rare paths: non-finite
// (flag d), |x| > 3 pi (flag 3 + d, when checked), |x| >= 2 pi (fmod fold)
// or caller-folded grid units.  (Out of line it cost 20-30 registers for
// the call; inline it is only a branch target.)
__device__ __forceinline__ double grid_coord_slow(unsigned long long *flags, unsigned long long idx, double x, int d,
                                              bool check, int check_bounds, int grid_units, double n, double scale) {
    double g = 0.0;
    if (!isfinite(x)) {
        if (check) atomicMin(&flags[d], idx);
    } else {
        if (check && check_bounds && fabs(x) > 3.0 * 3.141592653589793) atomicMin(&flags[3 + d], idx);
        if (grid_units) {
            g = x;  // caller already folded (bin_sort on grid coordinates, grid.py:202)
            if (g >= n) g -= n;
            if (g < 0.0) g = 0.0;
        } else {
            g = fold_scale(x, n, scale);
        }
    }
    return g;
}

// Fine sort key of one point; g receives its grid coordinates.  DIM = 0:
// the plan's dimension at run time (the unsorted path).  The common case
// |x| < 2 pi (finite, inside the 3 pi bound, fmod the identity) is
// fold_scale's arithmetic as selects, bit-identical, no branches.
template <int DIM = 0>
__device__ __forceinline__ int point_key(const SetptsArgs &a, int64_t i, const double *xin, double *gout, bool check) {
    int bin = 0, loc = 0, bmul = 1, lmul = 1;
    const double two_pi = 6.283185307179586;
#pragma unroll
    for (int d = 0; d < (DIM ? DIM : 3); ++d) {
        if (!DIM && d >= a.g.dim) break;
        const double x = xin[d];
        const double n = (double)a.g.n[d];
        double g;
        if (fabs(x) < two_pi && !a.grid_units) {
            double r = x < 0.0 ? x + two_pi : x;
            r = r >= two_pi ? 0.0 : r;
            g = r * a.scale[d];
            g = g >= n ? g - n : g;
        } else {
            g = grid_coord_slow(a.flags, (unsigned long long)(i + a.ibase), x, d, check, a.check_bounds, a.grid_units,
                                n, a.scale[d]);
        }
    gout[d] = g;
        int i0 = __double2int_rd(g - 0.5 * a.g.w + 1.0);  // floor (spreadinterp.py:117-120)
        if (i0 < 0) i0 += a.g.n[d];
        const int bs = a.g.bs[d];
        // power-of-two bins (the interpolation bins): shifts, else a float64 reciprocal
        const int q = a.bs_log2[d] >= 0 ? i0 >> a.bs_log2[d] : fast_div(i0, bs, a.inv_bs[d]);
        bin += q * bmul;
        bmul *= a.g.nb[d];
        loc += ((i0 - q * bs) >> a.sbl[d]) * lmul;
        lmul *= ((bs - 1) >> a.sbl[d]) + 1;
    }
    // (i < 2^31: a float64 reciprocal and one fix-up, not a 64-bit division)
    if (a.chunk_len > 0) bin += fast_div((int)i, (int)a.chunk_len, a.inv_chunk) * a.nbins_geo;
    return bin * a.spb + loc;
}

constexpr int kILP = 4;   // points in flight per thread (independent loads / atomics)
constexpr int kSILP = 8;  // record scatter: points in flight per thread

template <typename XT, int DIM, int U = kILP>
__device__ __forceinline__ void load_coords(const SetptsArgs &a, int64_t base, double (*x)[3]) {
    // all loads first (independent, read-only), compute afterwards
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t i = base + (int64_t)u * blockDim.x;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            x[u][d] = 0.0;
            if (d < DIM && i < a.M) x[u][d] = (double)__ldg(reinterpret_cast<const XT *>(a.x[d]) + i);
        }
    }
}

// Pass 1: key histogram (fire-and-forget REDs: no return trip, no per-point
// state written) plus the finite / bounds flags.  The ranks come from the
// scatter pass's fill cursors.
template <typename XT, int DIM>
__global__ void __launch_bounds__(256, 4) k_setpts_count(SetptsArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kILP;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * kILP + threadIdx.x; base < a.M; base += stride) {
        double x[kILP][3];
        load_coords<XT, DIM>(a, base, x);
        int key[kILP];
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            double g[3];
            key[u] = i < a.M ? point_key<DIM>(a, i, x[u], g, true) : -1;
        }
        // Clustered clouds put runs of consecutive points on one key, and
        // same-address REDs serialise in L2 (c2 on the disc quadrature: 1.05
        // ms/step).  A warp that sees equal keys on neighbouring lanes adds
        // once per key group (match.any); the others -- every warp of a
        // uniform cloud -- keep the plain fire-and-forget REDs (the test costs
        // one shuffle per point; an unconditional match.any cost c2 6 %).
        const int lane = threadIdx.x & 31;
        bool dup = false;
#pragma unroll
        for (int u = 0; u < kILP; ++u) {
            const int nb = __shfl_up_sync(0xffffffffu, key[u], 1);
            dup |= lane > 0 && nb == key[u] && nb >= 0;
        }
        if (__any_sync(0xffffffffu, dup)) {
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                const unsigned grp = __match_any_sync(0xffffffffu, key[u]);
                if (key[u] >= 0 && lane == __ffs(grp) - 1) atomicAdd(&a.key_count[key[u]], __popc(grp));
            }
        } else {
#pragma unroll
            for (int u = 0; u < kILP; ++u)
                if (key[u] >= 0) atomicAdd(&a.key_count[key[u]], 1);
        }
    }
}

// Pass 2: the key again (recomputed with the grid coordinates), pos = an
// atomic fill cursor of the key (key_count holds the key starts after the
// scan; L2-resident), then the point's full
// record {g, j} at pos with one 256-bit store (a whole L2 sector).  Batched
// fp32 plans keep pos in key[] for the strength permutation.  kSILP points
// per thread, all loads issued before the dependent gather.
template <typename XT, int DIM>
__global__ void __launch_bounds__(256) k_setpts_scatter(SetptsArgs a) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kSILP;
    uint64_t pol_first = 0, pol_last = 0;
    if (a.hints) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    }
    // input blocks in DESCENDING order: the count pass read the arrays front
    // to back, so L2 still holds their tail (ESN_SCATTER_REV=0: ascending)
    const int64_t per = (int64_t)blockDim.x * kSILP;
    const int64_t nblk = (a.M + per - 1) / per;
    (void)stride;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t base = (a.rev ? nblk - 1 - blk : blk) * per + threadIdx.x;
        int pos[kSILP];
        double x[kSILP][3];
        load_coords<XT, DIM, kSILP>(a, base, x);
        double g[kSILP][3];
#pragma unroll
        for (int u = 0; u < kSILP; ++u) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            g[u][0] = g[u][1] = g[u][2] = 0.0;
            pos[u] = i < a.M ? point_key<DIM>(a, i, x[u], g[u], false) : -1;
        }
        // fill cursors: plain atomics, all in flight at once -- unless the warp
        // holds runs of equal keys (clustered clouds), where the lanes of a key
        // group take a block of slots with one atomic of their leader (their
        // order inside the key is free)
        const int lane = threadIdx.x & 31;
        bool dup = false;
#pragma unroll
        for (int u = 0; u < kSILP; ++u) {
            const int nb = __shfl_up_sync(0xffffffffu, pos[u], 1);
            dup |= lane > 0 && nb == pos[u] && nb >= 0;
        }
        if (__any_sync(0xffffffffu, dup)) {
#pragma unroll
            for (int u = 0; u < kSILP; ++u) {  // (unrolled: pos[] must stay in registers)
                const unsigned grp = __match_any_sync(0xffffffffu, pos[u]);
                const int leader = __ffs(grp) - 1;
                int base = 0;
                if (pos[u] >= 0 && lane == leader) base = atomicAdd(a.key_count + pos[u], __popc(grp));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (pos[u] >= 0) pos[u] = base + __popc(grp & ((1u << lane) - 1u));
            }
        } else if (a.hints) {
            // the fill cursors (L2-resident key array) evict-last, the
            // streaming record stores evict-first: without the hints about
            // half of the cursor atomics missed the near L2 (ncu, c2)
#pragma unroll
            for (int u = 0; u < kSILP; ++u)
                if (pos[u] >= 0)
                    asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], 1, %2;"
                                 : "=r"(pos[u])
                                 : "l"(a.key_count + pos[u]), "l"(pol_last)
                                 : "memory");
        } else {
#pragma unroll
            for (int u = 0; u < kSILP; ++u)
                if (pos[u] >= 0) pos[u] = atomicAdd(a.key_count + pos[u], 1);  // fill cursor of the key
        }
#pragma unroll
        for (int u = 0; u < kSILP; ++u) {
            if (pos[u] < 0) continue;
            const int64_t i = base + (int64_t)u * blockDim.x;
            if (a.store_pos) a.key[i] = pos[u];
            const unsigned long long j = (unsigned long long)(unsigned)i;
            if (a.hints)
                asm volatile("st.global.L2::cache_hint.v4.u64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a.rec + pos[u]),
                             "l"(__double_as_longlong(g[u][0])), "l"(__double_as_longlong(g[u][1])),
                             "l"(__double_as_longlong(g[u][2])), "l"(j), "l"(pol_first)
                             : "memory");
            else
                asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(a.rec + pos[u]),
                             "l"(__double_as_longlong(g[u][0])), "l"(__double_as_longlong(g[u][1])),
                             "l"(__double_as_longlong(g[u][2])), "l"(j)
                             : "memory");
        }
    }
}

// ---- exclusive scan of the key histogram: block reduce -> down sweep (each
// tile sums the totals before it)
__device__ __forceinline__ int block_scan_excl(int v, int *total, int *wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int s = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) wsum[lane] = s;
    }
    __syncthreads();
    const int off = warp ? wsum[warp - 1] : 0;
    *total = wsum[nw - 1];
    __syncthreads();
    return off + x - v;
}

__global__ void __launch_bounds__(1024) k_scan_reduce(const int *cnt, int n, int *block_sums) {
    __shared__ int wsum[32];
    static_assert(kScanTile == 4 * 1024, "one 16-byte vector per thread");
    const int base = blockIdx.x * kScanTile + threadIdx.x * 4;
    int v = 0;
    if (base + 4 <= n) {
        const int4 q = *reinterpret_cast<const int4 *>(cnt + base);
        v = q.x + q.y + q.z + q.w;
    } else {
        for (int i = base; i < n; ++i) v += cnt[i];
    }
    int total;
    block_scan_excl(v, &total, wsum);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// writes cursor[k] = exclusive prefix (kept: the spreaders read key starts)
// and the same into cnt[k] (the scatter's fill cursors), and bin_start at
// every bin head
__global__ void __launch_bounds__(1024) k_scan_down(int *cnt, int n, const int *block_sums, int *cursor,
                                                   int *bin_start, int spb, int nbins) {
    __shared__ int wsum[32];
    constexpr int U = kScanTile / 1024;
    const int base = blockIdx.x * kScanTile + threadIdx.x * U;  // each thread owns U consecutive keys
    static_assert(U == 4, "one 16-byte vector per thread");
    // full vectors as int4 (the tile base is 16-byte aligned): one 128-bit
    // load / store per thread instead of four strided 32-bit ones
    const bool full = base + U <= n;
    // this tile's offset = the sum of the tile totals before it, reduced
    // here (<= a few thousand tiles) instead of by a one-CTA scan kernel
    // between the two sweeps (one launch and its gap off the sort: ~7 us)
    int pv = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += 1024) pv += block_sums[i];
    int prefix;
    block_scan_excl(pv, &prefix, wsum);
    int v[U], s = 0;
    if (full) {
        const int4 q = *reinterpret_cast<const int4 *>(cnt + base);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = base + u < n ? cnt[base + u] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
    int total;
    int e = block_scan_excl(s, &total, wsum) + prefix;
    int o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        o[u] = e;
        const int k = base + u;
        if (k < n && k % spb == 0) bin_start[k / spb] = e;
        e += v[u];
    }
    if (full) {
        const int4 q = make_int4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<int4 *>(cursor + base) = q;
        *reinterpret_cast<int4 *>(cnt + base) = q;
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (base + u < n) {
                cursor[base + u] = o[u];
                cnt[base + u] = o[u];
            }
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        bin_start[nbins] = prefix + total;
        cursor[n] = prefix + total;  // end of the last key (cell-range readers use key + 1)
    }
}

// Subproblem counts per bin (ceil(count / max_subprob)) -> exclusive scan ->
// total (single CTA over the bins).
__global__ void __launch_bounds__(1024) k_scan_subprob(const int *bin_start, int nbins, int maxsub, int *subofs,
                                                      int *nsub_total) {
    // 8 Ki bins per pass: bin starts staged through shared memory with
    // coalesced loads, 8 consecutive bins per thread (c4: 44 K bins, one
    // bin per thread per pass took 48 us)
    constexpr int U = 8;
    __shared__ int wsum[32];
    __shared__ int carry;
    __shared__ int s_b[1024 * U + 1];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nbins; b0 += 1024 * U) {
        const int nb = min(1024 * U, nbins - b0);
        for (int i = threadIdx.x; i <= nb; i += 1024) s_b[i] = bin_start[b0 + i];
        __syncthreads();
        int v[U], sum = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = threadIdx.x * U + u;
            const int c = i < nb ? s_b[i + 1] - s_b[i] : 0;
            v[u] = (c + maxsub - 1) / maxsub;
            sum += v[u];
        }
        int total;
        int e = block_scan_excl(sum, &total, wsum) + carry;  // (its barriers end the s_b reads)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s_b[threadIdx.x * U + u] = e;
            e += v[u];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += 1024) subofs[b0 + i] = s_b[i];  // coalesced
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *nsub_total = carry;
}

__global__ void k_fill_subprob(const int *bin_start, const int *subofs, int nbins, int maxsub, int4 *table) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += gridDim.x * blockDim.x) {
        const int c = bin_start[b + 1] - bin_start[b];
        const int o = subofs[b];
        for (int s = 0; s * maxsub < c; ++s)
            table[o + s] = make_int4(b, bin_start[b] + s * maxsub, min(maxsub, c - s * maxsub), 0);
    }
}

template <typename XT, int DIM>
static int setpts_impl(const SetptsArgs &a, int nbins, int maxsub, int4 *subprob, int *nsub, int *subofs,
                       cudaStream_t st, const SetptsAux *aux) {
    const int threads = 256;
    // persistent grids: exactly one wave of resident CTAs (a partial second
    // wave left SMs idle at the tail)
    auto resident = [](auto kernel) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, 0) != cudaSuccess || occ < 1) {
            cudaGetLastError();
            occ = 4;
        }
        return (int64_t)device_sm_count() * occ;
    };
    const int64_t cap_count = (int64_t)device_sm_count() * 8;  // (atomics: oversubscribed is faster)
    static PerDev<int64_t> cap_scatter_;
    int64_t &cap_scatter = cap_scatter_();
    if (cap_scatter == 0) {
        cap_scatter = resident(k_setpts_scatter<XT, DIM>);
        // ESN_SCATTER_CTAS=<k>: at most k CTAs per SM (the scatter is bound by
        // its random stores, not by occupancy; fewer resident CTAs leave SM
        // slots to a concurrent FFT / the subproblem tables)
        static const char *e = getenv("ESN_SCATTER_CTAS");
        if (e && atoi(e) > 0) cap_scatter = std::min<int64_t>(cap_scatter, (int64_t)device_sm_count() * atoi(e));
    }
    int64_t blocks = (a.M + threads * kILP - 1) / (threads * kILP);
    if (blocks > cap_count) blocks = cap_count;
    if (blocks < 1) blocks = 1;
    if (aux && aux->count_st) {
        if (a.M > 0) k_setpts_count<XT, DIM><<<(int)blocks, threads, 0, aux->count_st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
        ESN_CUDA_TRY(cudaEventRecord(aux->counted, aux->count_st));
        ESN_CUDA_TRY(cudaStreamWaitEvent(st, aux->counted, 0));
    } else if (a.M > 0) {
        k_setpts_count<XT, DIM><<<(int)blocks, threads, 0, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
    }
    const int nsb = (a.nkeys + kScanTile - 1) / kScanTile;
    k_scan_reduce<<<nsb, 1024, 0, st>>>(a.key_count, a.nkeys, a.block_sums);
    k_scan_down<<<nsb, 1024, 0, st>>>(a.key_count, a.nkeys, a.block_sums, a.cursor, a.bin_start, a.spb, nbins);
    ESN_CUDA_TRY(cudaGetLastError());
    // the subproblem tables depend on the bin starts only: with an aux stream
    // they are built beside the scatter (launched first, so their few CTAs
    // are placed before the scatter's wave takes the SMs)
    const bool fork = aux && aux->st && a.M > 0;
    cudaStream_t ts = fork ? aux->st : st;
    auto tables = [&]() -> int {
        k_scan_subprob<<<1, 1024, 0, ts>>>(a.bin_start, nbins, maxsub, subofs, nsub);
        int fb = (nbins + 255) / 256;
        k_fill_subprob<<<fb < 1 ? 1 : fb, 256, 0, ts>>>(a.bin_start, subofs, nbins, maxsub, subprob);
        ESN_CUDA_TRY(cudaGetLastError());
        return ESN_SUCCESS;
    };
    if (fork) {
        ESN_CUDA_TRY(cudaEventRecord(aux->fork, st));
        ESN_CUDA_TRY(cudaStreamWaitEvent(aux->st, aux->fork, 0));
        if (int rc = tables()) return rc;
        ESN_CUDA_TRY(cudaEventRecord(aux->join, aux->st));
    }
    if (a.M > 0) {
        int64_t sb = (a.M + threads * kSILP - 1) / (threads * kSILP);
        if (sb > cap_scatter) sb = cap_scatter;
        k_setpts_scatter<XT, DIM><<<(int)sb, threads, 0, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
    }
    if (fork) {
        ESN_CUDA_TRY(cudaStreamWaitEvent(st, aux->join, 0));
        return ESN_SUCCESS;
    }
    return tables();
}

// flag = 1 when one bin holds far more than its share of the points
// (clustered clouds): the batched owner-computes spreaders walk a bin's points
// with a single warp, so they hand such plans to the subproblem-balanced
// RED-flush kernel (esn_inst.cuh).  One CTA over the bin starts.
__global__ void __launch_bounds__(1024) k_bin_imbalance(const int *bin_start, int nbins, int64_t M, int *flag) {
    __shared__ int smax[32];
    int m = 0;
    for (int b = threadIdx.x; b < nbins; b += 1024) m = max(m, bin_start[b + 1] - bin_start[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = smax[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) {
            const int64_t mean = M / (nbins > 0 ? nbins : 1) + 1;
            *flag = (m > 2048 && (int64_t)m > 8 * mean) ? 1 : 0;
        }
    }
}

int launch_bin_imbalance(const int *bin_start, int nbins, int64_t M, int *flag, cudaStream_t st) {
    k_bin_imbalance<<<1, 1024, 0, st>>>(bin_start, nbins, M, flag);
    ESN_CUDA_TRY(cudaGetLastError());
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
    (void)dtype;
    if (M == 0) return ESN_SUCCESS;
    int fb = (nbins + 127) / 128;
    k_sort_view<<<fb, 128, 0, st>>>((const Rec *)rec, bin_start, nbins, perm, keys);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

// Records in ORIGINAL order (fold + grid scale + checks, no sort): for
// consumers that only need the records, not their order -- the small 1D
// type-1 plans, whose point-parallel global-atomic spreader (k_spread_global)
// sorts only for locality, which a 20000-cell grid in L2 does not need
// (c1: 1 kernel instead of 7, the sort was ~35 us of a ~90 us step).
template <typename XT>
__global__ void __launch_bounds__(256) k_setpts_unsorted(SetptsArgs a) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.M; i += (int64_t)gridDim.x * blockDim.x) {
        double x[3] = {0.0, 0.0, 0.0}, g[3] = {0.0, 0.0, 0.0};
        for (int d = 0; d < a.g.dim; ++d) x[d] = (double)__ldg(reinterpret_cast<const XT *>(a.x[d]) + i);
        point_key(a, i, x, g, true);
        const unsigned long long j = (unsigned long long)(unsigned)i;
        asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(a.rec + i), "l"(__double_as_longlong(g[0])),
                     "l"(__double_as_longlong(g[1])), "l"(__double_as_longlong(g[2])), "l"(j)
                     : "memory");
    }
}

int launch_setpts_unsorted(const SetptsArgs &a, cudaStream_t st) {
    if (a.M == 0) return ESN_SUCCESS;
    const int64_t b = std::min<int64_t>((a.M + 255) / 256, (int64_t)device_sm_count() * 8);
    if (a.coord_f32)
        k_setpts_unsorted<float><<<(int)b, 256, 0, st>>>(a);
    else
        k_setpts_unsorted<double><<<(int)b, 256, 0, st>>>(a);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

int launch_setpts(const SetptsArgs &a, int nbins, int max_subprob, int4 *subprob, int *nsub, int *subofs,
                  cudaStream_t st, const SetptsAux *aux) {
    auto run = [&](auto xt) {
        using XT = decltype(xt);
        switch (a.g.dim) {
            case 1: return setpts_impl<XT, 1>(a, nbins, max_subprob, subprob, nsub, subofs, st, aux);
            case 2: return setpts_impl<XT, 2>(a, nbins, max_subprob, subprob, nsub, subofs, st, aux);
            default: return setpts_impl<XT, 3>(a, nbins, max_subprob, subprob, nsub, subofs, st, aux);
        }
    };
    return a.coord_f32 ? run(0.0f) : run(0.0);
}

}  // namespace esn
