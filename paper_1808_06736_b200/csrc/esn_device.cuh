// esn_device.cuh -- sm_100a device code of the B200 ES-kernel NUFFT core:
// kernel-row evaluation, spreaders, interpolator, deconvolution and mode
// amplification.  Instantiated per precision by esn_inst_f64.cu / _f32.cu.
//
// Data layout in HBM:
//  * sorted grid coordinates gs[d][k] (plan dtype) and perm[k] (int32,
//    sorted slot -> original index), produced by esn_setpts.cu;
//  * strengths c (ntransf, M) and fine grids (ntransf, n3, n2, n1) as
//    interleaved complex of the plan dtype;
//  * bins are boxes of footprint origins i0 = floor(g - w/2 + 1) (wrapped
//    into [0, n)), so a bin of bs cells owns a tile of bs + w - 1 cells.
#pragma once

#include <cuda_runtime.h>

#include "esn_internal.h"

namespace esn {

template <typename T>
struct Cx;
template <>
struct Cx<double> {
    using type = double2;
};
template <>
struct Cx<float> {
    using type = float2;
};

// ---------------------------------------------------------------------------
// Kernel rows (spreadinterp.py:313-336): the w ordinates of one coordinate,
// by Horner on the piecewise polynomial (all pieces share t) or by exact
// exp/sqrt.  The Horner table lives in the kernel parameter bank; with W a
// compile-time constant every coefficient is a uniform constant operand.
template <typename T, int W>
__device__ __forceinline__ int kernel_row(T g, const KernelTab<T> &k, T *row) {
    int i0 = (int)floor(g - (T)(0.5 * W) + (T)1);
    if (k.use_exact) {
        const T step = (T)2 / (T)W;
        T z = step * ((T)i0 - g);
#pragma unroll
        for (int m = 0; m < W; ++m) {
            T a = (T)1 - z * z;
            a = a < (T)0 ? (T)0 : a;
            row[m] = exp(k.beta * (sqrt(a) - (T)1));
            z += step;
        }
    } else {
        const T t = (T)2 * ((T)i0 - g) + (T)(W - 1);
#pragma unroll
        for (int m = 0; m < W; ++m) {
            T v = k.coef[m * (W + 4)];
#pragma unroll
            for (int q = 1; q < W + 4; ++q) v = fma(v, t, k.coef[m * (W + 4) + q]);
            row[m] = v;
        }
    }
    return i0;
}

__device__ __forceinline__ int wrap_once(int i, int n) {
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

__device__ __forceinline__ void flag_min(unsigned long long *f, unsigned long long v) {
    atomicMin(f, v);
}

__device__ __forceinline__ void red_add(double2 *p, double2 v) {
    atomicAdd(&p->x, v.x);
    atomicAdd(&p->y, v.y);
}
__device__ __forceinline__ void red_add(float2 *p, float2 v) {
    atomicAdd(p, v);  // sm_90+: one vector RED.F32x2 per complex cell
}

template <typename T>
__device__ __forceinline__ bool finite2(typename Cx<T>::type v) {
    return isfinite(v.x) && isfinite(v.y);
}

// ---------------------------------------------------------------------------
// Global-atomic spreader: one thread per sorted point, w^d complex REDs
// straight into the fine grid (rows reused across the ntransf batch).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256) k_spread_global(SpreadArgs<T> a) {
    using C = typename Cx<T>::type;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.M;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int j = a.perm[k];
        T r1[W], r2[W], r3[W];
        int ix1[W], ix2[W], ix3[W];
        int i1 = kernel_row<T, W>(a.gs[0][k], a.k, r1);
#pragma unroll
        for (int m = 0; m < W; ++m) ix1[m] = wrap_once(i1 + m, n1);
        if (DIM > 1) {
            int i2 = kernel_row<T, W>(a.gs[1][k], a.k, r2);
#pragma unroll
            for (int m = 0; m < W; ++m) ix2[m] = wrap_once(i2 + m, n2);
        }
        if (DIM > 2) {
            int i3 = kernel_row<T, W>(a.gs[2][k], a.k, r3);
#pragma unroll
            for (int m = 0; m < W; ++m) ix3[m] = wrap_once(i3 + m, n3);
        }
        for (int t = 0; t < a.ntransf; ++t) {
            C c = reinterpret_cast<const C *>(a.c)[(int64_t)t * a.M + j];
            if (!finite2<T>(c)) flag_min(&a.flags[6], (unsigned long long)j);
            C *grid = reinterpret_cast<C *>(a.grid) + (int64_t)t * a.gstride;
            if (DIM == 1) {
#pragma unroll
                for (int m1 = 0; m1 < W; ++m1) red_add(grid + ix1[m1], C{c.x * r1[m1], c.y * r1[m1]});
            } else if (DIM == 2) {
#pragma unroll
                for (int m2 = 0; m2 < W; ++m2) {
                    C v{c.x * r2[m2], c.y * r2[m2]};
                    int64_t base = (int64_t)ix2[m2] * n1;
#pragma unroll
                    for (int m1 = 0; m1 < W; ++m1) red_add(grid + base + ix1[m1], C{v.x * r1[m1], v.y * r1[m1]});
                }
            } else {
#pragma unroll 1
                for (int m3 = 0; m3 < W; ++m3) {
                    C v3{c.x * r3[m3], c.y * r3[m3]};
#pragma unroll
                    for (int m2 = 0; m2 < W; ++m2) {
                        C v{v3.x * r2[m2], v3.y * r2[m2]};
                        int64_t base = ((int64_t)ix3[m3] * n2 + ix2[m2]) * n1;
#pragma unroll
                        for (int m1 = 0; m1 < W; ++m1)
                            red_add(grid + base + ix1[m1], C{v.x * r1[m1], v.y * r1[m1]});
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Tile spreader (one CTA per subproblem, persistent over a work queue): the
// bin's tile of (bs + w - 1)^d cells is accumulated in shared memory, then
// flushed to the periodic fine grid with one RED per tile cell.  Points are
// staged in chunks: phase A evaluates kernel rows (one thread per point),
// phase B lets each warp add one point at a time with lanes covering the
// w^d footprint cells (distinct cells per lane).
template <typename T, int DIM, int W>
struct TileCfg {
    static constexpr int CH = 64;  // points per staging chunk
    static constexpr int NT = 256;
};

template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256) k_spread_tile(SpreadArgs<T> a) {
    using C = typename Cx<T>::type;
    constexpr int CH = TileCfg<T, DIM, W>::CH;
    constexpr int FP = (DIM == 1 ? W : (DIM == 2 ? W * W : W * W * W));
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int T1 = a.g.bs[0] + W - 1;
    const int T2 = DIM > 1 ? a.g.bs[1] + W - 1 : 1;
    const int T3 = DIM > 2 ? a.g.bs[2] + W - 1 : 1;
    const int ncell = T1 * T2 * T3;
    C *tile = reinterpret_cast<C *>(smem_raw);
    T *rows = reinterpret_cast<T *>(tile + ncell);            // CH x DIM x W
    C *cs = reinterpret_cast<C *>(rows + CH * DIM * W);        // CH
    int *offs = reinterpret_cast<int *>(cs + CH);              // CH x DIM
    __shared__ int s_sub;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    const int nsub = *a.nsub;
    for (;;) {
        if (tid == 0) s_sub = atomicAdd(a.work, 1);
        __syncthreads();
        const int s = s_sub;
        __syncthreads();
        if (s >= nsub) break;
        const int4 sp = a.subprob[s];
        const int bin = sp.x, start = sp.y, cnt = sp.z;
        const int b1 = bin % a.g.nb[0];
        const int b2 = DIM > 1 ? (bin / a.g.nb[0]) % a.g.nb[1] : 0;
        const int b3 = DIM > 2 ? bin / (a.g.nb[0] * a.g.nb[1]) : 0;
        const int lo1 = b1 * a.g.bs[0], lo2 = b2 * a.g.bs[1], lo3 = b3 * a.g.bs[2];
        for (int t = 0; t < a.ntransf; ++t) {
            for (int i = tid; i < ncell; i += blockDim.x) tile[i] = C{(T)0, (T)0};
            const C *cin = reinterpret_cast<const C *>(a.c) + (int64_t)t * a.M;
            for (int p0 = 0; p0 < cnt; p0 += CH) {
                const int nch = min(CH, cnt - p0);
                __syncthreads();
                if (tid < nch) {
                    const int k = start + p0 + tid;
                    const int j = a.perm[k];
                    T r[W];
                    int i0 = kernel_row<T, W>(a.gs[0][k], a.k, r);
                    offs[tid * DIM + 0] = (i0 < 0 ? i0 + n1 : i0) - lo1;
#pragma unroll
                    for (int m = 0; m < W; ++m) rows[(tid * DIM + 0) * W + m] = r[m];
                    if (DIM > 1) {
                        i0 = kernel_row<T, W>(a.gs[1][k], a.k, r);
                        offs[tid * DIM + 1] = (i0 < 0 ? i0 + n2 : i0) - lo2;
#pragma unroll
                        for (int m = 0; m < W; ++m) rows[(tid * DIM + 1) * W + m] = r[m];
                    }
                    if (DIM > 2) {
                        i0 = kernel_row<T, W>(a.gs[2][k], a.k, r);
                        offs[tid * DIM + 2] = (i0 < 0 ? i0 + n3 : i0) - lo3;
#pragma unroll
                        for (int m = 0; m < W; ++m) rows[(tid * DIM + 2) * W + m] = r[m];
                    }
                    C c = cin[j];
                    if (!finite2<T>(c)) flag_min(&a.flags[6], (unsigned long long)j);
                    cs[tid] = c;
                }
                __syncthreads();
                for (int q = warp; q < nch; q += nwarp) {
                    const C c = cs[q];
                    const T *rq = rows + q * DIM * W;
                    const int o1 = offs[q * DIM];
                    const int o2 = DIM > 1 ? offs[q * DIM + 1] : 0;
                    const int o3 = DIM > 2 ? offs[q * DIM + 2] : 0;
                    for (int f = lane; f < FP; f += 32) {
                        const int m1 = f % W;
                        const int m2 = DIM > 1 ? (f / W) % W : 0;
                        const int m3 = DIM > 2 ? f / (W * W) : 0;
                        T v = rq[m1];
                        if (DIM > 1) v *= rq[W + m2];
                        if (DIM > 2) v *= rq[2 * W + m3];
                        T *cell = reinterpret_cast<T *>(tile + ((o3 + m3) * T2 + (o2 + m2)) * T1 + (o1 + m1));
                        atomicAdd(cell, c.x * v);
                        atomicAdd(cell + 1, c.y * v);
                    }
                }
            }
            __syncthreads();
            C *grid = reinterpret_cast<C *>(a.grid) + (int64_t)t * a.gstride;
            for (int i = tid; i < ncell; i += blockDim.x) {
                const C v = tile[i];
                if (v.x == (T)0 && v.y == (T)0) continue;
                const int q1 = i % T1;
                const int q2 = DIM > 1 ? (i / T1) % T2 : 0;
                const int q3 = DIM > 2 ? i / (T1 * T2) : 0;
                int g1 = lo1 + q1;
                while (g1 >= n1) g1 -= n1;
                int64_t gi = g1;
                if (DIM > 1) {
                    int g2 = lo2 + q2;
                    while (g2 >= n2) g2 -= n2;
                    gi += (int64_t)g2 * n1;
                }
                if (DIM > 2) {
                    int g3 = lo3 + q3;
                    while (g3 >= n3) g3 -= n3;
                    gi += (int64_t)g3 * n2 * n1;
                }
                red_add(grid + gi, v);
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Interpolator (spreadinterp.py:442-507): one thread per sorted point,
// separable weighted gather of the w^d patch (periodic indices), output in
// ORIGINAL point order (out[perm[k]], spreadinterp.py:453).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256) k_interp_thread(SpreadArgs<T> a, T *cout, const T *gridp) {
    using C = typename Cx<T>::type;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.M;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int j = a.perm[k];
        T r1[W], r2[W], r3[W];
        int ix1[W], ix2[W], ix3[W];
        int i1 = kernel_row<T, W>(a.gs[0][k], a.k, r1);
#pragma unroll
        for (int m = 0; m < W; ++m) ix1[m] = wrap_once(i1 + m, n1);
        if (DIM > 1) {
            int i2 = kernel_row<T, W>(a.gs[1][k], a.k, r2);
#pragma unroll
            for (int m = 0; m < W; ++m) ix2[m] = wrap_once(i2 + m, n2);
        }
        if (DIM > 2) {
            int i3 = kernel_row<T, W>(a.gs[2][k], a.k, r3);
#pragma unroll
            for (int m = 0; m < W; ++m) ix3[m] = wrap_once(i3 + m, n3);
        }
        for (int t = 0; t < a.ntransf; ++t) {
            const C *grid = reinterpret_cast<const C *>(gridp) + (int64_t)t * a.gstride;
            T are = 0, aim = 0;
            if (DIM == 1) {
#pragma unroll
                for (int m1 = 0; m1 < W; ++m1) {
                    C v = __ldg(grid + ix1[m1]);
                    are = fma(r1[m1], v.x, are);
                    aim = fma(r1[m1], v.y, aim);
                }
            } else if (DIM == 2) {
#pragma unroll
                for (int m2 = 0; m2 < W; ++m2) {
                    const C *row = grid + (int64_t)ix2[m2] * n1;
                    T pre = 0, pim = 0;
#pragma unroll
                    for (int m1 = 0; m1 < W; ++m1) {
                        C v = __ldg(row + ix1[m1]);
                        pre = fma(r1[m1], v.x, pre);
                        pim = fma(r1[m1], v.y, pim);
                    }
                    are = fma(r2[m2], pre, are);
                    aim = fma(r2[m2], pim, aim);
                }
            } else {
#pragma unroll 1
                for (int m3 = 0; m3 < W; ++m3) {
                    T p3re = 0, p3im = 0;
#pragma unroll
                    for (int m2 = 0; m2 < W; ++m2) {
                        const C *row = grid + ((int64_t)ix3[m3] * n2 + ix2[m2]) * n1;
                        T pre = 0, pim = 0;
#pragma unroll
                        for (int m1 = 0; m1 < W; ++m1) {
                            C v = __ldg(row + ix1[m1]);
                            pre = fma(r1[m1], v.x, pre);
                            pim = fma(r1[m1], v.y, pim);
                        }
                        p3re = fma(r2[m2], pre, p3re);
                        p3im = fma(r2[m2], pim, p3im);
                    }
                    are = fma(r3[m3], p3re, are);
                    aim = fma(r3[m3], p3im, aim);
                }
            }
            reinterpret_cast<C *>(cout)[(int64_t)t * a.M + j] = C{are, aim};
        }
    }
}

// ---------------------------------------------------------------------------
// Type-1 deconvolution / mode copy (transforms.py:165-171): out[k] =
// p1[k1] p2[k2] p3[k3] * FFT[k mod n], one thread per output mode, k1
// fastest so both the gather (two contiguous runs per row) and the store
// are coalesced.
template <typename T>
__global__ void k_deconv(int ntransf, int n1, int n2, int n3, int64_t N1, int64_t N2, int64_t N3,
                         const T *grid, const T *p1, const T *p2, const T *p3, T *f) {
    using C = typename Cx<T>::type;
    const int64_t per = N1 * N2 * N3, total = per * ntransf, G = (int64_t)n1 * n2 * n3;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = idx / per;
        int64_t r = idx - t * per;
        const int64_t k1i = r % N1;
        r /= N1;
        const int64_t k2i = r % N2;
        const int64_t k3i = r / N2;
        int64_t k1 = k1i - N1 / 2, k2 = k2i - N2 / 2, k3 = k3i - N3 / 2;
        if (k1 < 0) k1 += n1;
        if (k2 < 0) k2 += n2;
        if (k3 < 0) k3 += n3;
        T fac = p1[k1i];
        if (p2) fac *= p2[k2i];
        if (p3) fac *= p3[k3i];
        const C v = reinterpret_cast<const C *>(grid)[t * G + (k3 * n2 + k2) * n1 + k1];
        reinterpret_cast<C *>(f)[idx] = C{v.x * fac, v.y * fac};
    }
}

// Type-2 amplify + zero pad (transforms.py:194-200): writes the whole fine
// grid in one pass, p_k f_k at bins k mod n and zeros elsewhere.  Also the
// finiteness check of the mode coefficients (transforms.py:190).
template <typename T>
__global__ void k_amplify(int ntransf, int n1, int n2, int n3, int64_t N1, int64_t N2, int64_t N3,
                          const T *f, const T *p1, const T *p2, const T *p3, T *grid,
                          unsigned long long *flag) {
    using C = typename Cx<T>::type;
    const int64_t G = (int64_t)n1 * n2 * n3, total = G * ntransf, per = N1 * N2 * N3;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = idx / G;
        int64_t r = idx - t * G;
        const int64_t l1 = r % n1;
        r /= n1;
        const int64_t l2 = r % n2;
        const int64_t l3 = r / n2;
        // bin l -> centered mode k: k = l for l <= N - N/2 - 1, l - n for l >= n - N/2
        auto mode = [](int64_t l, int64_t n, int64_t N) -> int64_t {
            if (l <= N - N / 2 - 1) return l + N / 2;
            if (l >= n - N / 2) return l - n + N / 2;
            return -1;
        };
        const int64_t m1 = mode(l1, n1, N1), m2 = mode(l2, n2, N2), m3 = mode(l3, n3, N3);
        C out{(T)0, (T)0};
        if (m1 >= 0 && m2 >= 0 && m3 >= 0) {
            const int64_t fi = t * per + (m3 * N2 + m2) * N1 + m1;
            const C v = reinterpret_cast<const C *>(f)[fi];
            if (!finite2<T>(v)) flag_min(flag, (unsigned long long)fi);
            T fac = p1[m1];
            if (p2) fac *= p2[m2];
            if (p3) fac *= p3[m3];
            out = C{v.x * fac, v.y * fac};
        }
        reinterpret_cast<C *>(grid)[idx] = out;
    }
}

// ---------------------------------------------------------------------------
// dispatch helpers
template <typename T, template <typename, int, int> class Op, typename... Args>
int dispatch_dw(int dim, int w, Args &&...args) {
#define ESN_CASE_W(D, WW) \
    case WW:              \
        return Op<T, D, WW>::run(args...);
#define ESN_CASES(D)                                                                                    \
    switch (w) {                                                                                        \
        ESN_CASE_W(D, 2) ESN_CASE_W(D, 3) ESN_CASE_W(D, 4) ESN_CASE_W(D, 5) ESN_CASE_W(D, 6)            \
        ESN_CASE_W(D, 7) ESN_CASE_W(D, 8) ESN_CASE_W(D, 9) ESN_CASE_W(D, 10) ESN_CASE_W(D, 11)          \
        ESN_CASE_W(D, 12) ESN_CASE_W(D, 13) ESN_CASE_W(D, 14) ESN_CASE_W(D, 15) ESN_CASE_W(D, 16)       \
        default:                                                                                        \
            return fail(ESN_INTERNAL_ERROR, "unsupported kernel width %d", w);                          \
    }
    if (dim == 1) {
        ESN_CASES(1)
    } else if (dim == 2) {
        ESN_CASES(2)
    } else {
        ESN_CASES(3)
    }
#undef ESN_CASES
#undef ESN_CASE_W
}

}  // namespace esn
