// esn_device.cuh -- sm_100a device code of the B200 ES-kernel NUFFT core:
// kernel-row evaluation, spreaders, interpolator, deconvolution and mode
// amplification.  Instantiated per precision by esn_inst_f64.cu / _f32.cu.
//
// Data layout in HBM:
//  * sorted point records rec[k] = {g_1, g_2, g_3, j} (grid coordinates in
//    the plan dtype + original index), 32 B for float64 plans and 16 B for
//    float32 plans -- one aligned sector-sized record per point, written once
//    by setpts and read coalesced by the spreader / interpolator;
//  * strengths c (ntransf, M) and fine grids (ntransf, n3, n2, n1) as
//    interleaved complex of the plan dtype (C order, dimension 1 fastest);
//  * bins are boxes of footprint origins i0 = floor(g - w/2 + 1) (wrapped
//    into [0, n)); a bin of bs cells owns a tile of bs + w - 1 cells.
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
// Exact kernel row (spreadinterp.py:319-327), kept out of line: it is the
// validation path (use_exact_kernel) and would otherwise bloat every kernel.
template <typename T>
__device__ __noinline__ void exact_row(double g, int i0, int W, T beta, T *row) {
    const T step = (T)2 / (T)W;
    T z = (T)((2.0 / W) * ((double)i0 - g));
    for (int m = 0; m < W; ++m) {
        T a = (T)1 - z * z;
        a = a < (T)0 ? (T)0 : a;
        row[m] = exp(beta * (sqrt(a) - (T)1));
        z += step;
    }
}

#ifndef ESN_HORNER_SYM
#define ESN_HORNER_SYM 1
#endif
template <typename T, int W>
__device__ __forceinline__ int kernel_row(double g, const KernelTab<T> &k, T *row) {
    // footprint origin and local coordinate in float64 exactly as the
    // reference (spreadinterp.py:318, 329), then the plan dtype
    const int i0 = (int)floor(g - 0.5 * W + 1.0);
    if (k.use_exact) {
        // the out-of-line call writes a private scratch row; copying it keeps
        // the caller's row[] in registers (passing row itself would force it
        // to the stack on the hot Horner path as well)
        T tmp[W];
        exact_row<T>(g, i0, W, k.beta, tmp);
#pragma unroll
        for (int m = 0; m < W; ++m) row[m] = tmp[m];
    } else {
        const T t = (T)(2.0 * ((double)i0 - g) + (double)(W - 1));
#if ESN_HORNER_SYM
        // The ES kernel is even, so piece W-1-m is piece m mirrored:
        // p_{W-1-m}(t) = p_m(-t) (the fitted table is symmetric to ~3e-16).
        // With p_m(t) = E(t^2) + t O(t^2) the pair costs two half-length
        // Horner chains in t^2 plus two FMAs: (W+4) + 2 operations instead
        // of 2 (W+3) -- 62 instead of 108 FP64 operations per 2D point at w = 6.
        constexpr int NC = W + 4;        // coefficients per piece, highest degree first
        const T s2 = t * t;
#pragma unroll
        for (int m = 0; m < (W + 1) / 2; ++m) {
            // coefficient q multiplies t^(NC-1-q); split by the parity of the power
            constexpr int QE = (NC - 1) % 2 == 0 ? 0 : 1;  // first even-power coefficient
            constexpr int QO = 1 - QE;                      // first odd-power coefficient
            T e = k.coef[m * NC + QE];
#pragma unroll
            for (int q = QE + 2; q < NC; q += 2) e = fma(e, s2, k.coef[m * NC + q]);
            T o = k.coef[m * NC + QO];
#pragma unroll
            for (int q = QO + 2; q < NC; q += 2) o = fma(o, s2, k.coef[m * NC + q]);
            row[m] = fma(t, o, e);
            if (W - 1 - m != m) row[W - 1 - m] = fma(-t, o, e);
        }
#else
#pragma unroll
        for (int m = 0; m < W; ++m) {
            T v = k.coef[m * (W + 4)];
#pragma unroll
            for (int q = 1; q < W + 4; ++q) v = fma(v, t, k.coef[m * (W + 4) + q]);
            row[m] = v;
        }
#endif
    }
    return i0;
}

// Lane-parallel row evaluation: a lane that always evaluates ordinate m
// (runtime) keeps piece m's Horner coefficients in registers (loaded once per
// kernel by kernel_col), then evaluates one ordinate per coordinate.
template <typename T, int W>
__device__ __forceinline__ void kernel_col(const KernelTab<T> &k, int m, T *cf) {
#pragma unroll
    for (int q = 0; q < W + 4; ++q) cf[q] = (T)0;
#pragma unroll
    for (int p = 0; p < W; ++p) {
        if (p == m) {
#pragma unroll
            for (int q = 0; q < W + 4; ++q) cf[q] = k.coef[p * (W + 4) + q];
        }
    }
}

template <typename T, int W>
__device__ __forceinline__ T kernel_one(double g, int m, const T *cf, const KernelTab<T> &k, int *i0out) {
    const int i0 = (int)floor(g - 0.5 * W + 1.0);
    *i0out = i0;
    if (k.use_exact) {
        const T z = (T)((2.0 / W) * ((double)(i0 + m) - g));
        T a = (T)1 - z * z;
        a = a < (T)0 ? (T)0 : a;
        return exp(k.beta * (sqrt(a) - (T)1));
    }
    const T t = (T)(2.0 * ((double)i0 - g) + (double)(W - 1));
    T v = cf[0];
#pragma unroll
    for (int q = 1; q < W + 4; ++q) v = fma(v, t, cf[q]);
    return v;
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

// acc + v * w and v * w on an interleaved complex value.  float32: one packed
// FFMA2 / FMUL2 (fma.rn.f32x2, sm_100+: the scalar w is a broadcast operand in
// SASS) -- the same FMA-pipe time as two FFMAs in half the issue slots; each
// lane of the pair rounds like fmaf, so results are unchanged.
__device__ __forceinline__ float2 cfma(float2 v, float w, float2 acc) {
    const float2 ww = make_float2(w, w);
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const unsigned long long *>(&v)), "l"(*reinterpret_cast<const unsigned long long *>(&ww)),
          "l"(*reinterpret_cast<const unsigned long long *>(&acc)));
    return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 cmul(float2 v, float w) {
    const float2 ww = make_float2(w, w);
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const unsigned long long *>(&v)), "l"(*reinterpret_cast<const unsigned long long *>(&ww)));
    return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ double2 cfma(double2 v, double w, double2 acc) {
    return double2{fma(v.x, w, acc.x), fma(v.y, w, acc.y)};
}
__device__ __forceinline__ double2 cmul(double2 v, double w) { return double2{v.x * w, v.y * w}; }

template <typename T>
__device__ __forceinline__ bool finite2(typename Cx<T>::type v) {
    return isfinite(v.x) && isfinite(v.y);
}

// One 256-bit read-only load per record (LDG.E.ENL2.256).
__device__ __forceinline__ Rec load_rec(const Rec *r, int64_t k) {
    unsigned long long a, b, c, d;
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(r + k));
    Rec out;
    out.g[0] = __longlong_as_double((long long)a);
    out.g[1] = __longlong_as_double((long long)b);
    out.g[2] = __longlong_as_double((long long)c);
    out.j = (int)(d & 0xffffffffull);
    out.pad = 0;
    return out;
}

// Ampere-style asynchronous global -> shared copies (LDGSTS): no registers
// are held while the bytes are in flight; completion per thread by group.
__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(g)
                 : "memory");
}
// the same with an L2 eviction-policy hint (createpolicy): records that
// stream through once go evict-first, gathered strengths evict-last so the
// other values of each 32-byte sector are still in L2 when their points come
__device__ __forceinline__ void cp_async16_hint(void *smem, const void *g, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(g), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async8_hint(void *smem, const void *g, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(g), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------------------
// Global-atomic spreader: one thread per sorted point, w^d complex REDs
// straight into the fine grid (rows reused across the ntransf batch).  Used
// for 1D (where a point's footprint is a single contiguous run).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256) k_spread_global(SpreadArgs<T> a) {
    using C = typename Cx<T>::type;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.M;
         k += (int64_t)gridDim.x * blockDim.x) {
        const Rec rc = load_rec(a.rec, k);
        const int j = rc.j;
        T r1[W], r2[W], r3[W];
        int ix1[W], ix2[W], ix3[W];
        int i1 = kernel_row<T, W>(rc.g[0], a.k, r1);
#pragma unroll
        for (int m = 0; m < W; ++m) ix1[m] = wrap_once(i1 + m, n1);
        if (DIM > 1) {
            int i2 = kernel_row<T, W>(rc.g[1], a.k, r2);
#pragma unroll
            for (int m = 0; m < W; ++m) ix2[m] = wrap_once(i2 + m, n2);
        }
        if (DIM > 2) {
            int i3 = kernel_row<T, W>(rc.g[2], a.k, r3);
#pragma unroll
            for (int m = 0; m < W; ++m) ix3[m] = wrap_once(i3 + m, n3);
        }
        for (int t = 0; t < a.ntransf; ++t) {
            C c = reinterpret_cast<const C *>(a.c)[(int64_t)t * a.M + j];
            if (!finite2<T>(c)) flag_min(&a.flags[6], (unsigned long long)(j + a.ibase));
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
                    const int iz = wrap_once(ix3[0] + m3, n3);
#pragma unroll
                    for (int m2 = 0; m2 < W; ++m2) {
                        C v{v3.x * r2[m2], v3.y * r2[m2]};
                        int64_t base = ((int64_t)iz * n2 + ix2[m2]) * n1;
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
// Row spreader (2D / 3D).  One CTA per subproblem (persistent over a work
// queue).  Every thread OWNS one x-row of the bin's tile (rows indexed by
// (y, z) in the tile) and accumulates it in registers: acc[X] with
// X = BX + W - 1.  For each staged point the warps whose row block meets the
// point's w x w row footprint add c * r2[dy] * r3[dz] * r1[m] into
// acc[ox + m]; the x offset ox is warp-uniform, so a switch over its BX values
// gives static register indices.  No shared-memory atomics: the only atomics
// are the final coalesced REDs of the tile (staged through shared memory)
// into the periodic fine grid.
//
// Thread layout: 3D -- warps are 8 (y) x 4 (z) row blocks over a RY x RZ
// row grid; 2D -- warps are 32 consecutive y rows.
template <typename T, int DIM, int W>
__device__ __forceinline__ void rows_accumulate(typename Cx<T>::type *acc, int ox,
                                                typename Cx<T>::type v, const T *r1) {
    constexpr int BX = RowsCfg<T, DIM, W>::BX;
    // one flat switch (a single jump-table dispatch); cases >= BX are empty
#define ESN_ROWS_CASE(OX)                                          \
    case OX:                                                       \
        if constexpr (OX < BX) {                                   \
            _Pragma("unroll") for (int m = 0; m < W; ++m) {        \
                const T r = r1[m];                                 \
                acc[OX + m].x = fma(v.x, r, acc[OX + m].x);        \
                acc[OX + m].y = fma(v.y, r, acc[OX + m].y);        \
            }                                                      \
        }                                                          \
        break;
    switch (ox) {
        ESN_ROWS_CASE(0) ESN_ROWS_CASE(1) ESN_ROWS_CASE(2) ESN_ROWS_CASE(3)
        ESN_ROWS_CASE(4) ESN_ROWS_CASE(5) ESN_ROWS_CASE(6) ESN_ROWS_CASE(7)
        ESN_ROWS_CASE(8) ESN_ROWS_CASE(9) ESN_ROWS_CASE(10) ESN_ROWS_CASE(11)
        ESN_ROWS_CASE(12) ESN_ROWS_CASE(13) ESN_ROWS_CASE(14) ESN_ROWS_CASE(15)
        ESN_ROWS_CASE(16) ESN_ROWS_CASE(17) ESN_ROWS_CASE(18) ESN_ROWS_CASE(19)
        ESN_ROWS_CASE(20) ESN_ROWS_CASE(21) ESN_ROWS_CASE(22) ESN_ROWS_CASE(23)
        ESN_ROWS_CASE(24) ESN_ROWS_CASE(25) ESN_ROWS_CASE(26) ESN_ROWS_CASE(27)
        ESN_ROWS_CASE(28) ESN_ROWS_CASE(29) ESN_ROWS_CASE(30) ESN_ROWS_CASE(31)
        default:
            break;
    }
#undef ESN_ROWS_CASE
}

template <typename T, int DIM, int W>
__global__ void __launch_bounds__(RowsCfg<T, DIM, W>::NT, RowsCfg<T, DIM, W>::MINB) k_spread_rows(SpreadArgs<T> a) {
    using C = typename Cx<T>::type;
    using Cfg = RowsCfg<T, DIM, W>;
    constexpr int X = Cfg::X, RY = Cfg::RY, RZ = Cfg::RZ, CH = Cfg::CH, NT = Cfg::NT;
    constexpr int NW = NT / 32;                 // warps = row blocks
    constexpr int WBY = DIM == 3 ? 8 : 32;      // row-block extent in y
    constexpr int WBZ = DIM == 3 ? 4 : 1;       // row-block extent in z
    constexpr int NWY = RY / WBY;
    constexpr int NZ = DIM == 3 ? W : 1;        // entries of the (c * r3) table
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // staging per point (one thread each): c * r3[m] (complex, NZ), r2[W],
    // r1[W], offsets (ox, oy, oz); per warp the list of staged points whose
    // row footprint meets its block
    C *s_cz = reinterpret_cast<C *>(smem_raw);                    // CH x NZ
    T *s_r2 = reinterpret_cast<T *>(s_cz + CH * NZ);              // CH x W
    T *s_r1 = s_r2 + CH * W;                                      // CH x W
    int *s_o = reinterpret_cast<int *>(s_r1 + CH * W);            // CH x 4
    unsigned char *s_list = reinterpret_cast<unsigned char *>(s_o + CH * 4);  // NW x CH
    C *s_tile = reinterpret_cast<C *>(smem_raw);                  // reused for the flush: RY*RZ x X
    __shared__ int s_sub;
    __shared__ int s_cnt[NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wy = warp % NWY, wz = warp / NWY;
    const int ry = wy * WBY + (DIM == 3 ? (lane & 7) : lane);
    const int rz = DIM == 3 ? wz * WBZ + (lane >> 3) : 0;
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
        const int b2 = (bin / a.g.nb[0]) % a.g.nb[1];
        const int b3 = DIM > 2 ? bin / (a.g.nb[0] * a.g.nb[1]) : 0;
        const int lo1 = b1 * a.g.bs[0], lo2 = b2 * a.g.bs[1], lo3 = b3 * a.g.bs[2];
        for (int t = 0; t < a.ntransf; ++t) {
            C acc[X];
#pragma unroll
            for (int x = 0; x < X; ++x) acc[x] = C{(T)0, (T)0};
            const C *cin = reinterpret_cast<const C *>(a.c) + (int64_t)t * a.M;
            // chunk ci stages points ci, ci + nck, ... of the subproblem: the
            // sort is fine (sub-cell order), so strided chunks sample the whole
            // bin and keep every row block busy
            const int nck = (cnt + CH - 1) / CH;
            for (int ci = 0; ci < nck; ++ci) {
                const int nch = (cnt - ci + nck - 1) / nck;
                __syncthreads();
                if (tid < NW) s_cnt[tid] = 0;
                __syncthreads();
                if (tid < nch) {  // phase A: one thread per staged point
                    const Rec rc = load_rec(a.rec, start + ci + tid * nck);
                    C c = cin[rc.j];
                    if (!finite2<T>(c)) flag_min(&a.flags[6], (unsigned long long)(rc.j + a.ibase));
                    T r[W];
                    int i0 = kernel_row<T, W>(rc.g[0], a.k, r);
                    const int ox = (i0 < 0 ? i0 + n1 : i0) - lo1;
#pragma unroll
                    for (int m = 0; m < W; ++m) s_r1[tid * W + m] = r[m];
                    i0 = kernel_row<T, W>(rc.g[1], a.k, r);
                    const int oy = (i0 < 0 ? i0 + n2 : i0) - lo2;
#pragma unroll
                    for (int m = 0; m < W; ++m) s_r2[tid * W + m] = r[m];
                    int oz = 0;
                    if (DIM > 2) {
                        i0 = kernel_row<T, W>(rc.g[2], a.k, r);
                        oz = (i0 < 0 ? i0 + n3 : i0) - lo3;
#pragma unroll
                        for (int m = 0; m < W; ++m) s_cz[tid * NZ + m] = C{c.x * r[m], c.y * r[m]};
                    } else {
                        s_cz[tid] = c;
                    }
                    *reinterpret_cast<int4 *>(s_o + tid * 4) = make_int4(ox, oy, oz, 0);
                    // enqueue this point for every row block its w x w rows meet
                    const int y0 = oy / WBY, y1 = (oy + W - 1) / WBY;
                    const int z0 = DIM > 2 ? oz / WBZ : 0, z1 = DIM > 2 ? (oz + W - 1) / WBZ : 0;
                    for (int zz = z0; zz <= z1; ++zz)
                        for (int yy = y0; yy <= y1; ++yy) {
                            const int wb = zz * NWY + yy;
                            const int slot = atomicAdd(&s_cnt[wb], 1);
                            s_list[wb * CH + slot] = (unsigned char)tid;
                        }
                }
                __syncthreads();
                // phase B: the row owners of each block accumulate in registers
                const int nq = s_cnt[warp];
                for (int i = 0; i < nq; ++i) {
                    const int q = s_list[warp * CH + i];
                    const int4 o = *reinterpret_cast<const int4 *>(s_o + q * 4);
                    const int dy = ry - o.y, dz = rz - o.z;
                    const bool cov = dy >= 0 && dy < W && (DIM < 3 || (dz >= 0 && dz < W));
                    const T f = cov ? s_r2[q * W + dy] : (T)0;
                    const C cz = s_cz[q * NZ + ((DIM > 2 && cov) ? dz : 0)];
                    const C v{cz.x * f, cz.y * f};
                    T r1[W];
#pragma unroll
                    for (int m = 0; m < W; ++m) r1[m] = s_r1[q * W + m];
                    rows_accumulate<T, DIM, W>(acc, o.x, v, r1);
                }
            }
            // flush: stage the owned rows in shared memory, then coalesced REDs
            __syncthreads();
            const int nrow = RY * RZ;
            const int myrow = rz * RY + ry;
#pragma unroll
            for (int x = 0; x < X; ++x) s_tile[myrow * X + x] = acc[x];
            __syncthreads();
            C *grid = reinterpret_cast<C *>(a.grid) + (int64_t)t * a.gstride;
            for (int i = tid; i < nrow * X; i += NT) {
                const C v = s_tile[i];
                if (v.x == (T)0 && v.y == (T)0) continue;
                const int row = i / X, x = i - row * X;
                const int yy = row % RY, zz = row / RY;
                int g1 = lo1 + x;
                while (g1 >= n1) g1 -= n1;
                int g2 = lo2 + yy;
                while (g2 >= n2) g2 -= n2;
                int64_t gi = (int64_t)g2 * n1 + g1;
                if (DIM > 2) {
                    int g3 = lo3 + zz;
                    while (g3 >= n3) g3 -= n3;
                    gi += (int64_t)g3 * n2 * n1;
                }
                red_add(grid + gi, v);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 3D row spreader, pipelined ("rows3").  Same register ownership as
// k_spread_rows (thread = one x-row of the bin tile, warps = 8 y x 4 z row
// blocks), restructured around three measured costs of that kernel (c3 ncu:
// 61 issue slots per (point, warp) pair for 16 FP64 ops, 24 % barrier and
// exposed load latency in phase A):
//  * the sort key inside a 3D bin is the x cell of the footprint origin only
//    (plan: sbl = {0, inf, inf}), so a CONTIGUOUS chunk of the bin is ordered
//    by x offset: each warp's list of covering points is a sequence of runs
//    of equal ox, and the ox dispatch (static register window) is one switch
//    per run instead of one per point;
//  * a point's staged record (r1, r2 + a zero, c * r3, offsets) is one padded
//    AoS block: every phase-B load is a broadcast or a conflict-free gather
//    with an immediate offset, coverage is folded into the r2 index (uncovered
//    rows read the zero), no per-lane predication;
//  * phase A of chunk k + 1 (records + strength gather by cp.async two / one
//    chunk ahead, Horner rows) runs after phase B of chunk k behind ONE barrier
//    per chunk; lists are built per warp by ballot compaction (no atomics).
// Warp-list entry of the 3D row spreader.  Wide (default): four words --
// the packed word (record offset / 16 | ox << 16 | last-of-run << 31), then
// the BYTE offsets of the lane-relative r2 operand, the c * r3 operand and the
// record, ready to add to the lane's bases: a pass spends 2 integer adds on
// addresses instead of ~8 shifts / masks on a two-word packed entry
// (ESN_R3_WIDE=0 keeps the packed entry).
#ifndef ESN_R3_WIDE
#define ESN_R3_WIDE 1
#endif
#if ESN_R3_WIDE
using Rows3Entry = uint4;
#else
using Rows3Entry = uint2;
#endif

template <typename T, int W>
struct Rows3Cfg {
    using R = Rows3Geo<T, W>;
    static constexpr int BX = R::BX, X = R::X, RY = R::RY, RZ = R::RZ, NT = R::NT, MINB = NT == 512 ? 1 : 2;
    static constexpr int LY = R::LY, LZ = R::LZ, WY = R::WY, WZ = R::WZ;
    static constexpr int NW = NT / 32;
    static constexpr int VT = 16 / (int)sizeof(T);                // T per 16-byte vector
    static constexpr int OFN = VT;                                // (oy, oz, ox, pad) ints
    static constexpr int R1N = (W + VT - 1) / VT * VT;           // r1, whole vectors
    // thin tile: r2 and c * r3 zero-padded over every (dy, dz) a listed point
    // can meet (dy in [-(LY-1), LY+W-2], dz in [-(BZ-1), LZ-1]), so the
    // pass indexes them with no coverage test; square tile: r2 + one zero
    static constexpr bool PAD = true;
    static constexpr int PY = LY - 1;                             // index biases
    static constexpr int PZ = (LZ - 1 < R::BZ - 1) ? LZ - 1 : R::BZ - 1;
    static constexpr int R2E = PAD ? 2 * LY + W - 2 : W + 1;      // r2 entries
    static constexpr int CZE = !PAD ? W : (R::WZ == 1 ? PZ + LZ : PZ + LZ + W - 1);  // c * r3 entries (complex)
    static constexpr int R2N = (R2E + VT - 1) / VT * VT;
    static constexpr int CZN = 2 * CZE;
    static constexpr int O_R1 = OFN, O_R2 = OFN + R1N, O_CZ = OFN + R1N + R2N;
    static constexpr int RECN = (O_CZ + CZN + VT - 1) / VT * VT;
    // stride: an ODD number of 16-byte units keeps the phase-A vector stores
    // of a quarter-warp's eight records on distinct bank groups (an even
    // count made them 2-way conflicts: 7.5 wavefronts per STS.128 in the
    // source-level ncu view of fp64 w = 7, whose 42 doubles got a pad to 44)
    static constexpr int RECS = ((RECN / VT) % 2 == 1) ? RECN : RECN + VT;
    // points per chunk: 128 (64 for the widest records), trimmed in steps of
    // 4 when that keeps two CTAs per SM with the four-word list entries
    // (fp64 w = 7: 124)
    static constexpr size_t smem_for(int ch) {
        return (size_t)2 * ch * RECS * sizeof(T) + (size_t)2 * ch * sizeof(Rec) + (size_t)ch * 2 * sizeof(T) +
               (size_t)NW * ch * sizeof(Rows3Entry);
    }
    static constexpr int pick_ch() {
        const int ch0 = (2 * 128 * RECS * (int)sizeof(T) <= 100 * 1024) ? 128 : 64;
        const size_t budget = 233472 / 2 - 1024 - 128;  // two CTAs: 228 KB less the reserved KB and the static words
        if (MINB != 2 || smem_for(ch0) <= budget) return ch0;
        for (int ch = ch0 - 4; ch >= ch0 - 16; ch -= 4)
            if (smem_for(ch) <= budget) return ch;
        return ch0;
    }
    static constexpr int CH = pick_ch();
    static constexpr size_t STAGE_B = (size_t)CH * RECS * sizeof(T);
    static constexpr size_t RING_B = (size_t)2 * CH * sizeof(Rec);
    static constexpr size_t CRING_B = (size_t)CH * 2 * sizeof(T);
    static constexpr size_t LIST_B = (size_t)NW * CH * sizeof(Rows3Entry);
    static constexpr size_t SMEM = 2 * STAGE_B + RING_B + CRING_B + LIST_B;
    static_assert(2 * STAGE_B / 16 <= 0xffff && (RECS * sizeof(T)) % 16 == 0, "list entries address 16-byte units");
    static_assert(2 * STAGE_B / sizeof(T) + RECS + 128 <= 0xffff && O_CZ % 2 == 0, "operand indices fit 16 bits");
    static_assert(BX <= 32, "list entries pack ox in 5 bits");
    static constexpr int EBIAS = 64;  // operand-index bias of the list entries (> any oy, oz)
    static_assert(RY - W + 1 < EBIAS && RZ - W + 1 < EBIAS, "biased indices stay positive");
    static constexpr size_t TILE_B = (size_t)RY * RZ * X * 2 * sizeof(T);
    // flush passes over z slabs so one slab fits the two stages (the record
    // ring may still have copies in flight)
    static constexpr size_t FL_B = 2 * STAGE_B;
    static constexpr int FP = TILE_B <= FL_B ? 1 : (TILE_B <= 2 * FL_B ? 2 : (TILE_B <= 4 * FL_B ? 4 : 8));
};

// phase-B operands of one point, loaded one point ahead (software pipeline)
template <typename T>
struct Rows3Pre {
    typename Cx<T>::type cz;
    T f;
    unsigned off;  // record offset in bytes
};

// One warp-list entry (two words):
//   x = record offset in 16-byte units | ox << 16 | last-of-run << 31
//   y = (T index of r2[PY - oy] + EBIAS) | (complex index of cz[PZ - oz] + EBIAS) << 16
// so a lane's operands are base_f + sizeof(T) * (y & 0xffff) and
// base_cz + sizeof(C) * (y >> 16) with lane-constant bases (ry, rz folded in).
template <typename T, int W>
__device__ __forceinline__ Rows3Pre<T> rows3_load(const unsigned char *stage, Rows3Entry e,
                                                  const unsigned char *base_f, const unsigned char *base_cz) {
    using C = typename Cx<T>::type;
    Rows3Pre<T> p;
#if ESN_R3_WIDE
    p.off = e.w;  // record offset in bytes
    p.f = *reinterpret_cast<const T *>(base_f + e.y);
    p.cz = *reinterpret_cast<const C *>(base_cz + e.z);
#else
    p.off = 16u * (e.x & 0xffffu);
    p.f = *reinterpret_cast<const T *>(base_f + (unsigned)sizeof(T) * (e.y & 0xffffu));
    p.cz = *reinterpret_cast<const C *>(base_cz + (unsigned)sizeof(C) * (e.y >> 16));
#endif
    (void)stage;
    return p;
}

template <typename T, int W, int OX>
__device__ __forceinline__ void rows3_apply(typename Cx<T>::type *acc, const unsigned char *stage,
                                            const Rows3Pre<T> &p) {
    using C = typename Cx<T>::type;
    using Cfg = Rows3Cfg<T, W>;
    const T *rec = reinterpret_cast<const T *>(stage + p.off);
    const C v = cmul(p.cz, p.f);
    T r1[Cfg::R1N];
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int m = 0; m < Cfg::R1N; m += 2) {
            const double2 q = *reinterpret_cast<const double2 *>(rec + Cfg::O_R1 + m);
            r1[m] = q.x;
            r1[m + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int m = 0; m < Cfg::R1N; m += 4) {
            const float4 q = *reinterpret_cast<const float4 *>(rec + Cfg::O_R1 + m);
            r1[m] = q.x;
            r1[m + 1] = q.y;
            r1[m + 2] = q.z;
            r1[m + 3] = q.w;
        }
    }
#pragma unroll
    for (int m = 0; m < W; ++m) acc[OX + m] = cfma(v, r1[m], acc[OX + m]);
}

// one run of equal x offset OX from the warp list; bit 31 of an entry's first
// word marks the last point of its run (and of the list)
template <typename T, int W, int OX>
__device__ __forceinline__ int rows3_run(typename Cx<T>::type *acc, const unsigned char *stage, const Rows3Entry *list,
                                         int i, const unsigned char *base_f, const unsigned char *base_cz) {
    // float32: two points of the run per step (both points' operand loads in
    // flight before either's FMAs; c3f 1.65 -> 1.57 ms); float64 keeps one
    // (same time, fewer spills)
    if constexpr (sizeof(T) == 4) {
    for (;;) {
        const Rows3Entry e0 = list[i++];
        if (e0.x >> 31) {
            rows3_apply<T, W, OX>(acc, stage, rows3_load<T, W>(stage, e0, base_f, base_cz));
            break;
        }
        const Rows3Entry e1 = list[i++];
        const Rows3Pre<T> p0 = rows3_load<T, W>(stage, e0, base_f, base_cz);
        const Rows3Pre<T> p1 = rows3_load<T, W>(stage, e1, base_f, base_cz);
        rows3_apply<T, W, OX>(acc, stage, p0);
        rows3_apply<T, W, OX>(acc, stage, p1);
        if (e1.x >> 31) break;
    }
    } else {
    for (;;) {
        const Rows3Entry e = list[i++];
        rows3_apply<T, W, OX>(acc, stage, rows3_load<T, W>(stage, e, base_f, base_cz));
        if (e.x >> 31) break;
    }
    }
    return i;
}

template <typename T, int W, bool ROLL = false>
__global__ void __launch_bounds__(Rows3Cfg<T, W>::NT, Rows3Cfg<T, W>::MINB) k_spread_rows3(SpreadArgs<T> a) {
    using C = typename Cx<T>::type;
    using Cfg = Rows3Cfg<T, W>;
    constexpr int X = Cfg::X, RY = Cfg::RY, RZ = Cfg::RZ, CH = Cfg::CH, NT = Cfg::NT, RECS = Cfg::RECS;
    constexpr int BX = Cfg::BX;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *s_stage = reinterpret_cast<T *>(smem_raw);                                        // 2 x CH x RECS
    Rec *s_ring = reinterpret_cast<Rec *>(smem_raw + 2 * Cfg::STAGE_B);                  // 2 x CH
    C *s_c = reinterpret_cast<C *>(smem_raw + 2 * Cfg::STAGE_B + Cfg::RING_B);           // CH
    Rows3Entry *s_list = reinterpret_cast<Rows3Entry *>(smem_raw + 2 * Cfg::STAGE_B + Cfg::RING_B + Cfg::CRING_B);  // NW x CH
    C *s_tile = reinterpret_cast<C *>(smem_raw);  // flush slab (aliases the stages)
    __shared__ int s_sub;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int LY = Cfg::LY, LZ = Cfg::LZ, WY = Cfg::WY, WZ = Cfg::WZ;
    const int wy = warp % WY, wz = warp / WY;  // WY x WZ row blocks of LY (y) x LZ (z)
    const int ry = wy * LY + (lane % LY), rz = wz * LZ + (lane / LY);
    const int by0 = wy * LY, bz0 = wz * LZ;
    // point threads (phase A, one staged point each) are the four warps of
    // the edge row blocks (z edges of the square tile, y edges of the thin
    // one), whose lists are the shortest
    static_assert(NT % 32 == 0 && CH <= 128, "four point-thread warps");
    int edge = -1;
    if constexpr (WZ > 1) edge = wz == 0 ? wy : (wz == WZ - 1 ? 2 + wy : -1);
    else edge = wy < 2 ? wy : (wy >= WY - 2 ? wy - (WY - 2) + 2 : -1);
    static_assert(WZ > 1 ? WY == 2 : WY >= 4, "edge warps 0..3");
    const int pt = edge >= 0 ? edge * 32 + lane : CH;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    const int nsub = *a.nsub;
    Rows3Entry *mylist = s_list + warp * CH;
    // lane-constant operand bases (entries carry the per-point parts, biased by EBIAS)
    static_assert(Cfg::PAD, "two-word entries index the zero-padded r2 / c * r3");
    const unsigned char *base_f = smem_raw + (int)sizeof(T) * (ry - Cfg::EBIAS);
    // rz_eff: the lane's z row relative to the current bin's first plane
    // (= rz, except in the z-rolling mode below where the lane's plane stays
    // fixed while the bins advance)
    int rz_eff = rz;
    const unsigned char *base_cz = smem_raw + (int)sizeof(C) * (rz - Cfg::EBIAS);
    uint64_t pol_first, pol_last;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    C acc[X];
#pragma unroll
    for (int x = 0; x < X; ++x) acc[x] = C{(T)0, (T)0};
    // flush of the tile rows whose rz_eff < zcount (all rows: zcount = RZ)
    // through the shared-memory slab (aliases the stages): coalesced REDs
    auto flush_planes = [&](int t, int lo1, int lo2, int lo3, int zcount) {
        C *grid = reinterpret_cast<C *>(a.grid) + (int64_t)t * a.gstride;
        constexpr int ZS = RZ / Cfg::FP;  // z rows per pass
#pragma unroll 1
        for (int zlo = 0; zlo < zcount; zlo += ZS) {
            const int zn = min(ZS, zcount - zlo);
            if (rz_eff >= zlo && rz_eff < zlo + zn) {
                C *dst = s_tile + ((rz_eff - zlo) * RY + ry) * X;
#pragma unroll
                for (int x = 0; x < X; ++x) dst[x] = acc[x];
            }
            __syncthreads();
            for (int i = tid; i < zn * RY * X; i += NT) {
                const C v = s_tile[i];
                if (v.x == (T)0 && v.y == (T)0) continue;
                const int row = i / X, x = i - row * X;
                const int yy = row % RY, zz = zlo + row / RY;
                int g1 = lo1 + x;
                while (g1 >= n1) g1 -= n1;
                int g2 = lo2 + yy;
                while (g2 >= n2) g2 -= n2;
                int g3 = lo3 + zz;
                while (g3 >= n3) g3 -= n3;
                red_add(grid + ((int64_t)g3 * n2 + g2) * n1 + g1, v);
            }
            __syncthreads();
        }
        if (rz_eff < zcount) {
#pragma unroll
            for (int x = 0; x < X; ++x) acc[x] = C{(T)0, (T)0};
        }
    };
    // one subproblem's points into acc; unless rolling, each transform's
    // tile is flushed whole when its last chunk is done
    auto run_sub = [&](int s, bool rolling) __attribute__((always_inline)) {
        const int4 sp = a.subprob[s];

        const int bin = sp.x, start = sp.y, cnt = sp.z;
        const int b1 = bin % a.g.nb[0];
        const int b2 = (bin / a.g.nb[0]) % a.g.nb[1];
        const int b3 = bin / (a.g.nb[0] * a.g.nb[1]);
        const int lo1 = b1 * a.g.bs[0], lo2 = b2 * a.g.bs[1], lo3 = b3 * a.g.bs[2];
        const int nck = (cnt + CH - 1) / CH;
        const int nsteps = nck * a.ntransf;
        auto nch_of = [&](int ci) { return min(CH, cnt - ci * CH); };
        // asynchronous staging: each point thread copies and later reads only
        // its own ring / strength slots (no cross-thread hazards)
        auto issue_rec = [&](int st) {
            if (st < nsteps) {
                const int ci = st % nck;
                if (pt < nch_of(ci)) {
                    const Rec *src = a.rec + start + ci * CH + pt;
                    Rec *dst = s_ring + (st & 1) * CH + pt;
                    cp_async16_hint(dst, src, pol_first);
                    cp_async16_hint(reinterpret_cast<char *>(dst) + 16, reinterpret_cast<const char *>(src) + 16,
                                    pol_first);
                }
            }
            cp_async_commit();
        };
        auto issue_c = [&](int st) {
            if (st < nsteps) {
                const int ci = st % nck, t = st / nck;
                if (pt < nch_of(ci)) {
                    const int j = s_ring[(st & 1) * CH + pt].j;
                    const C *src = reinterpret_cast<const C *>(a.c) + (int64_t)t * a.M + j;
                    if constexpr (sizeof(C) == 16) {
                        cp_async16_hint(s_c + pt, src, pol_last);
                    } else {
                        cp_async8_hint(s_c + pt, src, pol_last);
                    }
                }
            }
            cp_async_commit();
        };
        // phase A: kernel rows of the thread's point of step st -> stage
        auto phase_a = [&](int st) {
            const int ci = st % nck;
            if (st < nsteps && pt < nch_of(ci)) {
                const Rec rc = s_ring[(st & 1) * CH + pt];
                const C c = s_c[pt];
                if (!finite2<T>(c)) flag_min(&a.flags[6], (unsigned long long)(rc.j + a.ibase));
                T *rec = s_stage + (st & 1) * CH * RECS + pt * RECS;
                T r[W];
                int i0 = kernel_row<T, W>(rc.g[0], a.k, r);
                const int ox = (i0 < 0 ? i0 + n1 : i0) - lo1;
#pragma unroll
                for (int m = 0; m < Cfg::R1N; ++m) rec[Cfg::O_R1 + m] = m < W ? r[m] : (T)0;
                i0 = kernel_row<T, W>(rc.g[1], a.k, r);
                const int oy = (i0 < 0 ? i0 + n2 : i0) - lo2;
                constexpr int B2 = Cfg::PAD ? Cfg::PY : 0, BZ3 = Cfg::PAD ? Cfg::PZ : 0;
#pragma unroll
                for (int m = 0; m < Cfg::R2N; ++m)
                    rec[Cfg::O_R2 + m] = (m >= B2 && m < B2 + W) ? r[m - B2 < W ? m - B2 : 0] : (T)0;
                i0 = kernel_row<T, W>(rc.g[2], a.k, r);
                const int oz = (i0 < 0 ? i0 + n3 : i0) - lo3;
#pragma unroll
                for (int m = 0; m < Cfg::CZN / 2; ++m) {
                    const T rm = (m >= BZ3 && m < BZ3 + W) ? r[m - BZ3 < W ? m - BZ3 : 0] : (T)0;
                    *reinterpret_cast<C *>(rec + Cfg::O_CZ + 2 * m) = C{c.x * rm, c.y * rm};
                }
                *reinterpret_cast<int4 *>(rec) = make_int4(oy, oz, ox, 0);
            }
        };
        // list of the chunk's points whose w x w row footprint meets this
        // warp's row block, in chunk (= x offset) order
        int nq = 0;
        auto build_list = [&](int st) {
            const int nch = nch_of(st % nck);
            const T *stg = s_stage + (st & 1) * CH * RECS;
            int n = 0;
            for (int b = 0; b < nch; b += 32) {
                const int q = b + lane;
                bool cov = false;
                int ox = 0, oy = 0, oz = 0;
                if (q < nch) {
                    const int4 o = *reinterpret_cast<const int4 *>(stg + q * RECS);
                    cov = o.x <= by0 + LY - 1 && o.x + W - 1 >= by0 && o.y <= bz0 + LZ - 1 && o.y + W - 1 >= bz0;
                    ox = o.z;
                    oy = o.x;
                    oz = o.y;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, cov);
                if (cov) {
                    const unsigned rb = (unsigned)((st & 1) * Cfg::STAGE_B + q * RECS * sizeof(T));  // record byte offset
                    const unsigned fi = rb / (unsigned)sizeof(T) + Cfg::O_R2 + Cfg::PY - oy + Cfg::EBIAS;
                    const unsigned zi = rb / (unsigned)sizeof(C) + Cfg::O_CZ / 2 + Cfg::PZ - oz + Cfg::EBIAS;
#if ESN_R3_WIDE
                    mylist[n + __popc(bal & ((1u << lane) - 1u))] =
                        make_uint4((rb / 16) | ((unsigned)ox << 16), fi * (unsigned)sizeof(T), zi * (unsigned)sizeof(C), rb);
#else
                    mylist[n + __popc(bal & ((1u << lane) - 1u))] = make_uint2((rb / 16) | ((unsigned)ox << 16), fi | (zi << 16));
#endif
                }
                n += __popc(bal);
            }
            __syncwarp();
            // run ends: bit 31 where the next entry's x offset differs (or at the end)
            for (int i = lane; i < n; i += 32) {
                const unsigned e = mylist[i].x;
                const unsigned en = i + 1 < n ? mylist[i + 1].x : 0xffffffffu;
                if (((e ^ en) >> 16) & 31u || i + 1 == n) mylist[i].x = e | 0x80000000u;
            }
            __syncwarp();
            nq = n;
        };
        // prologue: step 0 staged and listed
        issue_rec(0);
        cp_async_wait<0>();
        issue_c(0);
        issue_rec(1);
        cp_async_wait<1>();
        phase_a(0);
        __syncthreads();
        build_list(0);
#pragma unroll 1
        for (int st = 0; st < nsteps; ++st) {
            cp_async_wait<0>();  // own record of step st + 1
            issue_c(st + 1);
            issue_rec(st + 2);
            // phase B: runs of equal x offset, one static dispatch per run
            {
                const unsigned char *stg = smem_raw;
                int i = 0;
                while (i < nq) {
                    const int ox = (mylist[i].x >> 16) & 31;
                    switch (ox) {
#define ESN_R3_CASE(OX)                                                                  \
    case OX:                                                                             \
        if constexpr (OX < BX) i = rows3_run<T, W, OX>(acc, stg, mylist, i, base_f, base_cz); \
        else i = nq;                                                                     \
        break;
                        ESN_R3_CASE(0) ESN_R3_CASE(1) ESN_R3_CASE(2) ESN_R3_CASE(3)
                        ESN_R3_CASE(4) ESN_R3_CASE(5) ESN_R3_CASE(6) ESN_R3_CASE(7)
                        ESN_R3_CASE(8) ESN_R3_CASE(9) ESN_R3_CASE(10) ESN_R3_CASE(11)
                        ESN_R3_CASE(12) ESN_R3_CASE(13) ESN_R3_CASE(14) ESN_R3_CASE(15)
                        ESN_R3_CASE(16) ESN_R3_CASE(17) ESN_R3_CASE(18) ESN_R3_CASE(19)
                        ESN_R3_CASE(20) ESN_R3_CASE(21) ESN_R3_CASE(22) ESN_R3_CASE(23)
                        ESN_R3_CASE(24) ESN_R3_CASE(25) ESN_R3_CASE(26) ESN_R3_CASE(27)
                        ESN_R3_CASE(28) ESN_R3_CASE(29) ESN_R3_CASE(30) ESN_R3_CASE(31)
#undef ESN_R3_CASE
                        default:
                            i = nq;
                            break;
                    }
                }
            }
            cp_async_wait<1>();  // own strength of step st + 1
            if (!rolling && (st + 1) % nck == 0) {  // transform st / nck complete
                __syncthreads();
                flush_planes(st / nck, lo1, lo2, lo3, RZ);
            }
            phase_a(st + 1);
            __syncthreads();
            if (st + 1 < nsteps) build_list(st + 1);
        }
        cp_async_wait<0>();
    };
    const int nb0 = a.g.nb[0], nb1 = a.g.nb[1], nb2 = a.g.nb[2];
    const int nbins = nb0 * nb1 * nb2;
    auto nsub_of = [&](int bin) { return (bin + 1 < nbins ? a.subofs[bin + 1] : nsub) - a.subofs[bin]; };
    // a bin is rolled when it is one subproblem of at most ROLLMAX points:
    // larger bins (clustered data, large pipeline chunks) stay independent
    // subproblems so no segment carries many times a CTA's share of the work
    constexpr int ROLLMAX = 1024;
    auto rolled = [&](int bin) {
        return nsub_of(bin) == 1 && a.bin_start[bin + 1] - a.bin_start[bin] <= ROLLMAX;
    };
    auto claim = [&](int q) {  // next item of work queue q (CTA-uniform)
        if (tid == 0) s_sub = atomicAdd(a.work + q, 1);
        __syncthreads();
        const int v = s_sub;
        __syncthreads();
        return v;
    };
    // Work: plain mode -- every subproblem of queue 0 with a whole-tile
    // flush.  z-rolling mode (thin tiles, one transform): queue 0 holds
    // columns (b1, b2) x segments of ZB bins along z.  A bin's tile is planes
    // [lo3, lo3 + RZ); after the bin only its first BZ planes are complete,
    // so only those rows are flushed and the lanes holding them take over the
    // next bin's top planes (a lane's plane stays fixed, rz_eff = (plane -
    // lo3) mod RZ): BZ / RZ of the tile per bin instead of all of it.  Bins
    // split into several subproblems (clustered points) go to queue 1, whose
    // subproblems run one by one with whole-tile flushes.  One call site of
    // run_sub (code size).
    // segment length: up to 8 bins, fewer when that would leave under ~8
    // segments per CTA (tail balance)
    constexpr int ZBMAX = 8;
    __shared__ int s_nsb[ZBMAX], s_sof[ZBMAX];
    const int ZB = max(1, min(ZBMAX, nbins / (8 * (int)gridDim.x)));
    // (ROLL is a template flag: the plain instantiation keeps rz_eff == rz
    // a constant and the rolling driver out of its code)
    const bool roll = ROLL && WZ == 1 && a.ntransf == 1 && a.subofs != nullptr;
    const int BZ = a.g.bs[2];
    const int nitems = nb0 * nb1 * ((nb2 + ZB - 1) / ZB);
    const int reach = (RZ - 1) / BZ;  // bins before b3 whose tiles reach b3's first plane
    int phase = roll ? 0 : 2;
    int b3 = 0, b3s = 0, b3b = 0, lo1r = 0, lo2r = 0, lo3r = 0, last_pts = -1000000;
    for (;;) {
        int s = -1;
        if (phase == 0) {
            if (b3 >= b3b) {  // next segment
                const int item = claim(0);
                if (item >= nitems) {
                    phase = 1;
                    if constexpr (ROLL) {
                        rz_eff = rz;
                        base_cz = smem_raw + (int)sizeof(C) * (rz - Cfg::EBIAS);
                    }
                    continue;
                }
                const int b1 = item % nb0, b2 = (item / nb0) % nb1, seg = item / (nb0 * nb1);
                lo1r = b1 * a.g.bs[0];
                lo2r = b2 * a.g.bs[1];
                b3 = b3s = seg * ZB;
                b3b = min(nb2, b3 + ZB);
                lo3r = b3 * BZ;
                last_pts = -1000000;
                if constexpr (ROLL) {
                    rz_eff = ((rz - lo3r) % RZ + RZ) % RZ;
                    base_cz = smem_raw + (int)sizeof(C) * (rz_eff - Cfg::EBIAS);
                }
                // the segment's subproblem counts, loaded at once (empty
                // columns then cost one memory latency, not one per bin)
                if (tid < b3b - b3) {
                    const int bin = b1 + nb0 * (b2 + nb1 * (b3 + tid));
                    s_sof[tid] = a.subofs[bin];
                    s_nsb[tid] = rolled(bin) ? 1 : 0;
                }
                __syncthreads();
            }
            if (s_nsb[b3 - b3s] == 1) s = s_sof[b3 - b3s];
        } else if (phase == 1) {
            s = claim(1);
            if (s >= nsub) break;
            const int bin = a.subprob[s].x;
            if (rolled(bin) || nsub_of(bin) == 0) continue;  // (done by a segment)
        } else {
            s = claim(0);
            if (s >= nsub) break;
        }
        if (s >= 0) run_sub(s, phase == 0);
        if (phase == 0) {
            if (s >= 0) last_pts = b3;
            // the bin's first BZ planes are complete (all of them at the
            // segment end); nothing to flush unless a bin with points reached them
            const bool last = b3 + 1 >= b3b;
            if (last_pts >= b3 - reach) {
                __syncthreads();
                flush_planes(0, lo1r, lo2r, lo3r, last ? RZ : BZ);
            }
            ++b3;
            lo3r += BZ;
            if constexpr (ROLL) {
                rz_eff = ((rz - lo3r) % RZ + RZ) % RZ;
                base_cz = smem_raw + (int)sizeof(C) * (rz_eff - Cfg::EBIAS);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Batched 2D spreader (ntransf > 1): lanes are transforms.  A CTA owns one
// bin tile (rows y of length X in registers) for 32 transforms at a time
// (one warp per tile row, lane = transform); every staged point is applied by
// the warps of its w rows with identical kernel values, so there is no lane
// waste and the point data is a broadcast.
// Per-point kernel rows for the batched 2D spreader: evaluated once per
// point (not once per warp visit), 2W floats + the wrapped origins.
template <int W>
struct alignas(16) PtRows2 {
    float r1[W];
    float r2[W];
    int i1, i2;
};

template <typename T, int W>
__global__ void __launch_bounds__(256) k_rows2d(SpreadArgs<T> a, PtRows2<W> *tab) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.M; k += (int64_t)gridDim.x * blockDim.x) {
        const Rec rc = load_rec(a.rec, k);
        PtRows2<W> e;
        T r[W];
        int i0 = kernel_row<T, W>(rc.g[0], a.k, r);
        e.i1 = i0 < 0 ? i0 + a.g.n[0] : i0;
#pragma unroll
        for (int m = 0; m < W; ++m) e.r1[m] = (float)r[m];
        i0 = kernel_row<T, W>(rc.g[1], a.k, r);
        e.i2 = i0 < 0 ? i0 + a.g.n[1] : i0;
#pragma unroll
        for (int m = 0; m < W; ++m) e.r2[m] = (float)r[m];
        tab[k] = e;
    }
}

// batched 2D spreader: points staged per warp per batch
constexpr int kBatchPts = 16;
template <typename T, int W>
constexpr size_t batch2d_stage_bytes() {  // points + strength lines + one row of key starts
    return (size_t)kBatchPts * (sizeof(PtRows2<W>) + 32 * 2 * sizeof(T)) +
           (size_t)((Batch2Cfg<T, W>::BX + 1 + 3) / 4 + 1) * 16;
}
template <typename T, int W>
constexpr size_t batch2d_smem_bytes() {  // 4 warps x 2 stages (the flush slab aliases them)
    return 4 * 2 * batch2d_stage_bytes<T, W>();
}

// flush of one warp's tile row: transpose the 32 transforms x X cells
// through the warp's shared-memory slab (aliasing its idle staging ring) so
// each RED burst is one transform's contiguous row (lanes = x): lanes =
// transforms would scatter 32 planes apart, which runs at ~4e10 ops/s on
// B200 vs ~3.7e11 coalesced (measured)
template <typename T, int W>
__device__ __forceinline__ void batch2d_flush(const typename Cx<T>::type *acc, unsigned char *wbase, int lane,
                                              int lo1, int lo2, int row, int tg, const SpreadArgs<T> &a) {
    using C = typename Cx<T>::type;
    constexpr int X = Batch2Cfg<T, W>::X;
    const int n1 = a.g.n[0], n2 = a.g.n[1];
    C *slab = reinterpret_cast<C *>(wbase);
#pragma unroll
    for (int x = 0; x < X; ++x) slab[lane * (X + 1) + x] = acc[x];
    __syncwarp();
    int g2 = lo2 + row;
    while (g2 >= n2) g2 -= n2;
    int g1 = lo1 + lane;
    while (g1 >= n1) g1 -= n1;
    const int tmax = min(32, a.ntransf - tg * 32);
    for (int tt = 0; tt < tmax; ++tt) {
        if (lane < X) {
            const C v = slab[tt * (X + 1) + lane];
            if (v.x != (T)0 || v.y != (T)0)
                red_add(reinterpret_cast<C *>(a.grid) + (int64_t)(tg * 32 + tt) * a.gstride + (int64_t)g2 * n1 + g1, v);
        }
    }
    __syncwarp();
}

// zero `n16` 16-byte units of the grid when *flag is set (the RED-flush
// batched spreader taking over from an owner-computes one needs a zeroed grid)
template <typename T>  // (a template only so that every instantiation unit may define it)
__global__ void __launch_bounds__(256) k_zero_if(int4 *p, size_t n16, const int *flag) {
    if (!*flag) return;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_int4(0, 0, 0, 0);
}

template <typename T, int W, bool CELLKEYS>
__global__ void __launch_bounds__(128) k_spread_batch2d(SpreadArgs<T> a, const T *cperm, const PtRows2<W> *tab) {
    // (plans that may switch: this kernel runs only when the sort found the
    // bins badly imbalanced; the owner-computes kernel launched before it
    // then exited at once)
    if (a.imb && !*a.imb) return;
    // Warp-independent: a persistent warp takes work items (subproblem,
    // transform group, tile row) from an atomic queue.  Lane = transform.
    // The item's points are one contiguous run of the finely sorted bin
    // (oy in [row - W + 1, row]); their kernel rows come precomputed
    // (k_rows2d), their strengths as one 256-byte line per point.  Both are
    // staged per warp in batches of kBatchPts points with cp.async, one
    // batch ahead (double buffer), so the loop reads only shared memory.
    // No block barriers.
    using C = typename Cx<T>::type;
    using Cfg = Batch2Cfg<T, W>;
    constexpr int X = Cfg::X, RY = Cfg::RY;
    constexpr int TB = sizeof(PtRows2<W>), CB = 32 * sizeof(C);
    constexpr size_t STAGE = batch2d_stage_bytes<T, W>();
    static_assert(TB % 16 == 0 && CB % 16 == 0, "16-byte staging chunks");
    static_assert(2 * STAGE >= (size_t)32 * (X + 1) * sizeof(C), "flush slab must fit the warp's ring");
    extern __shared__ __align__(16) unsigned char b2_smem[];
    const int lane = threadIdx.x & 31;
    unsigned char *wbase = b2_smem + (threadIdx.x >> 5) * 2 * STAGE;
    const int n1 = a.g.n[0], n2 = a.g.n[1];
    const int nsub = *a.nsub;
    const int ngroups = (a.ntransf + 31) / 32;
    const int nitems = nsub * ngroups * RY;
    const int kx = a.g.bs[0] >> a.sbl[0];
    // the next work item is claimed one item ahead (the atomic's latency
    // overlaps the current item)
    int next = 0;
    if (lane == 0) next = atomicAdd(a.work, 1);
    for (;;) {
        const int item = __shfl_sync(0xffffffffu, next, 0);
        if (item >= nitems) break;
        if (lane == 0) next = atomicAdd(a.work, 1);
        const int row = item % RY;
        const int sg = item / RY;
        const int tg = sg % ngroups;
        const int4 sp = a.subprob[sg / ngroups];
        const int bin = sp.x, start = sp.y, cnt = sp.z;
        const int b1 = bin % a.g.nb[0], b2 = bin / a.g.nb[0];
        const int lo1 = b1 * a.g.bs[0], lo2 = b2 * a.g.bs[1];
        const int ylo = max(0, row - W + 1), yhi = min(row, a.g.bs[1] - 1);
        if (ylo > yhi) continue;
        const int *ks = a.kstart + (int64_t)bin * a.spb;
        const int k0 = max(start, ks[(ylo >> a.sbl[1]) * kx]);
        const int r1k = (yhi >> a.sbl[1]) + 1;
        const int k1 = min(start + cnt, r1k * kx < a.spb ? ks[r1k * kx] : 0x7fffffff);
        if (k0 >= k1) continue;
        const C *cg = reinterpret_cast<const C *>(cperm) + (int64_t)tg * a.M * 32;
        if constexpr (CELLKEYS) {
            // Cell-resolution keys: inside one y row of the bin the points
            // are grouped by x cell, and every point of a cell shares (ox,
            // dy).  Pieces of <= kBatchPts points never straddle a y row;
            // the x offset is swept as a compile-time loop, so the register
            // window needs no per-point dispatch.
            constexpr int BX = Cfg::BX;
            constexpr int KSOFF = kBatchPts * (TB + CB);
            const int end = start + cnt;
            // first key start of rows ylo .. yhi + 1, one per lane (one load per item)
            const int ly = ylo + lane;
            const int rowk = (lane <= yhi - ylo + 1) ? (ly * kx < a.spb ? ks[ly * kx] : 0x7fffffff) : 0x7fffffff;
            auto row_lo = [&](int y) { return max(start, __shfl_sync(0xffffffffu, rowk, y - ylo)); };
            auto row_hi = [&](int y) { return min(end, __shfl_sync(0xffffffffu, rowk, y - ylo + 1)); };
            // piece state: y row, [kb, ke)
            int py = ylo, pb = row_lo(ylo);
            auto advance = [&](int &y, int &kb) {  // next non-empty piece start after [kb, ke)
                const int he = row_hi(y);
                const int ke = min(kb + kBatchPts, he);
                if (ke < he) { kb = ke; return; }
                for (++y; y <= yhi; ++y) {
                    kb = row_lo(y);
                    if (kb < row_hi(y)) return;
                }
            };
            if (pb >= row_hi(py)) advance(py, pb);  // (first row may be empty)
            auto issue_piece = [&](int y, int kb, int buf) {
                if (y <= yhi) {
                    const int n = min(kBatchPts, row_hi(y) - kb);
                    const char *src = reinterpret_cast<const char *>(tab + kb);
                    unsigned char *dst = wbase + buf * STAGE;
                    for (int c = lane; c < n * TB / 16; c += 32) cp_async16(dst + 16 * c, src + 16 * c);
                    const char *src2 = reinterpret_cast<const char *>(cg + (int64_t)kb * 32);
                    unsigned char *dst2 = dst + kBatchPts * TB;
                    for (int c = lane; c < n * CB / 16; c += 32) cp_async16(dst2 + 16 * c, src2 + 16 * c);
                    // key starts of this row's x cells (+ the next row's first)
                    const char *src3 = reinterpret_cast<const char *>(ks + y * kx);
                    for (int c = lane; c < (BX + 1 + 3) / 4; c += 32) cp_async16(dst + KSOFF + 16 * c, src3 + 16 * c);
                }
                cp_async_commit();
            };
            C acc[X];
#pragma unroll
            for (int x = 0; x < X; ++x) acc[x] = C{(T)0, (T)0};
            issue_piece(py, pb, 0);
            int buf = 0;
            while (py <= yhi) {
                int ny = py, nb = pb;
                advance(ny, nb);
                issue_piece(ny, nb, buf ^ 1);
                cp_async_wait<1>();
                __syncwarp();
                const int ke = min(pb + kBatchPts, row_hi(py));
                const int dy = row - py;
                const PtRows2<W> *tb = reinterpret_cast<const PtRows2<W> *>(wbase + buf * STAGE);
                const C *cq = reinterpret_cast<const C *>(wbase + buf * STAGE + kBatchPts * TB) + lane;
                const int *sks = reinterpret_cast<const int *>(wbase + buf * STAGE + KSOFF);
                // piece-local [lo, hi) of every x cell
                int lo = min(max(sks[0], pb), ke) - pb;
#pragma unroll
                for (int ox = 0; ox < BX; ++ox) {
                    const int hi = ox + 1 < BX ? min(max(sks[ox + 1], pb), ke) - pb : ke - pb;
#pragma unroll 1
                    for (int k = lo; k < hi; ++k) {
                        const PtRows2<W> &e = tb[k];
                        const T wy = (T)e.r2[dy];
                        const C cc = cq[k * 32];
                        const C v{cc.x * wy, cc.y * wy};
#pragma unroll
                        for (int m = 0; m < W; ++m) {
                            const T r = (T)e.r1[m];
                            acc[ox + m].x = fma(v.x, r, acc[ox + m].x);
                            acc[ox + m].y = fma(v.y, r, acc[ox + m].y);
                        }
                    }
                    lo = hi;
                }
                __syncwarp();
                buf ^= 1;
                py = ny;
                pb = nb;
            }
            cp_async_wait<0>();
            __syncwarp();
            batch2d_flush<T, W>(acc, wbase, lane, lo1, lo2, row, tg, a);
        } else {
        auto issue = [&](int kb, int buf) {  // stage points [kb, min(kb + NB, k1))
            const int n = min(kBatchPts, k1 - kb);
            if (n > 0) {
                const char *src = reinterpret_cast<const char *>(tab + kb);
                unsigned char *dst = wbase + buf * STAGE;
                for (int c = lane; c < n * TB / 16; c += 32) cp_async16(dst + 16 * c, src + 16 * c);
                const char *src2 = reinterpret_cast<const char *>(cg + (int64_t)kb * 32);
                unsigned char *dst2 = dst + kBatchPts * TB;
                for (int c = lane; c < n * CB / 16; c += 32) cp_async16(dst2 + 16 * c, src2 + 16 * c);
            }
            cp_async_commit();
        };
        C acc[X];
#pragma unroll
        for (int x = 0; x < X; ++x) acc[x] = C{(T)0, (T)0};
        issue(k0, 0);
        int buf = 0;
        for (int kb = k0; kb < k1; kb += kBatchPts) {
            issue(kb + kBatchPts, buf ^ 1);
            cp_async_wait<1>();
            __syncwarp();
            const int n = min(kBatchPts, k1 - kb);
            const PtRows2<W> *tb = reinterpret_cast<const PtRows2<W> *>(wbase + buf * STAGE);
            const C *cq = reinterpret_cast<const C *>(wbase + buf * STAGE + kBatchPts * TB);
            const int row2 = row + lo2;
            for (int i = 0; i < n; ++i) {
                const PtRows2<W> &e = tb[i];  // shared memory: loads below are broadcasts
                const int dy = row2 - e.i2;
                if ((unsigned)dy >= (unsigned)W) continue;  // warp-uniform (sub-cell edges)
                const T wy = (T)e.r2[dy];                   // dynamic index into shared memory
                const C ccur = cq[i * 32 + lane];
                const C v{ccur.x * wy, ccur.y * wy};
                T r1[W];
#pragma unroll
                for (int m = 0; m < W; ++m) r1[m] = (T)e.r1[m];
                rows_accumulate<T, 2, W>(acc, e.i1 - lo1, v, r1);
            }
            __syncwarp();
            buf ^= 1;
        }
        cp_async_wait<0>();
        __syncwarp();
        batch2d_flush<T, W>(acc, wbase, lane, lo1, lo2, row, tg, a);
        }
    }
}

// ---------------------------------------------------------------------------
// Batched 2D spreader, owner-computes ("b2own").  A bin of 16 x 16 footprint
// origins is also an OUTPUT block: the warp of work item (bin, transform
// group, output row pair) owns fine cells [lo1, lo1 + 16) of rows gy, gy + 1
// for 32 transforms (lane = transform) and gathers every point whose
// footprint reaches them -- origins in rows gy - w + 1 .. gy + 1 (wrapped,
// possibly in the bin below) and columns lo1 - w + 1 .. lo1 + 15 (wrapped,
// possibly in the bin to the left).  Each fine cell is written exactly once
// with a plain coalesced store: no grid memset, no atomics, no halo flush
// (the tile spreader k_spread_batch2d spent ~1/3 of its time in RED flushes
// and the grid was zeroed first); DRAM traffic is the algorithmic bytes
// (ncu: 570 MB read, 500 MB written for c5).  Points come in pieces of
// <= kBatchPts staged by cp.async one piece ahead (tab rows + 256-byte
// strength lines) in source-cell order; the x offset (= source cell, kept
// per slot, so periodic duplicates on tiny grids are ordinary cells) selects
// a static register window through one switch per point (a branch tree on
// sm_100a, ~10 instructions) that serves both output rows, and only the
// FMAs that land in owned columns are formed.
// per-warp shared memory: 2 piece stages + per source row the lanes' first
// point / staged offset (plus the row's total and run mask)
constexpr int kB2Rows = 2;  // output rows per work item (register window per row: 2 (w - 1) + 16 cells)
template <typename T, int W>
constexpr size_t b2own_row_bytes() { return ((size_t)(W + kB2Rows - 1) * (2 * 32 + 2) * sizeof(int) + 15) / 16 * 16; }
template <typename T, int W>
constexpr size_t b2own_smem_bytes() { return 4 * (2 * batch2d_stage_bytes<T, W>() + b2own_row_bytes<T, W>()); }

template <typename T, int W>
__global__ void __launch_bounds__(128) k_spread_b2own(SpreadArgs<T> a, const T *cperm, const PtRows2<W> *tab) {
    if (a.imb && *a.imb) return;  // imbalanced bins: the RED-flush kernel launched next takes over
    constexpr int R = kB2Rows;
    using C = typename Cx<T>::type;
    constexpr int BX = Batch2Cfg<T, W>::BX, BY = Batch2Cfg<T, W>::BY;
    constexpr int H = W - 1;            // halo cells
    constexpr int SRC = BX + H;         // source cells per source row (lanes)
    constexpr int NR = W + R - 1;       // source rows per item
    constexpr int NB = kBatchPts;
    constexpr int TB = sizeof(PtRows2<W>), CB = 32 * sizeof(C);
    constexpr size_t STAGE = batch2d_stage_bytes<T, W>();
    static_assert(SRC < 32, "one lane per source cell (+ the end lane)");
    static_assert((size_t)NB * (TB + CB) + NB <= STAGE, "stage holds a piece and its x offsets");
    static_assert(2 * STAGE >= (size_t)32 * (BX + 1) * sizeof(C), "store slab fits the ring");
    static_assert(BY % R == 0, "row groups tile the bin");
    extern __shared__ __align__(16) unsigned char b2_smem[];
    const int lane = threadIdx.x & 31;
    unsigned char *wbase = b2_smem + (threadIdx.x >> 5) * (2 * STAGE + b2own_row_bytes<T, W>());
    int *rs = reinterpret_cast<int *>(wbase + 2 * STAGE);  // [d][32] first point of the lane's cell
    int *ro = rs + NR * 32;                                  // [d][32] staged offset of the lane's cell
    int *rt = ro + NR * 32;                                  // [d] row total
    unsigned *rr = reinterpret_cast<unsigned *>(rt + NR);    // [d] run-start mask
    const int n1 = a.g.n[0], n2 = a.g.n[1], nb0 = a.g.nb[0];
    const int ngroups = (a.ntransf + 31) / 32;
    const int nitems = a.g.nb[0] * a.g.nb[1] * ngroups * (BY / R);
    int next = 0;
    if (lane == 0) next = atomicAdd(a.work, 1);
    for (;;) {
        const int item = __shfl_sync(0xffffffffu, next, 0);
        if (item >= nitems) break;
        if (lane == 0) next = atomicAdd(a.work, 1);
        const int yp = item % (BY / R);
        const int sg = item / (BY / R);
        const int tg = sg % ngroups, bin = sg / ngroups;
        const int lo1 = (bin % nb0) * BX, lo2 = (bin / nb0) * BY;
        const int gy = lo2 + R * yp;  // output rows gy .. gy + R - 1 (acc[0..R))
        if (gy >= n2) continue;       // partial last bin row
        // lane k < SRC: source cell column lo1 - H + k (wrapped); own columns
        // past n1 (partial last bin) hold no points
        int xa = lo1 - H + lane;
        const bool valid = lane < SRC && !(lane >= H && xa >= n1);
        while (xa < 0) xa += n1;  // (loops only on grids narrower than the halo)
        while (xa >= n1) xa -= n1;
        __syncwarp();  // previous item's readers of the row tables are done
        // source row d: origin row gy + R - 1 - d (output row gy + rr takes r2[rr + d - R + 1])
#pragma unroll
        for (int d = 0; d < NR; ++d) {
            int r = gy + R - 1 - d;
            while (r < 0) r += n2;
            while (r >= n2) r -= n2;
            int s = 0, e = 0;
            if (valid) {
                const int key = (((r / BY) * nb0 + xa / BX) * BY + (r % BY)) * BX + (xa % BX);
                s = a.kstart[key];
                e = a.kstart[key + 1];
            }
            const int cnt = e - s;
            int inc = cnt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += v;
            }
            const int eprev = __shfl_up_sync(0xffffffffu, e, 1);
            // a run is a chain of abutting ranges (empty cells may start one)
            const unsigned runs = __ballot_sync(0xffffffffu, valid && (lane == 0 || s != eprev));
            rs[d * 32 + lane] = s;
            ro[d * 32 + lane] = inc - cnt;  // lane SRC holds the row total
            if (lane == 31) {
                rt[d] = inc;
                rr[d] = runs;
            }
        }
        __syncwarp();
        const C *cg = reinterpret_cast<const C *>(cperm) + (int64_t)tg * a.M * 32;
        // stage piece (d, q0): staged indices [q0, q0 + NB) of source row d
        auto issue_piece = [&](int d, int q0, int buf) {
            if (d < NR) {
                unsigned char *dst = wbase + buf * STAGE;
                const int tot = rt[d];
                const int q1 = min(q0 + NB, tot);
                unsigned rm = rr[d];
                while (rm) {
                    const int k0 = __ffs(rm) - 1;
                    rm &= rm - 1;
                    const int k1 = rm ? __ffs(rm) - 1 : 32;
                    const int ok0 = ro[d * 32 + k0];
                    const int ok1 = k1 < 32 ? ro[d * 32 + k1] : tot;
                    const int a0 = max(ok0, q0), a1 = min(ok1, q1);
                    if (a0 >= a1) continue;
                    const int n = a1 - a0, src0 = rs[d * 32 + k0] + (a0 - ok0), slot0 = a0 - q0;
                    const char *ts = reinterpret_cast<const char *>(tab + src0);
                    for (int c = lane; c < n * TB / 16; c += 32)
                        cp_async16(dst + slot0 * TB + 16 * c, ts + 16 * c);
                    const char *cs = reinterpret_cast<const char *>(cg + (int64_t)src0 * 32);
                    for (int c = lane; c < n * CB / 16; c += 32)
                        cp_async16(dst + NB * TB + slot0 * CB + 16 * c, cs + 16 * c);
                }
                // x offset (= source cell) of every staged slot
                unsigned char *sox = dst + NB * (TB + CB);
                const int myo = ro[d * 32 + lane];
                const int c0 = max(myo, q0), c1 = min(lane + 1 < 32 ? ro[d * 32 + lane + 1] : myo, q1);
                for (int q = c0; q < c1; ++q) sox[q - q0] = (unsigned char)lane;
            }
            cp_async_commit();
        };
        auto advance = [&](int &d, int &q0) {  // next non-empty piece after (d, q0)
            q0 += NB;
            if (q0 < rt[d]) return;
            q0 = 0;
            for (++d; d < NR && rt[d] == 0; ++d) {
            }
        };
        // owned cells only: contributions that land in the halo columns
        // belong to the neighbouring block's warp and are never formed
        C acc[R][BX];
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int x = 0; x < BX; ++x) acc[rr][x] = C{(T)0, (T)0};
        int pd = 0, pq = 0;
        while (pd < NR && rt[pd] == 0) ++pd;
        issue_piece(pd, pq, 0);
        int buf = 0;
        while (pd < NR) {
            int nd = pd, nq = pq;
            advance(nd, nq);
            issue_piece(nd, nq, buf ^ 1);
            cp_async_wait<1>();
            __syncwarp();
            const int np = min(NB, rt[pd] - pq);
            const unsigned char *sb = wbase + buf * STAGE;
            const PtRows2<W> *tb = reinterpret_cast<const PtRows2<W> *>(sb);
            const C *cq = reinterpret_cast<const C *>(sb + NB * TB) + lane;
            int wi[R];
            bool wh[R];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                const int dy = rr + pd - (R - 1);
                wh[rr] = dy >= 0 && dy < W;
                wi[rr] = wh[rr] ? dy : 0;
            }
            const unsigned char *sox = sb + NB * (TB + CB);
#pragma unroll 1
            for (int k = 0; k < np; ++k) {
                const PtRows2<W> &e = tb[k];
                const C cc = cq[k * 32];
                C v[R];
#pragma unroll
                for (int rr = 0; rr < R; ++rr) {
                    const T wy = wh[rr] ? (T)e.r2[wi[rr]] : (T)0;
                    v[rr] = C{cc.x * wy, cc.y * wy};
                }
                T r1[W];
#pragma unroll
                for (int m = 0; m < W; ++m) r1[m] = (T)e.r1[m];
                // one static dispatch per point (branch tree) serves all R rows
#define ESN_B2O_CASE(OX)                                                      \
    case OX:                                                                  \
        if constexpr (OX < SRC) {                                             \
            _Pragma("unroll") for (int m = 0; m < W; ++m) {                   \
                constexpr int XL = OX - H;                                    \
                if (XL + m >= 0 && XL + m < BX) {                             \
                    _Pragma("unroll") for (int rr = 0; rr < R; ++rr) {        \
                        acc[rr][XL + m].x = fma(v[rr].x, r1[m], acc[rr][XL + m].x); \
                        acc[rr][XL + m].y = fma(v[rr].y, r1[m], acc[rr][XL + m].y); \
                    }                                                         \
                }                                                             \
            }                                                                 \
        }                                                                     \
        break;
                switch (sox[k]) {
                    ESN_B2O_CASE(0) ESN_B2O_CASE(1) ESN_B2O_CASE(2) ESN_B2O_CASE(3)
                    ESN_B2O_CASE(4) ESN_B2O_CASE(5) ESN_B2O_CASE(6) ESN_B2O_CASE(7)
                    ESN_B2O_CASE(8) ESN_B2O_CASE(9) ESN_B2O_CASE(10) ESN_B2O_CASE(11)
                    ESN_B2O_CASE(12) ESN_B2O_CASE(13) ESN_B2O_CASE(14) ESN_B2O_CASE(15)
                    ESN_B2O_CASE(16) ESN_B2O_CASE(17) ESN_B2O_CASE(18) ESN_B2O_CASE(19)
                    ESN_B2O_CASE(20) ESN_B2O_CASE(21) ESN_B2O_CASE(22) ESN_B2O_CASE(23)
                    ESN_B2O_CASE(24) ESN_B2O_CASE(25) ESN_B2O_CASE(26) ESN_B2O_CASE(27)
                    ESN_B2O_CASE(28) ESN_B2O_CASE(29) ESN_B2O_CASE(30)
                    default:
                        break;
                }
#undef ESN_B2O_CASE
            }
            __syncwarp();
            buf ^= 1;
            pd = nd;
            pq = nq;
        }
        cp_async_wait<0>();
        __syncwarp();
        // owned cells: transpose through the warp's ring so
        // each store covers one transform's contiguous 16-cell run (two
        // transforms per instruction)
        C *slab = reinterpret_cast<C *>(wbase);
        const int hx = lane & (BX - 1), ht = lane / BX;
        const int g1 = lo1 + hx;
        const int tmax = min(32, a.ntransf - tg * 32);
#pragma unroll
        for (int row = 0; row < R; ++row) {
            const int gyr = gy + row;
#pragma unroll
            for (int x = 0; x < BX; ++x) slab[lane * (BX + 1) + x] = acc[row][x];
            __syncwarp();
            if (g1 < n1 && gyr < n2) {
                for (int tt = ht; tt < tmax; tt += 32 / BX) {
                    C *dstp = reinterpret_cast<C *>(a.grid) + (int64_t)(tg * 32 + tt) * a.gstride +
                              (int64_t)gyr * n1 + g1;
                    const C v = slab[tt * (BX + 1) + hx];
                    if (a.accumulate)
                        red_add(dstp, v);  // concurrent partial spreads (pipelined host path) into one grid
                    else
                        *dstp = v;
                }
            }
            __syncwarp();
        }
    }
}

// Batched strengths into sorted order, 32 transforms per point:
// cperm[g][pos(j)][l] = c[32 g + l][j] with pos(j) the sorted position setpts
// left in key[j].
// A 32 x 32 tile transpose through shared memory: coalesced reads along j,
// one contiguous 32-transform record per point on the write side.  Also the
// finiteness check of the strengths.
template <typename T>
__global__ void __launch_bounds__(1024) k_permute_strengths(SpreadArgs<T> a, const int *key,
                                                            const int *kstart, T *cperm) {
    // U tiles of 32 points per iteration: U loads in flight per thread and
    // one barrier pair per U tiles
    using C = typename Cx<T>::type;
    constexpr int U = 4;
    __shared__ C tile[U][32][33];
    (void)kstart;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int ngroups = (a.ntransf + 31) / 32;
    const int64_t jblocks = (a.M + 32 * U - 1) / (32 * U);
    for (int64_t b = blockIdx.x; b < jblocks * ngroups; b += gridDim.x) {
        const int g = (int)(b % ngroups);
        const int64_t j0 = (b / ngroups) * 32 * U;
        const int t = g * 32 + ty;
        C v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + u * 32 + tx;
            v[u] = C{(T)0, (T)0};
            if (t < a.ntransf && j < a.M) v[u] = reinterpret_cast<const C *>(a.c)[(int64_t)t * a.M + j];
        }
        int pos[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t jj = j0 + u * 32 + ty;
            pos[u] = jj < a.M ? key[jj] : -1;  // setpts leaves each point's sorted position in key[]
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + u * 32 + tx;
            if (t < a.ntransf && j < a.M && !finite2<T>(v[u]))
                flag_min(&a.flags[6], (unsigned long long)(j + a.ibase));
            tile[u][ty][tx] = v[u];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (pos[u] >= 0) reinterpret_cast<C *>(cperm)[((int64_t)g * a.M + pos[u]) * 32 + tx] = tile[u][tx][ty];
        __syncthreads();
    }
}

constexpr int kInterpSlice = 1024;  // point records staged per slice (32 KB)

// CTAs per SM the interpolators are register-capped for: 3 (<= 80 registers)
// only where the body fits without spilling (2D, w <= 7)
template <int DIM, int W>
constexpr int interp_minb() { return (DIM == 2 && W <= 7) ? 3 : 2; }

// ---------------------------------------------------------------------------
// Tile interpolator (spreadinterp.py:442-507).  One CTA per subproblem
// (persistent work queue): the bin's periodic patch of (bs + w - 1)^d fine
// cells is staged once in shared memory with coalesced loads, then each
// thread interpolates sorted points from it (separable weighted sum, row
// partial sums in registers).  Consecutive threads hold consecutive finely
// sorted points, so the shared-memory gathers of a warp hit a few adjacent
// cells (near-broadcast, conflict-light).  Output in ORIGINAL point order
// (spreadinterp.py:453).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256, interp_minb<DIM, W>()) k_interp_tile(SpreadArgs<T> a, T *cout, const T *gridp) {
    using C = typename Cx<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Rec *s_rec = reinterpret_cast<Rec *>(smem_raw);               // kInterpSlice records
    C *patch = reinterpret_cast<C *>(s_rec + kInterpSlice);
    __shared__ int s_sub;
    const int tid = threadIdx.x;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    const int P1 = a.g.bs[0] + W - 1;
    const int P2 = DIM > 1 ? a.g.bs[1] + W - 1 : 1;
    const int P3 = DIM > 2 ? a.g.bs[2] + W - 1 : 1;
    const int ncell = P1 * P2 * P3;
    const int nsub = *a.nsub;
    const int nwork = nsub * a.ntransf;
    for (;;) {
        if (tid == 0) s_sub = atomicAdd(a.work, 1);
        __syncthreads();
        const int s = s_sub;
        if (s >= nwork) break;
        const int t = s / nsub;
        const int4 sp = a.subprob[s - t * nsub];
        const int bin = sp.x % (a.g.nb[0] * a.g.nb[1] * a.g.nb[2]), start = sp.y, cnt = sp.z;  // geometric bin
        const int b1 = bin % a.g.nb[0];
        const int b2 = DIM > 1 ? (bin / a.g.nb[0]) % a.g.nb[1] : 0;
        const int b3 = DIM > 2 ? bin / (a.g.nb[0] * a.g.nb[1]) : 0;
        const int lo1 = b1 * a.g.bs[0], lo2 = b2 * a.g.bs[1], lo3 = b3 * a.g.bs[2];
        const C *grid = reinterpret_cast<const C *>(gridp) + (int64_t)t * a.gstride;
        // patch: 4 independent loads in flight per thread, then the stores
        for (int i0 = tid; i0 < ncell; i0 += 4 * blockDim.x) {
            C v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i >= ncell) break;
                const int q1 = i % P1;
                const int r = i / P1;
                const int q2 = DIM > 1 ? r % P2 : 0;
                const int q3 = DIM > 2 ? r / P2 : 0;
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
                v[u] = __ldg(grid + gi);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < ncell) patch[i] = v[u];
            }
        }
        __syncthreads();
        // point records are staged slice by slice into shared memory with
        // all threads' loads in flight at once (a per-thread prefetch chain
        // cannot cover the DRAM latency at this loop length)
        for (int s0 = 0; s0 < cnt; s0 += kInterpSlice) {
        const int sn = min(kInterpSlice, cnt - s0);
        __syncthreads();
        {
            // four independent 256-bit loads per thread, then the stores
            Rec tmp[4];
            const int nt = blockDim.x;
#pragma unroll
            for (int u = 0; u < 4; ++u) tmp[u] = load_rec(a.rec, start + s0 + min(tid + u * nt, sn - 1));
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (tid + u * nt < sn) s_rec[tid + u * nt] = tmp[u];
        }
        __syncthreads();
        for (int kk = tid; kk < sn; kk += blockDim.x) {
            const Rec rc = s_rec[kk];
            T r1[W], r2[W], r3[W];
            int i1 = kernel_row<T, W>(rc.g[0], a.k, r1);
            const int o1 = (i1 < 0 ? i1 + n1 : i1) - lo1;
            int o2 = 0, o3 = 0;
            if (DIM > 1) {
                const int i2 = kernel_row<T, W>(rc.g[1], a.k, r2);
                o2 = (i2 < 0 ? i2 + n2 : i2) - lo2;
            }
            if (DIM > 2) {
                const int i3 = kernel_row<T, W>(rc.g[2], a.k, r3);
                o3 = (i3 < 0 ? i3 + n3 : i3) - lo3;
            }
            T are = 0, aim = 0;
            if (DIM == 1) {
#pragma unroll
                for (int m1 = 0; m1 < W; ++m1) {
                    const C v = patch[o1 + m1];
                    are = fma(r1[m1], v.x, are);
                    aim = fma(r1[m1], v.y, aim);
                }
            } else if (DIM == 2) {
                const C *base = patch + o2 * P1 + o1;
                // rows not unrolled: keeps ~W row loads in flight instead of
                // W^2 (register budget -> 3 CTAs per SM)
#pragma unroll 1
                for (int m2 = 0; m2 < W; ++m2) {
                    T pre = 0, pim = 0;
#pragma unroll
                    for (int m1 = 0; m1 < W; ++m1) {
                        const C v = base[m2 * P1 + m1];
                        pre = fma(r1[m1], v.x, pre);
                        pim = fma(r1[m1], v.y, pim);
                    }
                    T w2 = r2[0];
#pragma unroll
                    for (int q = 1; q < W; ++q) w2 = (q == m2) ? r2[q] : w2;
                    are = fma(w2, pre, are);
                    aim = fma(w2, pim, aim);
                }
            } else {
                const C *base = patch + (o3 * P2 + o2) * P1 + o1;
                // planes not unrolled (W^2 body per plane; fits the registers)
#pragma unroll 1
                for (int m3 = 0; m3 < W; ++m3) {
                    T p3re = 0, p3im = 0;
#pragma unroll
                    for (int m2 = 0; m2 < W; ++m2) {
                        T pre = 0, pim = 0;
#pragma unroll
                        for (int m1 = 0; m1 < W; ++m1) {
                            const C v = base[(m3 * P2 + m2) * P1 + m1];
                            pre = fma(r1[m1], v.x, pre);
                            pim = fma(r1[m1], v.y, pim);
                        }
                        p3re = fma(r2[m2], pre, p3re);
                        p3im = fma(r2[m2], pim, p3im);
                    }
                    T w3 = r3[0];
#pragma unroll
                    for (int q = 1; q < W; ++q) w3 = (q == m3) ? r3[q] : w3;
                    are = fma(w3, p3re, are);
                    aim = fma(w3, p3im, aim);
                }
            }
            reinterpret_cast<C *>(cout)[(int64_t)t * a.M + rc.j] = C{are, aim};
        }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Asynchronous bulk copies (cp.async.bulk, global -> shared) completing on an
// mbarrier: the copy engine moves bytes without registers or LSU issue slots.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 16-byte store that asks L2 to keep the line (scattered outputs of one
// target chunk merge into whole sectors there before write-back)
__device__ __forceinline__ void st_keep(double2 *p, double2 v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void st_keep(float2 *p, float2 v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(policy)
                 : "memory");
}

// ---------------------------------------------------------------------------
// Batched 2D spreader, y-rolling owner-computes (ntransf > 1, float32): lanes
// are transforms.  A warp item is (strip of kRollBX owned columns, segment of
// kRollSeg owned rows, 32-transform group).  It walks the ORIGIN rows
// y0 - (w - 1) .. y0 + SEG - 1 in order; the points of one origin row whose
// origin column lies in [x0 - (w - 1), x0 + BX) come from <= 3 contiguous
// key ranges (the window crosses at most one bin edge and the wrap), listed
// once per item.  They are staged in pieces of kRollNB points (kernel rows
// + the group's 32 strengths, cp.async.bulk on an mbarrier, one piece
// ahead, pieces spanning rows) and each adds its w x w footprint into a ring
// of w output rows held in registers (acc[dy][col], owned columns only, one
// static dispatch per point on the origin column).  When the origin row
// advances past row y, row y is complete: its owned cells are stored once
// (no memset, no atomics) and the ring shifts.  Per point this is one warp
// visit per strip it reaches (1 + (w - 1) / BX) and (SEG + w - 1) / SEG row
// passes, against w / 2 + 1 item visits of k_spread_b2own.  Same sort keys
// and scratch as k_spread_b2own (cell-resolution keys over 16 x 16 bins,
// cperm, tab).  Reference: spreadinterp.py:354-368 (_spread_sub_2d), one
// pass per transform there (bench.py c5 runs 64 single transforms).
constexpr int kRollBX = 8;    // owned columns per strip
constexpr int kRollSeg = 32;  // owned rows per segment
constexpr int kRollNB = 16;   // staged points per piece
template <int W>
struct RollCfg {
    static constexpr int R = kRollSeg + W - 1;  // origin rows per item
    static constexpr int NC = kRollBX + W - 1;  // window cells per row
    static constexpr int RUNS = 4;              // run slots per row (<= 3 used)
    static constexpr uint32_t I1OFF = 2 * W * sizeof(float);  // PtRows2<W>::i1
    static constexpr size_t STAGE = (size_t)kRollNB * (sizeof(PtRows2<W>) + 32 * sizeof(float2));
    static constexpr size_t TABLE = (size_t)R * RUNS * 2 * sizeof(int) + (size_t)R * sizeof(int);
    static constexpr size_t WARP = 2 * STAGE + (TABLE + 127) / 128 * 128;
    static_assert((size_t)R * NC * 2 * sizeof(int) <= 2 * STAGE, "key ranges alias the stages");
};
template <int W>
constexpr size_t b2roll_smem_bytes() { return 4 * RollCfg<W>::WARP; }
__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// r1[W], r2[W] of one staged PtRows2<W> (16-byte aligned, 16-byte vectors)
template <int W>
__device__ __forceinline__ void lds_rows(uint32_t a, float *r1, float *r2) {
    constexpr int NV = (2 * W + 3) / 4;
    static_assert(NV * 16 <= (int)sizeof(PtRows2<W>), "vector loads stay inside the entry");
    float f[NV * 4];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const float4 q = lds_f4(a + 16 * i);
        f[4 * i] = q.x;
        f[4 * i + 1] = q.y;
        f[4 * i + 2] = q.z;
        f[4 * i + 3] = q.w;
    }
#pragma unroll
    for (int m = 0; m < W; ++m) {
        r1[m] = f[m];
        r2[m] = f[W + m];
    }
}
// grids this kernel handles: the window of one strip / segment must not wrap
// onto itself
template <int W>
__host__ __device__ inline bool b2roll_fits(int n1, int n2) { return n1 >= kRollBX + W - 1 && n2 >= kRollSeg + W - 1; }

// x-offset dispatch of the y-rolling batched spreader as a compare tree: the
// offset CS selects which of the point's w columns land on the strip's owned
// columns (static register indices).  (A switch compiled to a two-level
// jump table here -- an indexed constant load and an indirect branch on the
// critical path of every point.)
#ifndef ESN_B2_TAIL
#define ESN_B2_TAIL 1
#endif
#ifndef ESN_B2_TAIL_DIV
#define ESN_B2_TAIL_DIV 4
#endif
#ifndef ESN_ROLL_TREE
#define ESN_ROLL_TREE 1
#endif
template <typename T, int W, int BXS, int LO, int HI>
__device__ __forceinline__ void roll_apply(int cs, typename Cx<T>::type (&acc)[W][BXS],
                                           const typename Cx<T>::type (&v)[W], const T (&r1)[W]) {
    if constexpr (LO == HI) {
        constexpr int XL = LO - (W - 1);
#pragma unroll
        for (int m = 0; m < W; ++m) {
            if (XL + m >= 0 && XL + m < BXS) {
#pragma unroll
                for (int dy = 0; dy < W; ++dy) acc[dy][XL + m] = cfma(v[dy], r1[m], acc[dy][XL + m]);
            }
        }
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (cs <= MID) roll_apply<T, W, BXS, LO, MID>(cs, acc, v, r1);
        else roll_apply<T, W, BXS, MID + 1, HI>(cs, acc, v, r1);
    }
}

template <typename T, int W>
__global__ void __launch_bounds__(128, 3) k_spread_b2roll(SpreadArgs<T> a, const T *cperm, const PtRows2<W> *tab) {
    if (a.imb && *a.imb) return;  // imbalanced bins: the RED-flush kernel launched next takes over
    static_assert(sizeof(T) == 4, "float32 plans");
    using C = typename Cx<T>::type;
    using Cfg = RollCfg<W>;
    constexpr int BXS = kRollBX, NB = kRollNB, H = W - 1, NC = Cfg::NC, R = Cfg::R, RUNS = Cfg::RUNS;
    constexpr uint32_t TB = sizeof(PtRows2<W>), CB = 32 * sizeof(C);
    constexpr size_t STAGE = Cfg::STAGE;
    static_assert(NC <= 32, "one lane per window column");
    static_assert(TB % 16 == 0 && CB % 16 == 0, "bulk copies move 16-byte multiples");
    extern __shared__ __align__(128) unsigned char roll_smem[];
    __shared__ uint64_t s_bar[4][2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char *wbase = roll_smem + wid * Cfg::WARP;
    int *run_src = reinterpret_cast<int *>(wbase + 2 * STAGE);  // [R * RUNS]
    int *run_end = run_src + R * RUNS;                            // [R * RUNS]
    int *rowend = run_end + R * RUNS;                             // [R] slots through row r
    int *se = reinterpret_cast<int *>(wbase);                     // [R][NC][2] (item setup only)
    uint64_t *bar = s_bar[wid];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int n1 = a.g.n[0], n2 = a.g.n[1], nb0 = a.g.nb[0];
    // bins are 16 x 16 cells on this path (batched_owner checks bs)
    constexpr int bx = Batch2Cfg<float, W>::BX, by = Batch2Cfg<float, W>::BY;
    const int ngroups = (a.ntransf + 31) / 32;
    // Segments: full ones (kRollSeg rows) first, then HALF segments over the
    // last 1 / ESN_B2_TAIL_DIV of the rows.  Items come off one queue in this
    // order, so every warp ends on a short item and the tail in which warps
    // idle is shorter (c5: 8192 items of ~190 us on 1776 resident warps left
    // a tail of ~half an item; the half segments pay (16 + w - 1) / 16
    // instead of (32 + w - 1) / 32 origin rows per owned row).  The gain
    // depends on how the full items divide into waves of resident warps (c5
    // spread + permute, ms: none 1.085; last 1/2 1.048, 1/3 1.062, 1/4 1.0415,
    // 1/5 1.058, 1/6 1.097, 1/8 1.13).  ESN_B2_TAIL=0 in the build keeps
    // equal segments.
    const int nstrips = (n1 + BXS - 1) / BXS;
    const int nfull = n2 / kRollSeg;
    const int nbig = (ESN_B2_TAIL && nfull >= 10) ? nfull - nfull / ESN_B2_TAIL_DIV : nfull;
    const int rows_big = nbig * kRollSeg;
    constexpr int HSEG = (ESN_B2_TAIL) ? kRollSeg / 2 : kRollSeg;
    const int nsegs = nbig + (n2 - rows_big + HSEG - 1) / HSEG;
    const int nitems = nstrips * nsegs * ngroups;
    uint32_t par0 = 0, par1 = 0;  // mbarrier phase parity per buffer
    int next = 0;
    if (lane == 0) next = atomicAdd(a.work, 1);
    for (;;) {
        const int item = __shfl_sync(0xffffffffu, next, 0);
        if (item >= nitems) break;
        if (lane == 0) next = atomicAdd(a.work, 1);
        const int tg = item % ngroups;
        const int sid = item / ngroups;
        const int strip = sid % nstrips, seg = sid / nstrips;
        const int x0 = strip * BXS;
        const int y0 = seg < nbig ? seg * kRollSeg : rows_big + (seg - nbig) * HSEG;
        const int yend = min(y0 + (seg < nbig ? kRollSeg : HSEG), n2);  // owned rows y0 .. yend - 1
        const int nrows = yend - (y0 - H);         // origin rows of this item (<= R)
        int xb = x0 - H;
        while (xb < 0) xb += n1;  // window column k: (xb + k) mod n1
        int yb = y0 - H;
        while (yb < 0) yb += n2;
        // item setup 1: key range [s, e) of every (origin row, window cell),
        // all loads in flight at once
        for (int p = lane; p < nrows * NC; p += 32) {
            const int r = p / NC, k = p - r * NC;
            int yr = yb + r, xr = xb + k;
            if (yr >= n2) yr -= n2;
            if (xr >= n1) xr -= n1;
            const int key = (((yr / by) * nb0 + xr / bx) * by + (yr % by)) * bx + (xr % bx);
            se[2 * p] = a.kstart[key];
            se[2 * p + 1] = a.kstart[key + 1];
        }
        __syncwarp();
        // item setup 2: per row, its contiguous runs and the running slot count
        int tot = 0;
        for (int r = 0; r < nrows; ++r) {
            int s = 0, e = 0;
            if (lane < NC) {
                s = se[2 * (r * NC + lane)];
                e = se[2 * (r * NC + lane) + 1];
            }
            const int eprev = __shfl_up_sync(0xffffffffu, e, 1);
            const bool start = lane < NC && (lane == 0 || s != eprev);
            const unsigned smask = __ballot_sync(0xffffffffu, start);
            const bool last = lane < NC && (lane == NC - 1 || ((smask >> (lane + 1)) & 1u));
            const int idx = __popc(smask & ((2u << lane) - 1u)) - 1;  // run of this lane
            if (start && idx < RUNS) run_src[r * RUNS + idx] = s;
            if (last && idx < RUNS) run_end[r * RUNS + idx] = e;
            int cnt = lane < NC ? e - s : 0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
            const int nr = __popc(smask);
            if (lane < RUNS && lane >= nr) {  // unused run slots are empty
                run_src[r * RUNS + lane] = 0;
                run_end[r * RUNS + lane] = 0;
            }
            tot += cnt;
            if (lane == 0) rowend[r] = tot;
        }
        __syncwarp();
        const C *cg = reinterpret_cast<const C *>(cperm) + (int64_t)tg * a.M * 32;
        // producer state (lane 0): run pr (flat over rows), offset po in it
        int pr = 0, po = 0, issued = 0;
        auto issue = [&](int buf) -> int {  // next piece of up to NB slots into buf
            const int n = min(NB, tot - issued);
            if (lane == 0) {
                unsigned char *dst = wbase + buf * STAGE;
                mbar_expect_tx(&bar[buf], (uint32_t)n * (TB + CB));
                int slot = 0;
                while (slot < n) {
                    const int s0 = run_src[pr], len = run_end[pr] - s0 - po;
                    const int take = min(len, n - slot);
                    if (take > 0) {
                        const int src = s0 + po;
                        bulk_g2s(dst + slot * TB, tab + src, (uint32_t)take * TB, &bar[buf]);
                        bulk_g2s(dst + NB * TB + slot * CB, cg + (int64_t)src * 32, (uint32_t)take * CB, &bar[buf]);
                        slot += take;
                        po += take;
                    }
                    if (po >= run_end[pr] - s0) {
                        ++pr;
                        po = 0;
                    }
                }
            }
            issued += n;
            return n;
        };
        C acc[W][BXS];
#pragma unroll
        for (int r = 0; r < W; ++r)
#pragma unroll
            for (int x = 0; x < BXS; ++x) acc[r][x] = C{(T)0, (T)0};
        const bool vec = (n1 % 2) == 0 && x0 + BXS <= n1;
        const int t = tg * 32 + lane;
        int ycur = y0 - H;    // origin row of the next slot
        int rnext = rowend[0];  // slots through row ycur
        int rr = 0;
        // origin row ycur done: output row ycur is complete -> store, shift
        auto advance_row = [&]() {
            if (ycur >= y0 && t < a.ntransf) {
                C *dst = reinterpret_cast<C *>(a.grid) + (int64_t)t * a.gstride + (int64_t)ycur * n1 + x0;
                if (a.accumulate) {
#pragma unroll
                    for (int x = 0; x < BXS; ++x)
                        if (x0 + x < n1 && (acc[0][x].x != (T)0 || acc[0][x].y != (T)0)) red_add(dst + x, acc[0][x]);
                } else if (vec) {
#pragma unroll
                    for (int x = 0; x < BXS; x += 2)
                        *reinterpret_cast<float4 *>(dst + x) = make_float4(acc[0][x].x, acc[0][x].y, acc[0][x + 1].x,
                                                                           acc[0][x + 1].y);
                } else {
#pragma unroll
                    for (int x = 0; x < BXS; ++x)
                        if (x0 + x < n1) dst[x] = acc[0][x];
                }
            }
#pragma unroll
            for (int r = 0; r + 1 < W; ++r)
#pragma unroll
                for (int x = 0; x < BXS; ++x) acc[r][x] = acc[r + 1][x];
#pragma unroll
            for (int x = 0; x < BXS; ++x) acc[W - 1][x] = C{(T)0, (T)0};
            ++ycur;
            ++rr;
            rnext = rr < nrows ? rowend[rr] : 0x7fffffff;
        };
        int q = 0, buf = 0;
        int cn = tot > 0 ? issue(0) : 0;
        while (cn > 0) {
            const int nn = issued < tot ? issue(buf ^ 1) : 0;  // the other buffer's reader is done
            mbar_wait(&bar[buf], buf ? par1 : par0);
            if (buf) par1 ^= 1u; else par0 ^= 1u;
            // 32-bit shared addresses (explicit ld.shared): one register per
            // pointer, nothing for the compiler to re-derive inside the loop
            const uint32_t sb = smem_u32(wbase) + (uint32_t)(buf * STAGE);
            const uint32_t cb = sb + NB * TB + lane * (uint32_t)sizeof(C);
            // the piece in same-row segments: the hot loop carries no row logic
            for (int k0 = 0; k0 < cn;) {
                while (q >= rnext) advance_row();
                const int k1 = min(cn, k0 + (rnext - q));
                q += k1 - k0;
                // the origin column of the next point is loaded one point ahead,
                // so the dispatch of point k resolves while its rows load
                int i1n = lds_s32(sb + k0 * TB + Cfg::I1OFF);
#pragma unroll 1
            for (int k = k0; k < k1; ++k) {
                const int i1 = i1n;
                if (k + 1 < k1) i1n = lds_s32(sb + (k + 1) * TB + Cfg::I1OFF);
                T r1[W], r2[W];
                lds_rows<W>(sb + k * TB, r1, r2);
                const float2 cc = lds_f2(cb + k * CB);
                C v[W];
#pragma unroll
                for (int dy = 0; dy < W; ++dy) v[dy] = cmul(cc, r2[dy]);
                int cs = i1 - xb;
                if (cs < 0) cs += n1;
#define ESN_ROLL_CASE(CS)                                                                 \
    case CS:                                                                              \
        if constexpr (CS < NC) {                                                          \
            _Pragma("unroll") for (int m = 0; m < W; ++m) {                               \
                constexpr int XL = CS - H;                                                \
                if (XL + m >= 0 && XL + m < BXS) {                                        \
                    _Pragma("unroll") for (int dy = 0; dy < W; ++dy) {                    \
                        acc[dy][XL + m] = cfma(v[dy], r1[m], acc[dy][XL + m]);            \
                    }                                                                     \
                }                                                                         \
            }                                                                             \
        }                                                                                 \
        break;
#if ESN_ROLL_TREE
                if ((unsigned)cs < (unsigned)NC) roll_apply<T, W, BXS, 0, NC - 1>(cs, acc, v, r1);
#else
                switch (cs) {
                    ESN_ROLL_CASE(0) ESN_ROLL_CASE(1) ESN_ROLL_CASE(2) ESN_ROLL_CASE(3)
                    ESN_ROLL_CASE(4) ESN_ROLL_CASE(5) ESN_ROLL_CASE(6) ESN_ROLL_CASE(7)
                    ESN_ROLL_CASE(8) ESN_ROLL_CASE(9) ESN_ROLL_CASE(10) ESN_ROLL_CASE(11)
                    ESN_ROLL_CASE(12) ESN_ROLL_CASE(13) ESN_ROLL_CASE(14) ESN_ROLL_CASE(15)
                    ESN_ROLL_CASE(16) ESN_ROLL_CASE(17)
                    default:
                        break;
                }
#endif
#undef ESN_ROLL_CASE
            }
                k0 = k1;
            }
            __syncwarp();
            buf ^= 1;
            cn = nn;
        }
        while (rr < nrows) advance_row();  // trailing rows (and items with no points)
        __syncwarp();  // setup of the next item overwrites the stages and tables
    }
}

// One unit of interpolation work: a slice of one subproblem's point records.
struct InterpUnit {
    int valid, t, start, n;   // transform, first record, records in the slice
    int lo1, lo2, lo3, pb;    // patch origin and the patch buffer holding it
};

// Pipelined tile interpolator (same arithmetic and output as k_interp_tile).
// Work streams through a CTA as units (subproblem slices) in a two-slot
// ring.  Warp 0 also produces: it queues unit i+1's records -- and, on a new
// subproblem, its periodic patch row by row -- as bulk copies into the other
// slot ("full" mbarrier, transaction-counted) once every warp has released
// that slot ("empty" mbarrier, one arrival per warp).  No block-wide barrier:
// a warp that finishes its share of a unit moves on to the next one, and
// DRAM latency overlaps the fp64 work.  Records are fetched with an
// evict-first L2 policy and outputs stored evict-last, so the scattered
// outputs of one target chunk (see the plan's chunked sort key) merge into
// whole sectors in L2.  Requires complex128 cells (16-byte rows) and
// P_d <= n_d (each patch row wraps at most once).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256, interp_minb<DIM, W>())
    k_interp_bulk(SpreadArgs<T> a, T *cout, const T *gridp, int slice, int dprod, int pitch1, int R) {
    using C = typename Cx<T>::type;
    extern __shared__ __align__(16) unsigned char bulk_smem[];
    constexpr int RMAX = 4;  // record slots (R <= RMAX); the patches keep two
    __shared__ uint64_t s_full[RMAX], s_empty[RMAX];
    __shared__ InterpUnit s_unit[RMAX];
    __shared__ int s_plast[2];  // (producer) last unit that reads each patch slot
    // producer state, touched by lane 0 of warp 0 only (kept in shared
    // memory so it costs the compute threads no registers)
    __shared__ int s_prod[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    const int P1 = a.g.bs[0] + W - 1;
    const int P2 = DIM > 1 ? a.g.bs[1] + W - 1 : 1;
    const int P3 = DIM > 2 ? a.g.bs[2] + W - 1 : 1;
    // pitch1 >= P1: patch row pitch in cells (a multiple of 8 cells = 128
    // bytes keeps a quarter-warp that runs off a bin row's end onto the next
    // row on distinct banks)
    const int ncell = pitch1 * P2 * P3;
    Rec *const rec0 = reinterpret_cast<Rec *>(bulk_smem);              // R x slice records
    C *const patch0 = reinterpret_cast<C *>(rec0 + R * slice);         // 2 x ncell cells
    const int nsub = *a.nsub;
    const int nwork = nsub * a.ntransf;
    const int nbins_geo = a.g.nb[0] * a.g.nb[1] * a.g.nb[2];
    const C *gridc = reinterpret_cast<const C *>(gridp);
    int &p_start = s_prod[0], &p_cnt = s_prod[1], &p_off = s_prod[2], &p_pb = s_prod[3];
    int &p_t = s_prod[4], &p_lo1 = s_prod[5], &p_lo2 = s_prod[6], &p_lo3 = s_prod[7];
    int p_next = 0;  // (lane 0 of warp 0) work index claimed one subproblem ahead

    // producer warp: choose unit k and queue its copies into slot k mod R
    auto produce = [&](int k) -> int {
        const int rb = k % R;
        if (k >= R) mbar_wait(&s_empty[rb], ((k / R) - 1) & 1);  // every warp released unit k - R
        int fresh = 0, valid = 0, guard = -1;
        InterpUnit u;
        if (lane == 0) {
            while (p_off >= p_cnt) {
                const int s = p_next;
                if (s >= nwork) { p_cnt = -1; break; }
                p_next = atomicAdd(a.work, 1);
                p_t = s / nsub;
                const int4 sp = a.subprob[s - p_t * nsub];
                const int bin = sp.x % nbins_geo;  // geometric bin (key major part = target chunk)
                p_start = sp.y; p_cnt = sp.z; p_off = 0; fresh = 1;
                const int b1 = bin % a.g.nb[0];
                const int b2 = DIM > 1 ? (bin / a.g.nb[0]) % a.g.nb[1] : 0;
                const int b3 = DIM > 2 ? bin / (a.g.nb[0] * a.g.nb[1]) : 0;
                p_lo1 = b1 * a.g.bs[0]; p_lo2 = b2 * a.g.bs[1]; p_lo3 = b3 * a.g.bs[2];
            }
            if (p_cnt < 0) {
                u.valid = 0;
                p_cnt = 0; p_off = 0; fresh = 0;
            } else {
                if (fresh) {
                    p_pb ^= 1;  // the patch slot the previous subproblem did not use
                    // ... whose last reader (the subproblem before that) may
                    // still be in flight when the ring is deeper than two
                    if (s_plast[p_pb] > k - R) guard = s_plast[p_pb];
                }
                s_plast[p_pb] = k;
                u.valid = 1; u.t = p_t; u.start = p_start + p_off; u.n = min(slice, p_cnt - p_off);
                u.lo1 = p_lo1; u.lo2 = p_lo2; u.lo3 = p_lo3; u.pb = p_pb;
                p_off += slice;
            }
            valid = u.valid;
            s_unit[rb] = u;
            // arrival (release) publishes s_unit[rb]; the phase completes when
            // the copies' bytes have landed
            mbar_expect_tx(&s_full[rb],
                           valid ? (uint32_t)u.n * sizeof(Rec) + (fresh ? (uint32_t)(P1 * P2 * P3) * sizeof(C) : 0u)
                                 : 0u);
        }
        fresh = __shfl_sync(0xffffffffu, fresh, 0);
        valid = __shfl_sync(0xffffffffu, valid, 0);
        guard = __shfl_sync(0xffffffffu, guard, 0);
        if (!valid) return 0;
        // unit `guard` is released when its slot's empty barrier completes
        // phase guard / R (unit guard + R is not produced yet: unambiguous)
        if (guard >= 0) mbar_wait(&s_empty[guard % R], (guard / R) & 1);
        if (lane == 0)
            bulk_g2s_hint(rec0 + rb * slice, a.rec + u.start, (uint32_t)u.n * sizeof(Rec), &s_full[rb],
                          policy_evict_first());  // records stream through once
        if (fresh) {
            __syncwarp();
            const int t = p_t, lo1 = p_lo1, lo2 = p_lo2, lo3 = p_lo3, pb = p_pb;
            const C *grid = gridc + (int64_t)t * a.gstride;
            const int head = min(P1, n1 - lo1);  // cells before the x wrap
            for (int r = lane; r < P2 * P3; r += 32) {
                const int q2 = DIM > 1 ? r % P2 : 0;
                const int q3 = DIM > 2 ? r / P2 : 0;
                int g2 = lo2 + q2, g3 = lo3 + q3;
                if (g2 >= n2) g2 -= n2;
                if (g3 >= n3) g3 -= n3;
                const C *row = grid + ((int64_t)g3 * n2 + g2) * n1;
                C *dst = patch0 + pb * ncell + r * pitch1;
                bulk_g2s(dst, row + lo1, (uint32_t)head * sizeof(C), &s_full[rb]);
                if (head < P1) bulk_g2s(dst + head, row, (uint32_t)(P1 - head) * sizeof(C), &s_full[rb]);
            }
        }
        return 1;
    };

    if (tid == 0) {
        p_start = p_cnt = p_off = p_t = p_lo1 = p_lo2 = p_lo3 = 0;
        p_pb = 1;
        s_plast[0] = s_plast[1] = -(1 << 30);
        for (int r = 0; r < R; ++r) {
            mbar_init(&s_full[r], 1);
            mbar_init(&s_empty[r], dprod ? nwarps - 1 : nwarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // dprod: the last warp only produces (queues unit k + 1 as soon as every
    // consumer released unit k - 1); else warp 0 produces between its own
    // units, so a late warp 0 shortened the prefetch distance
    const int pw = dprod ? nwarps - 1 : 0;
    if (warp == pw && lane == 0) p_next = atomicAdd(a.work, 1);  // (the producer's own claim)
    __syncthreads();
    const int cthreads = dprod ? blockDim.x - 32 : blockDim.x;
    if (dprod && warp == pw) {
        for (int k = 0;; ++k)
            if (!produce(k)) break;
        return;
    }
    int producing = warp == pw ? produce(0) : 0;
    const uint64_t keep = policy_evict_last();
    for (int k = 0;; ++k) {
        const int rb = k % R;
        if (producing) producing = produce(k + 1);
        mbar_wait(&s_full[rb], (k / R) & 1);
        const InterpUnit u = s_unit[rb];
        if (!u.valid) break;
        const Rec *recs = rec0 + rb * slice;
        const C *patch = patch0 + u.pb * ncell;
        // a quarter-warp's eight 32-byte records: lanes 0-3 fetch the first
        // half then the second, lanes 4-7 the second then the first, so each
        // 128-bit load covers eight distinct 16-byte bank groups (all-first
        // halves sit on four of them: 2-way conflicts, 8-way for a 32-bit
        // load of j)
        const int hsel = (lane >> 2) & 1;
        for (int kk = tid; kk < u.n; kk += cthreads) {
            Rec rc;
            {
                // (no alignment assumed beyond 16 bytes: the dynamic segment
                // follows the static words)
                const uint32_t r0 = smem_u32(recs + kk);
                long long ax, ay, bx, by;
                asm volatile("ld.shared.v2.s64 {%0, %1}, [%2];" : "=l"(ax), "=l"(ay) : "r"(r0 + 16u * hsel));
                asm volatile("ld.shared.v2.s64 {%0, %1}, [%2];" : "=l"(bx), "=l"(by) : "r"(r0 + 16u - 16u * hsel));
                rc.g[0] = __longlong_as_double(hsel ? bx : ax);
                rc.g[1] = __longlong_as_double(hsel ? by : ay);
                rc.g[2] = __longlong_as_double(hsel ? ax : bx);
                rc.j = (int)(unsigned)((hsel ? ay : by) & 0xffffffffll);
            }
            T r1[W], r2[W], r3[W];
            const int i1 = kernel_row<T, W>(rc.g[0], a.k, r1);
            const int o1 = (i1 < 0 ? i1 + n1 : i1) - u.lo1;
            int o2 = 0, o3 = 0;
            if (DIM > 1) {
                const int i2 = kernel_row<T, W>(rc.g[1], a.k, r2);
                o2 = (i2 < 0 ? i2 + n2 : i2) - u.lo2;
            }
            if (DIM > 2) {
                const int i3 = kernel_row<T, W>(rc.g[2], a.k, r3);
                o3 = (i3 < 0 ? i3 + n3 : i3) - u.lo3;
            }
            T are = 0, aim = 0;
            const C *base = patch + (o3 * P2 + o2) * pitch1 + o1;
            // 2D: rows unrolled (static r2 index; a select chain per row cost
            // 2 (w - 1) instructions); 3D keeps rolled loops (registers)
            constexpr int U2 = DIM == 2 ? W : 1;
#pragma unroll 1
            for (int m3 = 0; m3 < (DIM > 2 ? W : 1); ++m3) {
                T p3re = 0, p3im = 0;
#pragma unroll U2
                for (int m2 = 0; m2 < (DIM > 1 ? W : 1); ++m2) {
                    T pre = 0, pim = 0;
#pragma unroll
                    for (int m1 = 0; m1 < W; ++m1) {
                        const C v = base[(m3 * P2 + m2) * pitch1 + m1];
                        pre = fma(r1[m1], v.x, pre);
                        pim = fma(r1[m1], v.y, pim);
                    }
                    if (DIM > 1) {
                        T w2 = r2[0];
#pragma unroll
                        for (int q = 1; q < W; ++q) w2 = (q == m2) ? r2[q] : w2;
                        p3re = fma(w2, pre, p3re);
                        p3im = fma(w2, pim, p3im);
                    } else {
                        p3re = pre;
                        p3im = pim;
                    }
                }
                if (DIM > 2) {
                    T w3 = r3[0];
#pragma unroll
                    for (int q = 1; q < W; ++q) w3 = (q == m3) ? r3[q] : w3;
                    are = fma(w3, p3re, are);
                    aim = fma(w3, p3im, aim);
                } else {
                    are = p3re;
                    aim = p3im;
                }
            }
            st_keep(reinterpret_cast<C *>(cout) + (int64_t)u.t * a.M + rc.j, C{are, aim}, keep);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[rb]);
    }
}

// ---------------------------------------------------------------------------
// Thread-per-point interpolator (spreadinterp.py:442-507) over the finely
// sorted records: the 32 lanes of a warp hold 32 consecutive points of the
// same few sub-cells, so each of the w^d gathers is a near-broadcast of a
// few cache lines; separable weighted sum in registers (w^(d-1) row partial
// sums), output in ORIGINAL point order (spreadinterp.py:453).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256, 2) k_interp_thread(SpreadArgs<T> a, T *cout, const T *gridp) {
    using C = typename Cx<T>::type;
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.M;
         k += (int64_t)gridDim.x * blockDim.x) {
        const Rec rc = load_rec(a.rec, k);
        T r1[W], r2[W], r3[W];
        int ix1[W];
        const int i1 = kernel_row<T, W>(rc.g[0], a.k, r1);
#pragma unroll
        for (int m = 0; m < W; ++m) ix1[m] = wrap_once(i1 + m, n1);
        int i2 = 0, i3 = 0;
        if (DIM > 1) i2 = kernel_row<T, W>(rc.g[1], a.k, r2);
        if (DIM > 2) i3 = kernel_row<T, W>(rc.g[2], a.k, r3);
        for (int t = 0; t < a.ntransf; ++t) {
            const C *grid = reinterpret_cast<const C *>(gridp) + (int64_t)t * a.gstride;
            T are = 0, aim = 0;
            if (DIM == 1) {
#pragma unroll
                for (int m1 = 0; m1 < W; ++m1) {
                    const C v = __ldg(grid + ix1[m1]);
                    are = fma(r1[m1], v.x, are);
                    aim = fma(r1[m1], v.y, aim);
                }
            } else if (DIM == 2) {
#pragma unroll
                for (int m2 = 0; m2 < W; ++m2) {
                    const C *row = grid + (int64_t)wrap_once(i2 + m2, n2) * n1;
                    T pre = 0, pim = 0;
#pragma unroll
                    for (int m1 = 0; m1 < W; ++m1) {
                        const C v = __ldg(row + ix1[m1]);
                        pre = fma(r1[m1], v.x, pre);
                        pim = fma(r1[m1], v.y, pim);
                    }
                    are = fma(r2[m2], pre, are);
                    aim = fma(r2[m2], pim, aim);
                }
            } else {
#pragma unroll 1
                for (int m3 = 0; m3 < W; ++m3) {
                    const C *plane = grid + (int64_t)wrap_once(i3 + m3, n3) * n2 * n1;
                    T p3re = 0, p3im = 0;
#pragma unroll
                    for (int m2 = 0; m2 < W; ++m2) {
                        const C *row = plane + (int64_t)wrap_once(i2 + m2, n2) * n1;
                        T pre = 0, pim = 0;
#pragma unroll
                        for (int m1 = 0; m1 < W; ++m1) {
                            const C v = __ldg(row + ix1[m1]);
                            pre = fma(r1[m1], v.x, pre);
                            pim = fma(r1[m1], v.y, pim);
                        }
                        p3re = fma(r2[m2], pre, p3re);
                        p3im = fma(r2[m2], pim, p3im);
                    }
                    // r3 is indexed by the runtime m3: select from registers
                    T w3 = r3[0];
#pragma unroll
                    for (int q = 1; q < W; ++q) w3 = (q == m3) ? r3[q] : w3;
                    are = fma(w3, p3re, are);
                    aim = fma(w3, p3im, aim);
                }
            }
            reinterpret_cast<C *>(cout)[(int64_t)t * a.M + rc.j] = C{are, aim};
        }
    }
}

// ---------------------------------------------------------------------------
// Lane-group interpolator (spreadinterp.py:442-507).  A group of G lanes
// (G = 8 for w <= 8, 16 for w <= 16) handles one sorted point: lane m owns
// ordinate m along x, evaluates r1[m], r2[m], r3[m] itself, and walks the
// w^(d-1) rows reading one contiguous run of w cells per row (coalesced
// 128-byte segments instead of 32 scattered lanes).  Row weights come from
// the owning lane by shuffle; a butterfly reduction finishes the sum, and
// the result is written in ORIGINAL point order (spreadinterp.py:453).
template <typename T, int DIM, int W>
__global__ void __launch_bounds__(256) k_interp_group(SpreadArgs<T> a, T *cout, const T *gridp, int chunk) {
    using C = typename Cx<T>::type;
    constexpr int G = W <= 8 ? 8 : 16;
    constexpr int PPW = 32 / G;  // points per warp per step
    const int n1 = a.g.n[0], n2 = a.g.n[1], n3 = a.g.n[2];
    const int lane = threadIdx.x & 31, gl = lane % G, gbase = lane - gl;
    const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int mm = gl < W ? gl : W - 1;
    T cf[W + 4];
    kernel_col<T, W>(a.k, mm, cf);
    // each CTA walks contiguous chunks of the sorted order so a bin's patch
    // stays hot in L1 while all of its points are interpolated
    for (int64_t c0 = (int64_t)blockIdx.x * chunk; c0 < a.M; c0 += (int64_t)gridDim.x * chunk) {
        const int64_t c1 = min(c0 + chunk, a.M);
        for (int64_t k0 = c0 + (int64_t)warp * PPW; k0 < c1; k0 += (int64_t)nwarp * PPW) {
            const int64_t k = k0 + lane / G;
            const bool live = k < c1;
            const Rec rc = load_rec(a.rec, live ? k : c1 - 1);
            int i1, i2 = 0, i3 = 0;
            const T r1 = kernel_one<T, W>(rc.g[0], mm, cf, a.k, &i1);
            T r2 = (T)1, r3 = (T)1;
            if (DIM > 1) r2 = kernel_one<T, W>(rc.g[1], mm, cf, a.k, &i2);
            if (DIM > 2) r3 = kernel_one<T, W>(rc.g[2], mm, cf, a.k, &i3);
            const int x = wrap_once(i1 + mm, n1);
            const T w1 = gl < W ? r1 : (T)0;
            for (int t = 0; t < a.ntransf; ++t) {
                const C *grid = reinterpret_cast<const C *>(gridp) + (int64_t)t * a.gstride;
                T are = 0, aim = 0;
                if (DIM == 1) {
                    const C v = __ldg(grid + x);
                    are = v.x;
                    aim = v.y;
                } else if (DIM == 2) {
#pragma unroll
                    for (int m2 = 0; m2 < W; ++m2) {
                        const T w2 = __shfl_sync(0xffffffffu, r2, gbase + m2);
                        const int y = wrap_once(i2 + m2, n2);
                        const C v = __ldg(grid + (int64_t)y * n1 + x);
                        are = fma(w2, v.x, are);
                        aim = fma(w2, v.y, aim);
                    }
                } else {
#pragma unroll 1
                    for (int m3 = 0; m3 < W; ++m3) {
                        const T w3 = __shfl_sync(0xffffffffu, r3, gbase + m3);
                        const int z = wrap_once(i3 + m3, n3);
                        T pre = 0, pim = 0;
#pragma unroll
                        for (int m2 = 0; m2 < W; ++m2) {
                            const T w2 = __shfl_sync(0xffffffffu, r2, gbase + m2);
                            const int y = wrap_once(i2 + m2, n2);
                            const C v = __ldg(grid + ((int64_t)z * n2 + y) * n1 + x);
                            pre = fma(w2, v.x, pre);
                            pim = fma(w2, v.y, pim);
                        }
                        are = fma(w3, pre, are);
                        aim = fma(w3, pim, aim);
                    }
                }
                are *= w1;
                aim *= w1;
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) {
                    are += __shfl_xor_sync(0xffffffffu, are, o);
                    aim += __shfl_xor_sync(0xffffffffu, aim, o);
                }
                if (gl == 0 && live) reinterpret_cast<C *>(cout)[(int64_t)t * a.M + rc.j] = C{are, aim};
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Type-1 deconvolution / mode copy (transforms.py:165-171): out[k] =
// p1[k1] p2[k2] p3[k3] * FFT[k mod n], one thread per output mode, k1
// fastest so both the gather (two contiguous runs per row) and the store
// are coalesced.

// Long mode rows (N1 >= 256): block items over rows (t, k3, k2) or 256-wide
// row segments; the row's bin offsets and correction factor are computed
// once per item and the k1 sweep is coalesced on both sides.
template <typename T>
__global__ void k_deconv_rows(int ntransf, int n1, int n2, int n3, int64_t N1, int64_t N2, int64_t N3,
                              const T *grid, const T *p1, const T *p2, const T *p3, T *f, int seg) {
    using C = typename Cx<T>::type;
    const int64_t G = (int64_t)n1 * n2 * n3;
    const int64_t rows = (int64_t)ntransf * N3 * N2;
    const int nn1 = (int)N1;
    const int nseg = (nn1 + seg - 1) / seg;
    for (int64_t item = blockIdx.x; item < rows * nseg; item += gridDim.x) {
        const int64_t row = item / nseg;
        const int s0 = (int)(item - row * nseg) * seg, s1 = min(nn1, s0 + seg);
        const int64_t t = row / (N3 * N2);
        const int64_t r = row - t * (N3 * N2);
        const int64_t k3i = r / N2, k2i = r - k3i * N2;
        int64_t k2 = k2i - N2 / 2, k3 = k3i - N3 / 2;
        if (k2 < 0) k2 += n2;
        if (k3 < 0) k3 += n3;
        const T f2 = p2 ? p2[k2i] : (T)1, f3 = p3 ? p3[k3i] : (T)1;
        const C *src = reinterpret_cast<const C *>(grid) + t * G + (k3 * n2 + k2) * n1;
        C *dst = reinterpret_cast<C *>(f) + row * N1;
        // four elements per thread per pass, all loads issued first
        constexpr int U = 4;
        for (int b = s0 + threadIdx.x; b < s1; b += U * blockDim.x) {
            C v[U];
            T fac[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k1i = b + u * blockDim.x;
                if (k1i < s1) {
                    int k1 = k1i - nn1 / 2;
                    if (k1 < 0) k1 += n1;
                    v[u] = src[k1];
                    fac[u] = p1[k1i];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k1i = b + u * blockDim.x;
                if (k1i < s1) {
                    T fc = fac[u];  // (p1 p2) p3
                    if (p2) fc *= f2;
                    if (p3) fc *= f3;
                    dst[k1i] = C{v[u].x * fc, v[u].y * fc};
                }
            }
        }
    }
}

// Short mode rows: one thread per mode.
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
// finiteness check of the mode coefficients (transforms.py:190).  One
// block-stride pass per grid row (t, l3, l2).
template <typename T>
__global__ void k_amplify(int ntransf, int n1, int n2, int n3, int64_t N1, int64_t N2, int64_t N3,
                          const T *f, const T *p1, const T *p2, const T *p3, T *grid,
                          unsigned long long *flag, int kRowSeg) {
    using C = typename Cx<T>::type;
    const int64_t G = (int64_t)n1 * n2 * n3, per = N1 * N2 * N3;
    const int64_t rows = (int64_t)ntransf * n3 * n2;
    // bin l -> centered mode k: k = l for l <= N - N/2 - 1, l - n for l >= n - N/2
    auto mode = [](int64_t l, int64_t n, int64_t N) -> int64_t {
        if (l <= N - N / 2 - 1) return l + N / 2;
        if (l >= n - N / 2) return l - n + N / 2;
        return -1;
    };
    const int nseg = (n1 + kRowSeg - 1) / kRowSeg;
    for (int64_t item = blockIdx.x; item < rows * nseg; item += gridDim.x) {
        const int64_t row = item / nseg;
        const int seg0 = (int)(item - row * nseg) * kRowSeg, seg1 = min(n1, seg0 + kRowSeg);
        const int64_t t = row / ((int64_t)n3 * n2);
        const int64_t r = row - t * ((int64_t)n3 * n2);
        const int64_t l3 = r / n2, l2 = r - l3 * n2;
        const int64_t m2 = mode(l2, n2, N2), m3 = mode(l3, n3, N3);
        C *dst = reinterpret_cast<C *>(grid) + t * G + (l3 * n2 + l2) * n1;
        if (m2 < 0 || m3 < 0) {
            for (int l1 = seg0 + threadIdx.x; l1 < seg1; l1 += blockDim.x) dst[l1] = C{(T)0, (T)0};
            continue;
        }
        const T f2 = p2 ? p2[m2] : (T)1, f3 = p3 ? p3[m3] : (T)1;
        const int64_t fbase = t * per + (m3 * N2 + m2) * N1;
        for (int l1 = seg0 + threadIdx.x; l1 < seg1; l1 += blockDim.x) {
            const int64_t m1 = mode(l1, n1, N1);
            C out{(T)0, (T)0};
            if (m1 >= 0) {
                const int64_t fi = fbase + m1;
                const C v = reinterpret_cast<const C *>(f)[fi];
                if (!finite2<T>(v)) flag_min(flag, (unsigned long long)fi);
                T fac = p1[m1];  // (p1 p2) p3
                if (p2) fac *= f2;
                if (p3) fac *= f3;
                out = C{v.x * fac, v.y * fac};
            }
            dst[l1] = out;
        }
    }
}

// ---------------------------------------------------------------------------
// dispatch helpers
template <typename T, int D, template <typename, int, int> class Op, typename... Args>
int dispatch_w(int w, Args &&...args) {
    switch (w) {
// ESN_WMASK (bit w set = width w compiled) trims a development build
#ifndef ESN_WMASK
#ifdef ESN_WMASK_DEV
#define ESN_WMASK (ESN_WMASK_DEV)
#else
#define ESN_WMASK 0x1fffc
#endif
#endif
#define ESN_CASE_W(WW)                                   \
    case WW:                                             \
        if constexpr ((ESN_WMASK >> WW) & 1) {           \
            return Op<T, D, WW>::run(args...);           \
        } else {                                         \
            return fail(ESN_INTERNAL_ERROR, "width %d not built (ESN_WMASK)", WW); \
        }
        ESN_CASE_W(2) ESN_CASE_W(3) ESN_CASE_W(4) ESN_CASE_W(5) ESN_CASE_W(6) ESN_CASE_W(7) ESN_CASE_W(8)
        ESN_CASE_W(9) ESN_CASE_W(10) ESN_CASE_W(11) ESN_CASE_W(12) ESN_CASE_W(13) ESN_CASE_W(14)
        ESN_CASE_W(15) ESN_CASE_W(16)
#undef ESN_CASE_W
        default:
            return fail(ESN_INTERNAL_ERROR, "unsupported kernel width %d", w);
    }
}

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
