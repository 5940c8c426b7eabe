// esn_inst.cuh -- launchers for one precision T (included by esn_inst_f64.cu
// and esn_inst_f32.cu so the two precisions compile in parallel).
#pragma once

#include <cstdlib>
#include <string>

// this unit compiles the widths of part ESN_PART only (esn_internal.h
// kWidthSplit), intersected with a development ESN_WMASK if one is given
#ifndef ESN_PART
#error "define ESN_PART (0: widths 2..8, 1: widths 9..16)"
#endif
#ifdef ESN_WMASK_DEV
#define ESN_WMASK ((ESN_WMASK_DEV) & (ESN_PART == 0 ? 0x1fc : 0x1fe00))
#else
#define ESN_WMASK (0x1fffc & (ESN_PART == 0 ? 0x1fc : 0x1fe00))
#endif

#include "esn_device.cuh"

namespace esn {

static inline int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = (int64_t)device_sm_count() * 16;
    if (b > cap) b = cap;
    return (int)(b < 1 ? 1 : b);
}

template <typename T, int D, int W>
struct SpreadGlobalOp {
    static int run(const SpreadArgs<T> &a, cudaStream_t st) {
        if (a.M == 0) return ESN_SUCCESS;
        k_spread_global<T, D, W><<<grid_for(a.M, 256), 256, 0, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
        return ESN_SUCCESS;
    }
};

template <typename K>
static int persistent_launch(K kernel, int threads, size_t smem, cudaStream_t st, const void *args_dummy,
                             int *grid_out) {
    (void)args_dummy;
    ESN_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ESN_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared));
    int occ = 0;
    ESN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem));
    if (occ < 1) return fail(ESN_RESOURCE_ERROR, "spreader CTA (%d threads, %zu B smem) does not fit an SM", threads, smem);
    *grid_out = device_sm_count() * occ;
    return ESN_SUCCESS;
}

template <typename T, int D, int W>
struct SpreadRowsOp {
    static int run(const SpreadArgs<T> &a, cudaStream_t st) {
        if (a.M == 0) return ESN_SUCCESS;
        if constexpr (D == 1) {
            return SpreadGlobalOp<T, D, W>::run(a, st);
        } else {
        if constexpr (D == 3) {
            static const bool old_rows = [] {
                const char *e = getenv("ESN_SPREAD3");
                return e && std::string(e) == "rows";
            }();
            if (!old_rows) {
                using Cfg3 = Rows3Cfg<T, W>;
                if (Cfg3::R::THIN && a.roll && a.ntransf == 1) {  // z-rolling segments (small bins, w <= 7)
                    static PerDev<int> gridr_;
                    int &gridr = gridr_();
                    if (gridr == 0) {
                        int rc = persistent_launch(k_spread_rows3<T, W, true>, Cfg3::NT, Cfg3::SMEM, st, nullptr, &gridr);
                        if (rc) return rc;
                    }
                    k_spread_rows3<T, W, true><<<gridr, Cfg3::NT, Cfg3::SMEM, st>>>(a);
                } else {
                    static PerDev<int> grid3_;
                    int &grid3 = grid3_();
                    if (grid3 == 0) {
                        int rc = persistent_launch(k_spread_rows3<T, W, false>, Cfg3::NT, Cfg3::SMEM, st, nullptr, &grid3);
                        if (rc) return rc;
                    }
                    k_spread_rows3<T, W, false><<<grid3, Cfg3::NT, Cfg3::SMEM, st>>>(a);
                }
                ESN_CUDA_TRY(cudaGetLastError());
                return ESN_SUCCESS;
            }
        }
        using Cfg = RowsCfg<T, D, W>;
        using C = typename Cx<T>::type;
        constexpr int NZ = D == 3 ? W : 1;
        const size_t stage = Cfg::CH * NZ * sizeof(C) + Cfg::CH * 2 * W * sizeof(T) + Cfg::CH * 4 * sizeof(int) +
                             (Cfg::NT / 32) * Cfg::CH;
        const size_t tile = (size_t)Cfg::RY * Cfg::RZ * Cfg::X * sizeof(C);
        const size_t smem = stage > tile ? stage : tile;
        static PerDev<int> grid_;
        int &grid = grid_();
        if (grid == 0) {
            int rc = persistent_launch(k_spread_rows<T, D, W>, Cfg::NT, smem, st, nullptr, &grid);
            if (rc) return rc;
        }
        k_spread_rows<T, D, W><<<grid, Cfg::NT, smem, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
        return ESN_SUCCESS;
        }
    }
};

template <typename T, int D, int W>
struct SpreadBatchOp {
    static int run(const SpreadArgs<T> &a, const int *key, const int *kstart, T *cperm,
                   cudaStream_t st) {
        if (a.M == 0) return ESN_SUCCESS;
        if constexpr (D == 2 && sizeof(T) == 4 && W <= 10) {
            using Cfg = Batch2Cfg<T, W>;
            const int ngroups = (a.ntransf + 31) / 32;
            int64_t pb = ((a.M + 31) / 32) * ngroups;
            if (pb > (int64_t)device_sm_count() * 16) pb = (int64_t)device_sm_count() * 16;
            k_permute_strengths<T><<<(int)pb, 1024, 0, st>>>(a, key, kstart, cperm);
            ESN_CUDA_TRY(cudaGetLastError());
            // per-point rows table lives behind the permuted strengths
            PtRows2<W> *tab = reinterpret_cast<PtRows2<W> *>(
                reinterpret_cast<char *>(cperm) + (size_t)ngroups * 32 * a.M * 2 * sizeof(T));
            k_rows2d<T, W><<<grid_for(a.M, 256), 256, 0, st>>>(a, tab);
            constexpr size_t smem = batch2d_smem_bytes<T, W>();
            // cell-resolution sort keys -> static x-offset sweep; else per-point dispatch
            bool rolled = false;
            // y-rolling owner-computes for w <= 6 (the w x 8 register ring fits 128 registers)
            if constexpr (W <= 6) {
                if (batched_owner(ESN_F32, 2, W, a.ntransf, ESN_METHOD_TILE, a.sbl, a.g.bs) &&
                    b2roll_fits<W>(a.g.n[0], a.g.n[1]) && !batched_roll_off()) {
                    constexpr size_t rsmem = b2roll_smem_bytes<W>();
                    static PerDev<int> grid_;
                    int &grid = grid_();
                    if (grid == 0) {
                        int rc = persistent_launch(k_spread_b2roll<T, W>, 128, rsmem, st, nullptr, &grid);
                        if (rc) return rc;
                    }
                    k_spread_b2roll<T, W><<<grid, 128, rsmem, st>>>(a, cperm, tab);
                    rolled = true;
                }
            }
            const bool owner = batched_owner(ESN_F32, 2, W, a.ntransf, ESN_METHOD_TILE, a.sbl, a.g.bs);
            if (rolled) {
            } else if (owner) {
                constexpr size_t osmem = b2own_smem_bytes<T, W>();
                static PerDev<int> grid_;
                int &grid = grid_();
                if (grid == 0) {
                    int rc = persistent_launch(k_spread_b2own<T, W>, 128, osmem, st, nullptr, &grid);
                    if (rc) return rc;
                }
                k_spread_b2own<T, W><<<grid, 128, osmem, st>>>(a, cperm, tab);
            }
            // clustered points: one warp walks every point of an owner item, so a
            // few dense items would carry the kernel (c5 on the disc-quadrature
            // cloud: 9.5 ms against 2.7 ms for the subproblem-balanced RED-flush
            // kernel).  setpts left a device flag; when it is set the kernels
            // above returned at once and these two run instead.
            if (owner && a.imb) {
                if (!a.accumulate) {
                    const size_t n16 = (size_t)a.gstride * a.ntransf * 2 * sizeof(T) / 16;
                    k_zero_if<T><<<device_sm_count() * 8, 256, 0, st>>>(reinterpret_cast<int4 *>(a.grid), n16, a.imb);
                }
                static PerDev<int> grid_;
                int &grid = grid_();
                if (grid == 0) {
                    int rc = persistent_launch(k_spread_batch2d<T, W, true>, 128, smem, st, nullptr, &grid);
                    if (rc) return rc;
                }
                k_spread_batch2d<T, W, true><<<grid, 128, smem, st>>>(a, cperm, tab);
            }
            if (owner) {
            } else if (a.sbl[0] == 0 && a.sbl[1] == 0 && a.g.bs[0] == Cfg::BX) {
                static PerDev<int> grid_;
                int &grid = grid_();
                if (grid == 0) {
                    int rc = persistent_launch(k_spread_batch2d<T, W, true>, 128, smem, st, nullptr, &grid);
                    if (rc) return rc;
                }
                k_spread_batch2d<T, W, true><<<grid, 128, smem, st>>>(a, cperm, tab);
            } else {
                static PerDev<int> grid_;
                int &grid = grid_();
                if (grid == 0) {
                    int rc = persistent_launch(k_spread_batch2d<T, W, false>, 128, smem, st, nullptr, &grid);
                    if (rc) return rc;
                }
                k_spread_batch2d<T, W, false><<<grid, 128, smem, st>>>(a, cperm, tab);
            }
            ESN_CUDA_TRY(cudaGetLastError());
            return ESN_SUCCESS;
        } else {
            return SpreadRowsOp<T, D, W>::run(a, st);
        }
    }
};

template <typename T, int D, int W>
struct InterpOp {
    static int run(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st) {
        if (a.M == 0) return ESN_SUCCESS;
        static const char *mode = getenv("ESN_INTERP");
        if (mode && std::string(mode) == "thread") {
            k_interp_thread<T, D, W><<<grid_for(a.M, 256), 256, 0, st>>>(a, cout, grid);
            ESN_CUDA_TRY(cudaGetLastError());
            return ESN_SUCCESS;
        }
        using C = typename Cx<T>::type;
        size_t cells = 1;
        bool fits = true;  // every patch row wraps at most once
        for (int d = 0; d < D; ++d) {
            cells *= (size_t)(a.g.bs[d] + W - 1);
            fits = fits && a.g.bs[d] + W - 1 <= a.g.n[d];
        }
        if constexpr (sizeof(C) == 16) if (fits && !(mode && std::string(mode) == "tile")) {
            static const char *sl = getenv("ESN_INTERP_SLICE");
            // record ring: ESN_INTERP_RING=<2..4> slots of ESN_INTERP_SLICE records
            static const char *re = getenv("ESN_INTERP_RING");
            const int R = re ? std::min(4, std::max(2, atoi(re))) : 2;
            int slice = sl ? atoi(sl) : 512;
            // patch row pitch: ESN_INTERP_PITCH=<cells> (>= bs + w - 1), 0 = rows packed;
            // default a multiple of 8 cells (128 bytes) for D >= 2
            static const char *pe = getenv("ESN_INTERP_PITCH");
            const int P1 = a.g.bs[0] + W - 1;
            int pitch1 = D >= 2 ? (P1 + 7) / 8 * 8 : P1;
            if (pe) pitch1 = atoi(pe) > P1 ? atoi(pe) : P1;
            cells = cells / (size_t)P1 * (size_t)pitch1;
            // three CTAs per SM when the patches allow it: 228 KB less 1 KB
            // reserved and the static words per CTA
            constexpr size_t kThree = 233472 / 3 - 1024 - 512;
            if (!sl)
                while (slice > 128 && 2 * cells * sizeof(C) + (size_t)R * slice * sizeof(Rec) > kThree) slice -= 32;
            const size_t bsmem = 2 * cells * sizeof(C) + (size_t)R * slice * sizeof(Rec);
            if (bsmem <= 112 * 1024) {
                static PerDev<size_t> bconf_;
                size_t &bconfigured = bconf_();
                if (bsmem > bconfigured) {
                    ESN_CUDA_TRY(cudaFuncSetAttribute(k_interp_bulk<T, D, W>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
                    bconfigured = bsmem;
                }
                int occ = 0;
                ESN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_interp_bulk<T, D, W>, 256, bsmem));
                if (occ < 1) occ = 1;
                static const int dprod = [] {
                    const char *e = getenv("ESN_INTERP_PRODUCER");
                    return e && e[0] == '0' ? 0 : 1;
                }();
                k_interp_bulk<T, D, W><<<device_sm_count() * occ, 256, bsmem, st>>>(a, cout, grid, slice, dprod, pitch1, R);
                ESN_CUDA_TRY(cudaGetLastError());
                return ESN_SUCCESS;
            }
        }
        const size_t smem = cells * sizeof(C) + kInterpSlice * sizeof(Rec);
        if (smem > 200 * 1024) {  // patch too large for shared memory: L1 path
            k_interp_thread<T, D, W><<<grid_for(a.M, 256), 256, 0, st>>>(a, cout, grid);
            ESN_CUDA_TRY(cudaGetLastError());
            return ESN_SUCCESS;
        }
        static PerDev<size_t> conf_;
        size_t &configured = conf_();
        if (smem > configured) {
            ESN_CUDA_TRY(cudaFuncSetAttribute(k_interp_tile<T, D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem));
            configured = smem;
        }
        int occ = 0;
        ESN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_interp_tile<T, D, W>, 256, smem));
        if (occ < 1) occ = 1;
        k_interp_tile<T, D, W><<<device_sm_count() * occ, 256, smem, st>>>(a, cout, grid);
        ESN_CUDA_TRY(cudaGetLastError());
        return ESN_SUCCESS;
    }
};

template <>
int launch_spread_dp<ESN_T, ESN_D, ESN_PART>(const SpreadArgs<ESN_T> &a, int method, const int *key,
                                             const int *kstart, ESN_T *cperm, cudaStream_t st) {
    if (method == ESN_METHOD_GLOBAL || ESN_D == 1) return dispatch_w<ESN_T, ESN_D, SpreadGlobalOp>(a.g.w, a, st);
    if (batched_spread(sizeof(ESN_T) == 8 ? ESN_F64 : ESN_F32, ESN_D, a.g.w, a.ntransf, method))
        return dispatch_w<ESN_T, ESN_D, SpreadBatchOp>(a.g.w, a, key, kstart, cperm, st);
    return dispatch_w<ESN_T, ESN_D, SpreadRowsOp>(a.g.w, a, st);
}

template <>
int launch_interp_dp<ESN_T, ESN_D, ESN_PART>(const SpreadArgs<ESN_T> &a, ESN_T *cout, const ESN_T *grid,
                                             cudaStream_t st) {
    return dispatch_w<ESN_T, ESN_D, InterpOp>(a.g.w, a, cout, grid, st);
}

#if ESN_D == 1 && ESN_PART == 0
template <>
int launch_deconv<ESN_T>(int dim, int ntransf, const int *n, const int64_t *N, const ESN_T *grid,
                         const ESN_T *p1, const ESN_T *p2, const ESN_T *p3, ESN_T *f, cudaStream_t st) {
    (void)dim;
    const int64_t total = N[0] * N[1] * N[2] * ntransf;
    if (total == 0) return ESN_SUCCESS;
    if (N[0] >= 256) {  // long rows: whole rows per block item when there are enough, else segments
        const int64_t rows = total / N[0];
        const int seg = rows >= (int64_t)device_sm_count() * 8 ? (int)N[0] : 256;
        const int64_t items = rows * ((N[0] + seg - 1) / seg);
        const int blocks = (int)std::min<int64_t>(items, (int64_t)device_sm_count() * 32);
        k_deconv_rows<ESN_T><<<blocks, 128, 0, st>>>(ntransf, n[0], n[1], n[2], N[0], N[1], N[2], grid, p1, p2,
                                                     p3, f, seg);
    } else {
        k_deconv<ESN_T><<<grid_for(total, 256), 256, 0, st>>>(ntransf, n[0], n[1], n[2], N[0], N[1], N[2], grid, p1,
                                                               p2, p3, f);
    }
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

template <>
int launch_amplify<ESN_T>(int dim, int ntransf, const int *n, const int64_t *N, const ESN_T *f,
                          const ESN_T *p1, const ESN_T *p2, const ESN_T *p3, ESN_T *grid,
                          unsigned long long *flag, cudaStream_t st) {
    (void)dim;
    const int64_t total = (int64_t)n[0] * n[1] * n[2] * ntransf;
    if (total == 0) return ESN_SUCCESS;
    const int64_t rows = total / n[0];
    const int seg = rows >= (int64_t)device_sm_count() * 8 ? n[0] : 256;
    const int64_t items = rows * ((n[0] + seg - 1) / seg);
    const int blocks = (int)std::min<int64_t>(items, (int64_t)device_sm_count() * 32);
    k_amplify<ESN_T><<<blocks, 256, 0, st>>>(ntransf, n[0], n[1], n[2], N[0], N[1], N[2],
                                             f, p1, p2, p3, grid, flag, seg);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

#endif  // ESN_D == 1

}  // namespace esn
