// esn_inst.cuh -- launchers for one precision T (included by esn_inst_f64.cu
// and esn_inst_f32.cu so the two precisions compile in parallel).
#pragma once

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

template <typename T, int D, int W>
struct SpreadTileOp {
    static int run(const SpreadArgs<T> &a, cudaStream_t st) {
        if (a.M == 0) return ESN_SUCCESS;
        const int dtype = sizeof(T) == 8 ? ESN_F64 : ESN_F32;
        const size_t smem = tile_smem_bytes(D, W, a.g.bs, dtype);
        static size_t configured = 0;
        if (smem > configured) {
            ESN_CUDA_TRY(cudaFuncSetAttribute(k_spread_tile<T, D, W>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            configured = smem;
        }
        int occ = 0;
        ESN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spread_tile<T, D, W>, 256, smem));
        if (occ < 1) return fail(ESN_RESOURCE_ERROR, "spread tile of %zu bytes does not fit in shared memory", smem);
        k_spread_tile<T, D, W><<<device_sm_count() * occ, 256, smem, st>>>(a);
        ESN_CUDA_TRY(cudaGetLastError());
        return ESN_SUCCESS;
    }
};

template <typename T, int D, int W>
struct InterpOp {
    static int run(const SpreadArgs<T> &a, T *cout, const T *grid, cudaStream_t st) {
        if (a.M == 0) return ESN_SUCCESS;
        k_interp_thread<T, D, W><<<grid_for(a.M, 256), 256, 0, st>>>(a, cout, grid);
        ESN_CUDA_TRY(cudaGetLastError());
        return ESN_SUCCESS;
    }
};

template <>
int launch_spread<ESN_T>(const SpreadArgs<ESN_T> &a, int method, int nbins, cudaStream_t st) {
    (void)nbins;
    if (method == ESN_METHOD_GLOBAL)
        return dispatch_dw<ESN_T, SpreadGlobalOp>(a.g.dim, a.g.w, a, st);
    return dispatch_dw<ESN_T, SpreadTileOp>(a.g.dim, a.g.w, a, st);
}

template <>
int launch_interp<ESN_T>(const SpreadArgs<ESN_T> &a, ESN_T *cout, const ESN_T *grid, cudaStream_t st) {
    return dispatch_dw<ESN_T, InterpOp>(a.g.dim, a.g.w, a, cout, grid, st);
}

template <>
int launch_deconv<ESN_T>(int dim, int ntransf, const int *n, const int64_t *N, const ESN_T *grid,
                         const ESN_T *p1, const ESN_T *p2, const ESN_T *p3, ESN_T *f, cudaStream_t st) {
    (void)dim;
    const int64_t total = N[0] * N[1] * N[2] * ntransf;
    if (total == 0) return ESN_SUCCESS;
    k_deconv<ESN_T><<<grid_for(total, 256), 256, 0, st>>>(ntransf, n[0], n[1], n[2], N[0], N[1], N[2],
                                                          grid, p1, p2, p3, f);
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
    k_amplify<ESN_T><<<grid_for(total, 256), 256, 0, st>>>(ntransf, n[0], n[1], n[2], N[0], N[1], N[2],
                                                           f, p1, p2, p3, grid, flag);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

}  // namespace esn
