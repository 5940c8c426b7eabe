// Microbenchmark for the type-2 sort redesign (c2 shape: M = 1e7 points,
// 4 Mi fine keys / 20 K coarse keys): where does the record scatter's time
// go -- the atomics with return, or the random 32-byte record stores?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_probe scatter_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <thrust/scan.h>
#include <thrust/execution_policy.h>

struct __align__(32) Rec { double g[3]; int j; int pad; };

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// A: fire-and-forget RED histogram over K fine keys
__global__ void k_red(const double *x, const double *y, int M, int K, int *cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        double s = x[i] + y[i];
        uint32_t k = hash32(i + (s > 1e300)) % K;
        atomicAdd(&cnt[k], 1);
    }
}
// B: atomic-with-return cursor + 32 B record store (the current scatter)
__global__ void k_scatter_rec(const double *x, const double *y, int M, int K, int *cur, Rec *out, int mask) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        double a = x[i], b = y[i];
        uint32_t k = hash32(i + (a > 1e300)) % K;
        int pos = atomicAdd(&cur[k], 1) & mask;
        Rec r; r.g[0] = a; r.g[1] = b; r.g[2] = 0; r.j = i; r.pad = 0;
        out[pos] = r;
    }
}
// C: atomic-with-return cursor + 4 B index store
__global__ void k_scatter_idx(const double *x, const double *y, int M, int K, int *cur, int *out, int mask) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        double a = x[i];
        uint32_t k = hash32(i + (a > 1e300)) % K;
        int pos = atomicAdd(&cur[k], 1) & mask;
        out[pos] = i;
    }
}
// D: no atomics, record store at a hashed position (random 32 B stores only)
__global__ void k_store_rec(const double *x, const double *y, int M, Rec *out, int mask, int run) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        double a = x[i], b = y[i];
        int pos = ((hash32(i / run) * run) + (i % run)) & mask;
        Rec r; r.g[0] = a; r.g[1] = b; r.g[2] = 0; r.j = i; r.pad = 0;
        out[pos] = r;
    }
}
// E: atomics with return only (no store)
__global__ void k_atom_only(const double *x, int M, int K, int *cur, int *sink) {
    int acc = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        double a = x[i];
        uint32_t k = hash32(i + (a > 1e300)) % K;
        acc += atomicAdd(&cur[k], 1);
    }
    if (acc == 0x7fffffff) *sink = acc;
}
// F: smem-privatised coarse histogram (K <= 24 K) flushed per CTA into a
// [K][ncta] matrix (no global atomics)
__global__ void k_smem_hist(const double *x, const double *y, int M, int K, int *mat) {
    extern __shared__ int h[];
    for (int k = threadIdx.x; k < K; k += blockDim.x) h[k] = 0;
    __syncthreads();
    const int per = (M + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per, hi = min(M, lo + per);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        double a = x[i] + y[i];
        uint32_t k = hash32(i + (a > 1e300)) % K;
        atomicAdd(&h[k], 1);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) mat[(size_t)k * gridDim.x + blockIdx.x] = h[k];
}
// G: the scatter of F's layout: smem cursors (start from mat after a scan,
// here just k * ncta spacing), record stores in per-(CTA, key) runs
__global__ void k_smem_scatter(const double *x, const double *y, int M, int K, const int *mat, Rec *out, int mask) {
    extern __shared__ int c[];
    for (int k = threadIdx.x; k < K; k += blockDim.x) c[k] = mat[(size_t)k * gridDim.x + blockIdx.x];
    __syncthreads();
    const int per = (M + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per, hi = min(M, lo + per);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        double a = x[i], b = y[i];
        uint32_t k = hash32(i + (a > 1e300)) % K;
        int pos = atomicAdd(&c[k], 1) & mask;
        Rec r; r.g[0] = a; r.g[1] = b; r.g[2] = 0; r.j = i; r.pad = 0;
        out[pos] = r;
    }
}

__device__ __forceinline__ void st256(Rec *p, double a, double b, int j, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "l"(__double_as_longlong(a)),
                 "l"(__double_as_longlong(b)), "l"(0ull), "l"((unsigned long long)(unsigned)j), "l"(pol)
                 : "memory");
}
// B2: the current scatter's shape: 8 points in flight, atomics with return
// (evict-last), 256-bit record stores (evict-first)
__global__ void __launch_bounds__(256) k_b2(const double *x, const double *y, int M, int K, int *cur, Rec *out, int mask) {
    uint64_t pf, pl;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    const int S = gridDim.x * blockDim.x * 8;
    for (int base = blockIdx.x * blockDim.x * 8 + threadIdx.x; base < M; base += S) {
        double a[8], b[8]; int pos[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { int i = base + u * blockDim.x; a[u] = i < M ? x[i] : 0; b[u] = i < M ? y[i] : 0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            int i = base + u * blockDim.x;
            uint32_t k = hash32(i + (a[u] > 1e300)) % K;
            if (i < M) asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], 1, %2;" : "=r"(pos[u]) : "l"(cur + k), "l"(pl) : "memory");
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) { int i = base + u * blockDim.x; if (i < M) st256(out + (pos[u] & mask), a[u], b[u], i, pf); }
    }
}
// D2: 256-bit stores at hashed positions in runs of `run`, 8 in flight
__global__ void __launch_bounds__(256) k_d2(const double *x, const double *y, int M, Rec *out, int mask, int run) {
    uint64_t pf;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    const int S = gridDim.x * blockDim.x * 8;
    for (int base = blockIdx.x * blockDim.x * 8 + threadIdx.x; base < M; base += S) {
        double a[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { int i = base + u * blockDim.x; a[u] = i < M ? x[i] : 0; b[u] = i < M ? y[i] : 0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            int i = base + u * blockDim.x;
            int pos = ((hash32(i / run) * run) + (i % run)) & mask;
            if (i < M) st256(out + pos, a[u], b[u], i, pf);
        }
    }
}
// G2: smem cursors per (CTA, key), 256-bit stores; the CTA walks its tile
// 4 points per thread in flight
__global__ void __launch_bounds__(1024) k_g2(const double *x, const double *y, int M, int K, const int *mat, Rec *out, int mask) {
    extern __shared__ int c[];
    uint64_t pf;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    for (int k = threadIdx.x; k < K; k += blockDim.x) c[k] = mat[(size_t)k * gridDim.x + blockIdx.x];
    __syncthreads();
    const int per = (M + gridDim.x - 1) / gridDim.x;
    const int lo = blockIdx.x * per, hi = min(M, lo + per);
    for (int base = lo + threadIdx.x; base < hi; base += 4 * blockDim.x) {
        double a[4], b[4]; int pos[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { int i = base + u * blockDim.x; a[u] = i < hi ? x[i] : 0; b[u] = i < hi ? y[i] : 0; }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int i = base + u * blockDim.x;
            uint32_t k = hash32(i + (a[u] > 1e300)) % K;
            if (i < hi) pos[u] = atomicAdd(&c[k], 1);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) { int i = base + u * blockDim.x; if (i < hi) st256(out + (pos[u] & mask), a[u], b[u], i, pf); }
    }
}

// C2: the current scatter's shape but a 4-byte index store (perm[pos] = j)
__global__ void __launch_bounds__(256) k_c2(const double *x, const double *y, int M, int K, int *cur, int *perm, int mask) {
    uint64_t pl;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    const int S = gridDim.x * blockDim.x * 8;
    for (int base = blockIdx.x * blockDim.x * 8 + threadIdx.x; base < M; base += S) {
        double a[8], b[8]; int pos[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { int i = base + u * blockDim.x; a[u] = i < M ? x[i] : 0; b[u] = i < M ? y[i] : 0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            int i = base + u * blockDim.x;
            uint32_t k = hash32(i + (a[u] + b[u] > 1e300)) % K;
            if (i < M) asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], 1, %2;" : "=r"(pos[u]) : "l"(cur + k), "l"(pl) : "memory");
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            int i = base + u * blockDim.x;
            if (i < M) asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" :: "l"(perm + (pos[u] & mask)), "r"(i), "l"(pl) : "memory");
        }
    }
}
// key positions with spatial locality like the real sort: key = (i*2654435761 >> 10) % K ... here:
// cursors start at k * (M / K) so positions are a true permutation-ish
__global__ void k_init_cur(int *cur, int K, int M) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) cur[k] = (int)((long)k * M / K);
}
// H: index gather of coordinates (interp-side): read perm sequentially,
// gather x[j], y[j]; j restricted to a window of C points (target chunk)
__global__ void k_gather(const int *perm, const double *x, const double *y, int M, double *sink) {
    double acc = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        int j = perm[i];
        acc += x[j] * y[j];
    }
    if (acc == 1.2345) *sink = acc;
}
__global__ void k_make_perm(int *perm, int M, int C) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
        int c0 = (i / C) * C, len = min(C, M - c0);
        perm[i] = c0 + (int)(hash32(i) % (uint32_t)len);
    }
}

static cudaEvent_t e0, e1;
#define TIME(name, launch)                                                  \
    do {                                                                    \
        launch; cudaDeviceSynchronize();                                    \
        cudaEventRecord(e0); for (int r = 0; r < 5; ++r) { launch; }        \
        cudaEventRecord(e1); cudaEventSynchronize(e1);                      \
        float ms; cudaEventElapsedTime(&ms, e0, e1);                        \
        printf("%-44s %8.1f us\n", name, ms * 1e3 / 5);                     \
    } while (0)

int main() {
    const int M = 10000000, KF = 4 << 20, mask = (1 << 24) - 1;
    double *x, *y, *dsink; int *cnt, *perm, *idx, *mat, *isink; Rec *rec;
    cudaMalloc(&x, M * 8); cudaMalloc(&y, M * 8); cudaMalloc(&dsink, 8); cudaMalloc(&isink, 4);
    cudaMalloc(&cnt, KF * 4); cudaMalloc(&perm, M * 4); cudaMalloc(&idx, (mask + 1) * 4);
    cudaMalloc(&rec, (size_t)(mask + 1) * sizeof(Rec)); cudaMalloc(&mat, 24576 * 1184 * 4);
    cudaMemset(x, 0, M * 8); cudaMemset(y, 0, M * 8); cudaMemset(cnt, 0, KF * 4);
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int nsm = 148;
    printf("scatter_probe: M = %d\n", M);
    TIME("A  RED histogram, 4 Mi keys", (k_red<<<nsm * 8, 256>>>(x, y, M, KF, cnt)));
    TIME("A' RED histogram, 20 K keys", (k_red<<<nsm * 8, 256>>>(x, y, M, 20480, cnt)));
    TIME("B  atom-ret + 32 B record, 4 Mi keys", (k_scatter_rec<<<nsm * 8, 256>>>(x, y, M, KF, cnt, rec, mask)));
    TIME("C  atom-ret + 4 B index, 4 Mi keys", (k_scatter_idx<<<nsm * 8, 256>>>(x, y, M, KF, cnt, idx, mask)));
    TIME("E  atom-ret only, 4 Mi keys", (k_atom_only<<<nsm * 8, 256>>>(x, M, KF, cnt, isink)));
    TIME("E' atom-ret only, 20 K keys", (k_atom_only<<<nsm * 8, 256>>>(x, M, 20480, cnt, isink)));
    for (int run = 1; run <= 16; run *= 2) {
        char nm[64]; snprintf(nm, 64, "D  32 B record stores, runs of %d", run);
        TIME(nm, (k_store_rec<<<nsm * 8, 256>>>(x, y, M, rec, mask, run)));
    }
    for (int K = 4096; K <= 24576; K *= 2) {
        if (K > 24576) break;
        for (int ncta : {148, 296, 592}) {
            size_t sm = (size_t)K * 4;
            cudaFuncSetAttribute(k_smem_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
            cudaFuncSetAttribute(k_smem_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
            char nm[96];
            snprintf(nm, 96, "F  smem hist K=%d ncta=%d", K, ncta);
            TIME(nm, (k_smem_hist<<<ncta, 1024, sm>>>(x, y, M, K, mat)));
            snprintf(nm, 96, "G  smem-cursor scatter K=%d ncta=%d", K, ncta);
            TIME(nm, (k_smem_scatter<<<ncta, 1024, sm>>>(x, y, M, K, mat, rec, mask)));
        }
    }

    TIME("B2 current-shape scatter, 4 Mi keys", (k_b2<<<nsm * 8, 256>>>(x, y, M, KF, cnt, rec, mask)));
    for (int run = 1; run <= 8; run *= 2) {
        char nm[64]; snprintf(nm, 64, "D2 256-bit record stores, runs of %d", run);
        TIME(nm, (k_d2<<<nsm * 8, 256>>>(x, y, M, rec, mask, run)));
    }
    cudaFuncSetAttribute(k_g2, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int K : {4096, 8192, 16384})
        for (int ncta : {148, 296, 444, 592}) {
            k_smem_hist<<<ncta, 1024, K * 4>>>(x, y, M, K, mat);
            thrust::exclusive_scan(thrust::device, mat, mat + (size_t)K * ncta, mat);
            char nm[96]; snprintf(nm, 96, "G2 smem-cursor scatter K=%d ncta=%d", K, ncta);
            TIME(nm, (k_g2<<<ncta, 1024, K * 4>>>(x, y, M, K, mat, rec, mask)));
        }

    {
        int *permb; cudaMalloc(&permb, (size_t)(mask + 1) * 4);
        TIME("C2 atom-ret + 4 B index (ILP 8, L2 hints), 4 Mi keys", (k_init_cur<<<1024, 256>>>(cnt, KF, M), k_c2<<<nsm * 8, 256>>>(x, y, M, KF, cnt, permb, mask)));
        TIME("B2 (same cursor init), 4 Mi keys", (k_init_cur<<<1024, 256>>>(cnt, KF, M), k_b2<<<nsm * 8, 256>>>(x, y, M, KF, cnt, rec, mask)));
        TIME("init only", (k_init_cur<<<1024, 256>>>(cnt, KF, M)));
    }
    for (int C : {M, M / 2, M / 4, M / 8, M / 16}) {
        k_make_perm<<<nsm * 8, 256>>>(perm, M, C);
        char nm[64]; snprintf(nm, 64, "H  gather x[j],y[j], chunk %d", C);
        TIME(nm, (k_gather<<<nsm * 8, 256>>>(perm, x, y, M, dsink)));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
