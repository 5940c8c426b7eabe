// FFMA vs FFMA2 (fma.rn.f32x2, sm_100+) issue and lane throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_peak ffma2_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) {
    unsigned long long ra = *reinterpret_cast<unsigned long long *>(&a), rc = *reinterpret_cast<unsigned long long *>(&c), rd;
    float2 b = make_float2(w, w);
    unsigned long long rb = *reinterpret_cast<unsigned long long *>(&b);
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
    return *reinterpret_cast<float2 *>(&rd);
}

template <int MODE>
__global__ void __launch_bounds__(256) k(float2 *o, int iters, float w0) {
    float2 acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, 1.f);
    float2 v = make_float2(1.0001f, 0.9999f);
    float w = w0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) {
                acc[i].x = fmaf(v.x, w, acc[i].x);
                acc[i].y = fmaf(v.y, w, acc[i].y);
            } else {
                acc[i] = ffma2(v, w, acc[i]);
            }
        }
    }
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 16; ++i) { s.x += acc[i].x; s.y += acc[i].y; }
    o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char *name) {
    float2 *o;
    int grid = 148 * 8, iters = 20000;
    cudaMalloc(&o, (size_t)grid * 256 * sizeof(float2));
    k<MODE><<<grid, 256>>>(o, 10, 1e-6f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<grid, 256>>>(o, iters, 1e-6f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)grid * 256 * iters * 32;
    printf("%-8s %.3f ms  %.3e lane-FMA/s  (%.1f FMA/clk/SM at 1.965 GHz)\n", name, ms, fma / (ms * 1e-3),
           fma / (ms * 1e-3) / 148 / 1.965e9);
    cudaFree(o);
}

int main() {
    run<0>("FFMA");
    run<1>("FFMA2");
    return 0;
}
