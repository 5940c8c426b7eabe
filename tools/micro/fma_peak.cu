// FP64 / FP32 FMA throughput on this GPU (the compute roofs quoted in
// DESIGN.md).  8 independent FMA chains per thread, 148 x 8 CTAs of 256.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T *out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (T)(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == (T)12345.678) out[0] = s;
}

template <typename T>
double run(const char *name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    T *out;
    cudaMalloc(&out, sizeof(T));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = 5.0 * blocks * threads * (double)iters * 8;
    const double tflops = 2.0 * fmas / (ms * 1e-3) / 1e12;
    printf("%s FMA: %.1f TFLOP/s (%.3g FMA/s)\n", name, tflops, fmas / (ms * 1e-3));
    cudaFree(out);
    return tflops;
}

int main() {
    run<double>("fp64");
    run<float>("fp32");
    return 0;
}
