// Shared-memory integer atomic throughput on sm_100a (fixed-point accumulation
// probe): 32-bit and 64-bit adds, conflict-free vs random addresses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms_bench atoms_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename I, int MODE>
__global__ void __launch_bounds__(256) k_atoms(I *out, int iters, int cells) {
    extern __shared__ unsigned char sm[];
    I *tile = reinterpret_cast<I *>(sm);
    for (int i = threadIdx.x; i < cells; i += blockDim.x) tile[i] = 0;
    __syncthreads();
    uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 40503u + 12345u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int it = 0; it < iters; ++it) {
        int idx;
        if (MODE == 0) {  // lanes -> consecutive cells, warp base varies
            s = s * 1664525u + 1013904223u;
            const uint32_t b = __shfl_sync(0xffffffffu, s, 0);
            idx = ((b >> 8) % (cells - 32)) + lane;
        } else if (MODE == 1) {  // fully random per lane
            s = s * 1664525u + 1013904223u;
            idx = (s >> 8) % cells;
        } else {  // footprint-like: lane = (dy,dz) row start, stride = row pitch 16, random base
            s = s * 1664525u + 1013904223u;
            const uint32_t b = __shfl_sync(0xffffffffu, s, 0);
            idx = ((b >> 8) % (cells - 32 * 16 - 8)) + lane * 16 + (it & 7);
        }
        atomicAdd(&tile[idx], (I)(it + lane));
    }
    __syncthreads();
    I acc = 0;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) acc += tile[i];
    if (acc == (I)0x7fffffff) out[blockIdx.x] = acc;
}

template <typename I, int MODE>
void run(const char *name, int cells) {
    int iters = 20000;
    I *out;
    cudaMalloc(&out, 4096 * sizeof(I));
    size_t smem = (size_t)cells * sizeof(I);
    cudaFuncSetAttribute(k_atoms<I, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = 148 * 2;
    k_atoms<I, MODE><<<grid, 256, smem>>>(out, 100, cells);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_atoms<I, MODE><<<grid, 256, smem>>>(out, iters, cells);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * 256 * iters;
    printf("%-28s cells %6d: %.3f ms, %.3e lane-atomics/s, %.2f lanes/clk/SM (1.965 GHz, 148 SMs) err=%s\n", name, cells,
           ms, ops / (ms * 1e-3), ops / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<int, 0>("s32 consecutive", 8192);
    run<int, 1>("s32 random", 8192);
    run<int, 2>("s32 strided-16", 8192);
    run<unsigned long long, 0>("u64 consecutive", 8192);
    run<unsigned long long, 1>("u64 random", 8192);
    run<unsigned long long, 2>("u64 strided-16", 8192);
    run<float, 0>("f32 consecutive (CAS?)", 8192);
    run<float, 1>("f32 random (CAS?)", 8192);
    return 0;
}
