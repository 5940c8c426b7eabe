// Microbenchmark: global RED throughput on B200 (coalesced / strided, f32x2 / f64) vs plain stores.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red_f32x2(float2* p, long n, long stride_elems, int reps) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long nthreads = gridDim.x * (long)blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (long i = tid; i < n; i += nthreads) {
      long idx = stride_elems > 1 ? ((i % 32) * stride_elems + i / 32) % n : i;
      atomicAdd(p + idx, make_float2(1.f, 2.f));
    }
}
__global__ void red_f64(double* p, long n, long stride_elems, int reps) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long nthreads = gridDim.x * (long)blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (long i = tid; i < n; i += nthreads) {
      long idx = stride_elems > 1 ? ((i % 32) * stride_elems + i / 32) % n : i;
      atomicAdd(p + idx, 1.0);
    }
}
__global__ void st_f32x2(float2* p, long n, long stride_elems, int reps) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long nthreads = gridDim.x * (long)blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (long i = tid; i < n; i += nthreads) {
      long idx = stride_elems > 1 ? ((i % 32) * stride_elems + i / 32) % n : i;
      p[idx] = make_float2(1.f * r, 2.f);
    }
}
template <typename F, typename P>
void run(const char* name, F f, P* p, long n, long stride, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f<<<148 * 8, 256>>>(p, n, stride, 1); cudaDeviceSynchronize();
  cudaEventRecord(a);
  f<<<148 * 8, 256>>>(p, n, stride, reps);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)n * reps;
  printf("%-28s n=%ld stride=%ld: %.3f ms  %.3g ops/s  (%.1f GB/s payload)\n", name, n, stride, ms, ops / ms * 1e3,
         ops * sizeof(P) / ms / 1e6);
}
int main() {
  long n = 1l << 26;  // 64 Mi elements
  float2* f; double* d;
  cudaMalloc(&f, n * sizeof(float2)); cudaMalloc(&d, n * sizeof(double));
  cudaMemset(f, 0, n * sizeof(float2)); cudaMemset(d, 0, n * sizeof(double));
  for (long stride : {1l, 1l << 20}) {
    run("RED.F32x2", red_f32x2, f, n, stride, 4);
    run("RED.F64", red_f64, d, n, stride, 4);
    run("STG.64 (float2)", st_f32x2, f, n, stride, 4);
  }
  // small L2-resident footprint
  long m = 1l << 22;  // 4 Mi float2 = 32 MB
  run("RED.F32x2 L2-resident", red_f32x2, f, m, 1, 32);
  run("RED.F64 L2-resident", red_f64, d, m, 1, 32);
  run("RED.F32x2 L2 strided", red_f32x2, f, m, 1l << 17, 32);
  cudaError_t e = cudaGetLastError(); printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
