// Microbenchmarks for the roofline denominators this path needs and that
// MEASURED_PEAKS.json does not carry: double2 HBM copy, L2-resident read
// bandwidth, and FP64 FMA throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void copy2(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = __ldg(a + i);
}
__global__ void read2(const double2* __restrict__ a, size_t n, size_t reps, double* out) {
  double acc = 0;
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (size_t r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += s) { double2 v = __ldg(a + i); acc += v.x + v.y; }
  if (acc == 12345.678) out[0] = acc;
}
__global__ void fma64(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d}\n", p.name, p.multiProcessorCount, p.l2CacheSize);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  size_t n = (size_t)1 << 26;  // 64 Mi double2 = 1 GiB
  double2 *a, *b; double* o; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16)); CK(cudaMalloc(&o, 8));
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  int grid = p.multiProcessorCount * 8;
  for (int w = 0; w < 3; ++w) copy2<<<grid, 256>>>(a, b, n);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); copy2<<<grid, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("{\"test\": \"hbm_copy_double2\", \"bytes\": %zu, \"ms\": %.4f, \"GBs\": %.1f}\n", 2 * n * 16, best, 2.0 * n * 16 / best / 1e6);
  best = 1e9;
  for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); read2<<<grid, 256>>>(a, n, 1, o); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("{\"test\": \"hbm_read_double2\", \"bytes\": %zu, \"ms\": %.4f, \"GBs\": %.1f}\n", n * 16, best, 1.0 * n * 16 / best / 1e6);
  for (size_t mb : {8, 16, 32, 48, 64, 96}) {
    size_t m = mb * 1024 * 1024 / 16; size_t reps = 64;
    read2<<<grid, 256>>>(a, m, 2, o);
    best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); read2<<<grid, 256>>>(a, m, reps, o); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("{\"test\": \"l2_read_double2\", \"mb\": %zu, \"ms\": %.4f, \"GBs\": %.1f}\n", mb, best, 1.0 * m * 16 * reps / best / 1e6);
  }
  int iters = 4096;
  for (int th : {256, 512}) {
    fma64<<<p.multiProcessorCount * 4, th>>>(o, 16);
    best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); fma64<<<p.multiProcessorCount * 4, th>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    double flops = 2.0 * 64 * iters * (double)p.multiProcessorCount * 4 * th;
    printf("{\"test\": \"fp64_fma\", \"threads\": %d, \"ms\": %.4f, \"TFLOPs\": %.2f}\n", th, best, flops / best / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
