// Microbenchmark: SHFL (64-bit via 2x32) vs LDS.128 throughput per SM on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_shfl(double* out, int iters) {
  double a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  for (int i = 0; i < iters; ++i) {
    a += __shfl_xor_sync(0xffffffffu, b, 1);
    b += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, d, 4);
    d += __shfl_xor_sync(0xffffffffu, a, 8);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_lds(double* out, int iters) {
  __shared__ double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int o = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double2 x0 = sm[(o + 0) & 2047], x1 = sm[(o + 64) & 2047], x2 = sm[(o + 128) & 2047], x3 = sm[(o + 192) & 2047];
    acc.x += x0.x + x1.x + x2.x + x3.x;
    acc.y += x0.y + x1.y + x2.y + x3.y;
    o += 7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}
__global__ void k_mix(double* out, int iters) {
  __shared__ double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  double a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  int o = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double2 x0 = sm[(o + 0) & 2047], x1 = sm[(o + 64) & 2047], x2 = sm[(o + 128) & 2047], x3 = sm[(o + 192) & 2047];
    acc.x += x0.x + x1.x + x2.x + x3.x;
    acc.y += x0.y + x1.y + x2.y + x3.y;
    o += 7;
    a += __shfl_xor_sync(0xffffffffu, b, 1);
    b += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, d, 4);
    d += __shfl_xor_sync(0xffffffffu, a, 8);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + a + b + c + d;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 1024 * 8);
  int iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_shfl<<<148, 512>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per SM: 16 warps * iters * 4 shfl64 (= 8 SHFL.32)
    double shfl32 = 16.0 * iters * 8;
    printf("SHFL.32 per SM per ns: %.3f  (%.3f per clk at 1.965 GHz)\n", shfl32 / (ms * 1e6), shfl32 / (ms * 1e6) / 1.965);
    cudaEventRecord(e0);
    k_lds<<<148, 512>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double lds = 16.0 * iters * 4;
    printf("LDS.128 warp-instr per SM per clk: %.3f\n", lds / (ms * 1e6) / 1.965);
    cudaEventRecord(e0);
    k_mix<<<148, 512>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mix: clk per iteration per warp-slot: %.2f (LDS alone 16, SHFL alone 8 if separate)\n", (ms * 1e6) * 1.965 / (16.0 * iters));
  }
  return 0;
}
