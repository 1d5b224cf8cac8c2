// Microbenchmark: TMA tile-load throughput vs box row width (B200).
// 148 CTAs, S-stage mbarrier pipeline, each CTA streams boxes of a 4-D f64 tensor;
// consumers only wait + arrive.  Reports GB/s of smem fill.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ bool trywait(uint64_t* b, unsigned ph) {
  unsigned ok;
  asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P; }"
               : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void tma4(void* d, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2,%3,%4,%5}], [%6];" ::"r"(sa(d)),
      "l"((unsigned long long)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(b))
      : "memory");
}
constexpr int S = 6;
// box dims b0 (doubles) x b1 x b2; nbox boxes per stage (consecutive along dim 2)
__global__ void __launch_bounds__(512, 1) k(const __grid_constant__ CUtensorMap m, int b0, int b1, int b2, int nbox,
                                            int n1t, int n2t, int n3t, int items, int pmod) {
  extern __shared__ __align__(128) unsigned char sm[];
  const unsigned stage_bytes = (unsigned)b0 * b1 * b2 * 8 * nbox;
  uint64_t* full = (uint64_t*)(sm + S * stage_bytes);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 16); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int it) {
    int s = it % S, u = it / S;
    if (u > 0) while (!trywait(&empty[s], (u - 1) & 1)) {}
    expect(&full[s], stage_bytes);
    int tile = blockIdx.x + (it / 128) * gridDim.x;
    int p = (it % 128) % pmod;
    int t3 = tile % n3t, t2 = (tile / n3t) % n2t, t1 = tile / (n3t * n2t) % n1t;
    for (int q = 0; q < nbox; ++q)
      tma4(sm + s * stage_bytes + q * (stage_bytes / nbox), &m, t3 * b0, t2 * b1, t1 * b2 * nbox + q * b2, p, &full[s]);
  };
  if (tid == 0) for (int i = 0; i < S - 1; ++i) issue(i);
  for (int it = 0; it < items; ++it) {
    if (tid == 0 && it + S - 1 < items) issue(it + S - 1);
    int s = it % S;
    while (!trywait(&full[s], (it / S) & 1)) {}
    __syncwarp();
    if (lane == 0) arrive(&empty[s]);
  }
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int n = 128;
  void* v;
  size_t bytes = (size_t)n * n * n * n * 16;
  cudaMalloc(&v, bytes);
  cudaMemset(v, 0, bytes);
  struct Cfg { int b0, b1, b2, nbox; const char* name; };
  Cfg cfgs[] = {{16, 8, 16, 1, "rows 128B, 16x8x16"}, {8, 8, 8, 4, "rows 64B"}, {32, 8, 8, 2, "rows 256B"},
                {64, 4, 8, 2, "rows 512B"}, {16, 8, 8, 4, "rows 128B 4 boxes"}, {256, 2, 4, 2, "rows 2KB"}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& c : cfgs) {
    CUtensorMap m;
    cuuint64_t dims[4] = {2ull * n, (cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t str[3] = {16ull * n, 16ull * n * n, 16ull * n * n * n};
    cuuint32_t box[4] = {(cuuint32_t)c.b0, (cuuint32_t)c.b1, (cuuint32_t)c.b2, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, v, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", (int)r); continue; }
    unsigned stage = c.b0 * c.b1 * c.b2 * 8 * c.nbox;
    size_t smem = S * stage + 256;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n1t = n / (c.b2 * c.nbox), n2t = n / c.b1, n3t = (2 * n) / c.b0;
    int tiles = n1t * n2t * n3t;
    int items = (tiles / 148) * 128;
    for (int pmod : {128, 2}) for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k<<<148, 512, smem>>>(m, c.b0, c.b1, c.b2, c.nbox, n1t, n2t, n3t, items, pmod);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double gb = (double)items * 148 * stage / 1e9;
      if (rep) printf("pmod %3d %-22s stage %6u B  %.3f ms  %.0f GB/s  err=%s\n", pmod, c.name, stage, ms, gb / ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
