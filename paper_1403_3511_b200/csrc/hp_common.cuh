// Shared definitions for the hprop_b200 CUDA library (sm_100a).
//
// Scalar arithmetic on the reference-order path uses explicit round-to-
// nearest intrinsics (__dmul_rn/__dadd_rn/__dsub_rn) so that no FMA
// contraction happens: numpy evaluates cdown*w[down] + cup*w[up] as two
// rounded products and a rounded sum (fast_apply.py:64-65, 74-92), and the
// device reproduces exactly that.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdio.h>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hprop_b200.h"
#include "hp_device.cuh"

#define HP_ABI 1

namespace hp {

void set_error(const std::string& msg);
void count_launch();
hp_status fail(hp_status code, const std::string& msg);
hp_status cuda_fail(cudaError_t e, const char* what);

#define HP_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return hp::cuda_fail(e_, #call); \
  } while (0)

// every kernel launch is followed by this check, which also counts it
// (hp_launch_count(): the "gpu_launches" figure of bench.py)
#define HP_LAUNCH_CHECK(what)                           \
  do {                                                  \
    hp::count_launch();                                 \
    cudaError_t e_ = cudaGetLastError();                \
    if (e_ != cudaSuccess) return hp::cuda_fail(e_, what); \
  } while (0)

// NVTX range around a C-ABI entry point (visible in Nsight timelines; a no-op without a tool
// attached).  NVTX v3 is header-only.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define HP_NVTX(name) hp::NvtxRange hp_nvtx_range_(name)

// Events of one streamed (host-buffer) call, destroyed on every exit path.  If the call fails
// after queueing copies on the shared copy streams, the destructor drains those streams first,
// so no queued copy still targets the caller's buffers when the error is returned.
struct StreamedEvents {
  std::vector<cudaEvent_t> ev;
  cudaStream_t drain[2] = {nullptr, nullptr};
  bool committed = false;
  hp_status create(size_t n) {
    ev.assign(n, nullptr);
    for (auto& e : ev) {
      cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return cuda_fail(r, "cudaEventCreateWithFlags");
    }
    return HP_OK;
  }
  cudaEvent_t& operator[](size_t i) { return ev[i]; }
  ~StreamedEvents() {
    if (!committed)
      for (cudaStream_t s : drain)
        if (s) cudaStreamSynchronize(s);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);  // released once the recorded work completes
  }
};

// ---------------------------------------------------------------- scalars
__device__ __forceinline__ double zero_of(double) { return 0.0; }
__device__ __forceinline__ double2 zero_of(double2) { return make_double2(0.0, 0.0); }

__device__ __forceinline__ double smul(double c, double x) { return __dmul_rn(c, x); }
__device__ __forceinline__ double2 smul(double c, double2 x) {
  return make_double2(__dmul_rn(c, x.x), __dmul_rn(c, x.y));
}
__device__ __forceinline__ double sadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double2 sadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double ssub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double2 ssub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double sdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double2 sdiv(double2 a, double b) {
  return make_double2(__ddiv_rn(a.x, b), __ddiv_rn(a.y, b));
}
// fused (contracted) variants for the fast path
__device__ __forceinline__ double sfma(double c, double x, double acc) { return fma(c, x, acc); }
__device__ __forceinline__ double2 sfma(double c, double2 x, double2 acc) {
  return make_double2(fma(c, x.x, acc.x), fma(c, x.y, acc.y));
}
__device__ __forceinline__ bool sfinite(double x) { return isfinite(x); }
__device__ __forceinline__ bool sfinite(double2 x) { return isfinite(x.x) && isfinite(x.y); }

template <class T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

}  // namespace hp

// The set handle (opaque to C callers).
struct hp_set_s {
  int dim = 0, bound = 0, kind = 0;
  int64_t n = 0;
  int device = 0;
  bool boxed = false;           // full cube or slab: stride arithmetic
  int lo = 0, hi = 0;           // slab planes along axis 1 (full: 0..bound+1)
  int64_t stride[HP_MAXDIM] = {0};
  int side[HP_MAXDIM] = {0};
  // tabled sets (hyperbolic, custom)
  int32_t* d_down[HP_MAXDIM] = {nullptr};
  int32_t* d_up[HP_MAXDIM] = {nullptr};
  int32_t* d_j[HP_MAXDIM] = {nullptr};
  // hyperbolic rank tables (host copy for position(); device copy for kernels)
  std::vector<int64_t> h_pref;  // concatenated prefix arrays
  std::vector<int64_t> h_off;   // (depth * (budget+1) + r) -> offset into h_pref, -1 if unused
  int64_t* d_pref = nullptr;
  int64_t* d_off = nullptr;
  // custom sets keep a host copy of the indices for position()
  std::vector<int64_t> h_indices;
  // full cubes: banded basis tables T_k(X_l / L) per axis, built on first use
  // of the fused evaluator (hp_fullgrid.cu) and cached per halfwidth
  mutable std::mutex fg_mtx;
  mutable double fg_L = 0.0;
  mutable double* fg_basis = nullptr;
  // single-pass evaluator: blocked tile order (packed i1 | i2 << 10 | i3 << 20)
  mutable int* fg_tiles = nullptr;
  mutable int fg_ntiles = 0;
  // the same for the quad kernel's 8 x 8 x 16 tiles (hp_fg4.cuh)
  mutable int* fg_tiles4 = nullptr;
  mutable int fg_ntiles4 = 0;
  // tabled sets: per-axis line order (ordinals grouped by axis line, hp_level.cu), built on
  // first use by the level kernels of outer axes
  mutable std::mutex perm_mtx;
  mutable int32_t* d_perm[HP_MAXDIM] = {nullptr};
  // tabled sets: precomputed +-K windows of an axis (hp_level.cu window_table), [2K][n] int32
  mutable int32_t* d_win[HP_MAXDIM] = {nullptr};
  mutable int d_win_k[HP_MAXDIM] = {0};
  // sqrt(j / 2) for j = -8 .. bound + 8 (entry j at [j + 8]): the ladder coefficients of the level
  // kernels (hp_level.cu ladder_table); boxes and hyperbolic crosses only (indices <= bound)
  mutable double* d_sqtab = nullptr;
  // tabled sets: sum_l j_l per ordinal, the oscillator levels of apply_hamiltonian (hp_level.cu level_sums)
  mutable int32_t* d_jsum = nullptr;

  hp::AxBox box(int a) const {
    hp::AxBox v;
    v.stride = stride[a];
    v.side = side[a];
    v.joff = (a == 0) ? lo : 0;
    return v;
  }
  hp::AxTab tab(int a) const {
    hp::AxTab v;
    v.down = d_down[a];
    v.up = d_up[a];
    v.jv = d_j[a];
    return v;
  }
};

namespace hp {
inline int grid_for(int64_t n, int block, int max_blocks = 148 * 16) {
  int64_t g = (n + block - 1) / block;
  if (g > max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace hp
