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

#define HP_MAXDIM 16
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

// Device-side bounds checks (compute-sanitizer is unavailable on this pool): compiled into the
// `make checks` variant (libhprop_b200_checks.so, -DHP_DEVICE_CHECKS) only; a failed check traps,
// which surfaces as a sticky CUDA error in the calling test.
#ifdef HP_DEVICE_CHECKS
#define HP_DCHECK(cond)                                                                          \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("HP_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,      \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define HP_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

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

// ---------------------------------------------------------------- axis views
// A view answers, for one axis and one ordinal: the (global) order j_l used
// in the ladder coefficients and the ordinals of the -/+ neighbours (-1 if
// absent).  Boxes (full cubes and j1-slabs of full cubes) use stride
// arithmetic; every other set uses device neighbour tables.
struct AxBox {
  int64_t stride;  // ordinal stride of this axis
  int side;        // local extent of this axis
  int joff;        // global offset of local j (slab shards, axis 1 only)
  __device__ __forceinline__ int jloc(int64_t o) const { return (int)((o / stride) % side); }
  __device__ __forceinline__ void at(int64_t o, int& j, int64_t& dn, int64_t& up) const {
    int jl = jloc(o);
    j = jl + joff;
    dn = jl > 0 ? o - stride : -1;
    up = jl < side - 1 ? o + stride : -1;
  }
  __device__ __forceinline__ int64_t dn_of(int64_t o) const { return jloc(o) > 0 ? o - stride : -1; }
  __device__ __forceinline__ int64_t up_of(int64_t o) const { return jloc(o) < side - 1 ? o + stride : -1; }
  // the axis line through o out to +-K: seg[K + d] = ordinal of j + d e, or -1 (one division)
  template <int K>
  __device__ __forceinline__ void segment(int64_t o, int& j, int64_t* seg) const {
    const int jl = o < (int64_t)0x7fffffff ? (int)(((unsigned)o / (unsigned)stride) % (unsigned)side) : jloc(o);
    j = jl + joff;
#pragma unroll
    for (int d = -K; d <= K; ++d) seg[K + d] = (jl + d >= 0 && jl + d < side) ? o + d * stride : -1;
  }
  // nothing to prefetch: stride arithmetic
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, int64_t* seg) const {
    segment<K>(o, j, seg);
  }
};

struct AxTab {
  const int32_t* down;
  const int32_t* up;
  const int32_t* jv;
  __device__ __forceinline__ void at(int64_t o, int& j, int64_t& dn, int64_t& up_) const {
    j = __ldg(jv + o);
    dn = __ldg(down + o);
    up_ = __ldg(up + o);
  }
  __device__ __forceinline__ int64_t dn_of(int64_t o) const { return __ldg(down + o); }
  __device__ __forceinline__ int64_t up_of(int64_t o) const { return __ldg(up + o); }
  // the axis line through o out to +-K via the tables (down chains never break in a
  // downward-closed set; up chains stop at the first pruned index)
  template <int K>
  __device__ __forceinline__ void segment(int64_t o, int& j, int64_t* seg) const {
    int64_t dn, up_;
    at(o, j, dn, up_);
    seg[K] = o;
    if (K > 0) {
      seg[K - 1] = dn;
      seg[K + 1] = up_;
    }
#pragma unroll
    for (int d = 2; d <= K; ++d) {
      seg[K - d] = seg[K - d + 1] >= 0 ? dn_of(seg[K - d + 1]) : -1;
      seg[K + d] = seg[K + d - 1] >= 0 ? up_of(seg[K + d - 1]) : -1;
    }
  }
  // no prefetch (batched levels: the walk is shared by the batch's vectors already)
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, int64_t* seg) const {
    segment<K>(o, j, seg);
  }
};

// The innermost axis of a tabled (lexicographic, downward-closed) set: its lines are contiguous
// ordinal runs starting at j = 0, so j - d e_N is o - d whenever j >= d, and o + d lies on the
// same line iff its own j equals j + d (the next line restarts at 0).  The window is formed from
// the j table alone -- K + 1 independent, coalesced loads instead of the dependent down/up walk.
struct AxInner : AxTab {
  AxInner() = default;
  explicit AxInner(const AxTab& t, int64_t n_) : AxTab(t), n(n_) {}
  int64_t n;
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, int64_t* seg) const {
    j = __ldg(jv + o);
    seg[K] = o;
#pragma unroll
    for (int d = 1; d <= K; ++d) {
      seg[K - d] = j >= d ? o - d : -1;
      seg[K + d] = (o + d < n && __ldg(jv + o + d) == j + d) ? o + d : -1;
    }
  }
};

// Precomputed windows (hp_level.cu window_table): row r < K holds the ordinal of j - (K - r) e_a,
// row r >= K that of j + (r - K + 1) e_a (-1 absent), so a level reads 2K independent coalesced
// ordinals instead of walking the down / up chains (whose second hops are scattered 4-byte reads).
struct AxWin : AxTab {
  AxWin() = default;
  AxWin(const AxTab& t, const int32_t* w, int64_t n_, int kw) : AxTab(t), win(w), n(n_), kwin(kw) {}
  const int32_t* win;
  int64_t n;
  int kwin;  // K of the stored table (>= the level's K)
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, int64_t* seg) const {
    j = __ldg(jv + o);
    seg[K] = o;
#pragma unroll
    for (int d = 1; d <= K; ++d) {
      seg[K - d] = __ldg(win + (int64_t)(kwin - d) * n + o);
      seg[K + d] = __ldg(win + (int64_t)(kwin + d - 1) * n + o);
    }
  }
};

// AxTab whose first walk hop is loaded one grid-stride iteration ahead (software pipelining of the
// dependent table chain: j / down / up of the next ordinal are in flight while the current one's
// windows are gathered).  Single-vector levels: cfg3 6.24 -> 5.91 ms; a batch of 4 slowed 1%.
struct AxTabPf : AxTab {
  AxTabPf() = default;
  explicit AxTabPf(const AxTab& t) : AxTab(t) {}
  struct Pre {
    int j;
    int32_t dn, up;
  };
  __device__ __forceinline__ Pre pre(int64_t o) const { return {__ldg(jv + o), __ldg(down + o), __ldg(up + o)}; }
  template <int K>
  __device__ __forceinline__ void segment_pre(const Pre& p, int64_t o, int& j, int64_t* seg) const {
    j = p.j;
    seg[K] = o;
    if (K > 0) {
      seg[K - 1] = p.dn;
      seg[K + 1] = p.up;
    }
#pragma unroll
    for (int d = 2; d <= K; ++d) {
      seg[K - d] = seg[K - d + 1] >= 0 ? dn_of(seg[K - d + 1]) : -1;
      seg[K + d] = seg[K + d - 1] >= 0 ? up_of(seg[K + d - 1]) : -1;
    }
  }
};

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
