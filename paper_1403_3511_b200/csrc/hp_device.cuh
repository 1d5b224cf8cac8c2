// Device-side building blocks of the hprop_b200 library: axis views, block reductions and the
// level kernel.  Self-contained (CUDA built-ins only) so that the same source is compiled twice:
// by nvcc into the library, and at run time by NVRTC with a level's structure as compile-time
// constants (hp_level_jit.cu embeds this file as a string).
#pragma once

#ifdef __CUDACC_RTC__
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
#else
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#endif

#define HP_MAXDIM 16

// Device-side bounds checks (compute-sanitizer is unavailable on this pool): compiled into the
// `make checks` variant (libhprop_b200_checks.so, -DHP_DEVICE_CHECKS) only; a failed check traps,
// which surfaces as a sticky CUDA error in the calling test.
#if defined(HP_DEVICE_CHECKS) && !defined(__CUDACC_RTC__)
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


namespace hp {

// ---------------------------------------------------------------- axis views
// A view answers, for one axis and one ordinal: the (global) order j_l used
// in the ladder coefficients and the ordinals of the -/+ neighbours (-1 if
// absent).  Boxes (full cubes and j1-slabs of full cubes) use stride
// arithmetic; every other set uses device neighbour tables.
struct AxBox {
  typedef int64_t Idx;  // window ordinals of a box can exceed 32 bits
  typedef int64_t UIdx;
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::AxBox"; }  // type name in runtime-compiled source
#endif
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
  template <int K, class I>
  __device__ __forceinline__ void segment(int64_t o, int& j, I* seg) const {
    const int jl = o < (int64_t)0x7fffffff ? (int)(((unsigned)o / (unsigned)stride) % (unsigned)side) : jloc(o);
    j = jl + joff;
#pragma unroll
    for (int d = -K; d <= K; ++d) seg[K + d] = (jl + d >= 0 && jl + d < side) ? (I)(o + d * stride) : (I)-1;
  }
  // nothing to prefetch: stride arithmetic
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K, class I>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, I* seg) const {
    segment<K>(o, j, seg);
  }
};

struct AxTab {
  typedef uint32_t UIdx;
  typedef int32_t Idx;  // tabled sets hold int32 ordinals: half the registers of the window
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::AxTab"; }  // type name in runtime-compiled source
#endif
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
  template <int K, class I>
  __device__ __forceinline__ void segment(int64_t o, int& j, I* seg) const {
    int64_t dn, up_;
    at(o, j, dn, up_);
    seg[K] = (I)o;
    if (K > 0) {
      seg[K - 1] = (I)dn;
      seg[K + 1] = (I)up_;
    }
#pragma unroll
    for (int d = 2; d <= K; ++d) {
      seg[K - d] = seg[K - d + 1] >= 0 ? (I)dn_of(seg[K - d + 1]) : (I)-1;
      seg[K + d] = seg[K + d - 1] >= 0 ? (I)up_of(seg[K + d - 1]) : (I)-1;
    }
  }
  // no prefetch (batched levels: the walk is shared by the batch's vectors already)
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K, class I>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, I* seg) const {
    segment<K>(o, j, seg);
  }
};

// The innermost axis of a tabled (lexicographic, downward-closed) set: its lines are contiguous
// ordinal runs starting at j = 0, so j - d e_N is o - d whenever j >= d, and o + d lies on the
// same line iff its own j equals j + d (the next line restarts at 0).  The window is formed from
// the j table alone -- K + 1 independent, coalesced loads instead of the dependent down/up walk.
struct AxInner : AxTab {
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::AxInner"; }  // type name in runtime-compiled source
#endif
  AxInner() = default;
  __host__ __device__ explicit AxInner(const AxTab& t, int64_t n_) : AxTab(t), n(n_) {}
  int64_t n;
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K, class I>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, I* seg) const {
    j = __ldg(jv + o);
    seg[K] = (I)o;
#pragma unroll
    for (int d = 1; d <= K; ++d) {
      seg[K - d] = j >= d ? (I)(o - d) : (I)-1;
      seg[K + d] = (o + d < n && __ldg(jv + o + d) == j + d) ? (I)(o + d) : (I)-1;
    }
  }
};

// Precomputed windows (hp_level.cu window_table): row r < K holds the ordinal of j - (K - r) e_a,
// row r >= K that of j + (r - K + 1) e_a (-1 absent), so a level reads 2K independent coalesced
// ordinals instead of walking the down / up chains (whose second hops are scattered 4-byte reads).
struct AxWin : AxTab {
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::AxWin"; }  // type name in runtime-compiled source
#endif
  AxWin() = default;
  __host__ __device__ AxWin(const AxTab& t, const int32_t* w, int64_t n_, int kw) : AxTab(t), win(w), n(n_), kwin(kw) {}
  const int32_t* win;
  int64_t n;
  int kwin;  // K of the stored table (>= the level's K)
  struct Pre {};
  __device__ __forceinline__ Pre pre(int64_t) const { return {}; }
  template <int K, class I>
  __device__ __forceinline__ void segment_pre(const Pre&, int64_t o, int& j, I* seg) const {
    j = __ldg(jv + o);
    seg[K] = (I)o;
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
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::AxTabPf"; }  // type name in runtime-compiled source
#endif
  AxTabPf() = default;
  __host__ __device__ explicit AxTabPf(const AxTab& t) : AxTab(t) {}
  struct Pre {
    int j;
    int32_t dn, up;
  };
  __device__ __forceinline__ Pre pre(int64_t o) const { return {__ldg(jv + o), __ldg(down + o), __ldg(up + o)}; }
  template <int K, class I>
  __device__ __forceinline__ void segment_pre(const Pre& p, int64_t o, int& j, I* seg) const {
    j = p.j;
    seg[K] = (I)o;
    if (K > 0) {
      seg[K - 1] = p.dn;
      seg[K + 1] = p.up;
    }
#pragma unroll
    for (int d = 2; d <= K; ++d) {
      seg[K - d] = seg[K - d + 1] >= 0 ? (I)dn_of(seg[K - d + 1]) : (I)-1;
      seg[K + d] = seg[K + d - 1] >= 0 ? (I)up_of(seg[K + d - 1]) : (I)-1;
    }
  }
};


// block-wide sum of a double2 (blockDim multiple of 32, <= 1024); result valid in thread 0
__device__ __forceinline__ double2 block_sum2(double2 v) {
  __shared__ double2 red_sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red_sh[w] = v;
  __syncthreads();
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? red_sh[lane] : make_double2(0.0, 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_down_sync(0xffffffffu, v.x, o);
      v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
  }
  return v;
}
// conj(a) * b accumulated into acc
__device__ __forceinline__ void cdot_acc(double2 a, double2 b, double2& acc) {
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
}


// ---------------------------------------------------------------- level kernel (hp_level.cu)

// a present window ordinal as an unsigned element index
__device__ __forceinline__ uint32_t lv_uidx(int32_t i) { return (uint32_t)i; }
__device__ __forceinline__ int64_t lv_uidx(int64_t i) { return i; }

constexpr int LV_MAXIN = 64;
constexpr int LV_MAXTG = 16;  // targets accumulate in registers
constexpr int LV_MAXENT = 160;
constexpr int LV_MAXDIRECT = 48;
constexpr int LV_WT = 640;  // dense weights: nin * (K + 1) * tgn doubles
constexpr int LV_MAXK = 4;

struct LvEnt {
  unsigned char input;  // index into in_buf
  unsigned char tg;     // index into tg_buf (accumulated target), or 0xFF: write w * T_k to `slot`
  signed char k;        // degree
  short slot;
  double w;
};

// a child vector with a single term: slot <- w T_k(X_a) input
struct LvDirect {
  short slot;
  signed char k;
  double w;
};
// One level as the kernel reads it (passed by value: constant bank).  Accumulated targets use a
// DENSE weight table wt[(i * (K + 1) + k) * tgn + q] (zero where input i, degree k does not feed
// target q), so the kernel's loops over degrees and targets are compile-time and an entry costs
// one complex FMA with a uniform operand -- no per-entry decoding.  Child vectors with a single
// term are written directly (`direct`), which keeps the accumulator count small.
struct LvLevel {
  int axis;
  int K;
  int nin, ntg;
  int tgn;                  // accumulators of the kernel instantiation (1, 2, 4, 8, 16): stride of wt
  short in_buf[LV_MAXIN];   // -2 = v, >= 0 slot
  short tg_buf[LV_MAXTG];   // -1 = y, >= 0 slot
  unsigned short in_pmask[LV_MAXIN];  // window positions (bit p = offset p - K) the entries of input i read
  unsigned char in_kmask[LV_MAXIN];   // degrees k of input i that feed accumulated targets
  unsigned char in_dmask[LV_MAXIN];   // degrees k of input i with directly written children
  short d_start[LV_MAXIN + 1];        // direct entries of input i: direct[d_start[i] .. d_start[i + 1])
  LvDirect direct[LV_MAXDIRECT];
  double wt[LV_WT];
  __device__ __forceinline__ int ntg_() const { return ntg; }
  __device__ __forceinline__ int tg_buf_(int q) const { return tg_buf[q]; }
  // every input vector of the level: T_k x at o from the band rows, then its entries
  template <int K, int TGN, class I>
  __device__ __forceinline__ void inputs(const double (&R)[K + 1][2 * K + 1], const I (&seg)[2 * K + 1],
                                         const double2* __restrict__ v, double2* __restrict__ slots, int64_t nbn,
                                         int64_t bo, int64_t o, double2 (&accs)[TGN]) const {
    constexpr int S = 2 * K + 1;
    for (int ii = 0; ii < nin; ++ii) {
      const int ib = in_buf[ii];
      const double2* x = ib == -2 ? v + bo : slots + (int64_t)ib * nbn + bo;
      asm volatile("" : "+l"(x));  // formed once per input, not rematerialised at every load
      const unsigned need = in_pmask[ii];  // window positions some entry of this input reads
      const unsigned km = in_kmask[ii], dm = in_dmask[ii];
      double2 xw[S];
#pragma unroll
      for (int p = 0; p < S; ++p) {
        xw[p] = ((need >> p) & 1u) && seg[p] >= 0 ? __ldg(x + lv_uidx(seg[p])) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k <= K; ++k) {
        if (!(((km | dm) >> k) & 1u)) continue;  // uniform: no entry of (input, degree)
        double2 tk = make_double2(0.0, 0.0);
        if (k == 0) tk = xw[K];
#pragma unroll
        for (int p = 0; p < S; ++p) {
          const int d = p - K;
          if (k == 0 || d < -k || d > k || ((d + k) & 1)) continue;
          tk.x = fma(R[k][p], xw[p].x, tk.x);
          tk.y = fma(R[k][p], xw[p].y, tk.y);
        }
        if ((km >> k) & 1u) {
#pragma unroll
          for (int q = 0; q < TGN; ++q) {
            const double w = wt[(ii * (K + 1) + k) * TGN + q];
            accs[q].x = fma(w, tk.x, accs[q].x);
            accs[q].y = fma(w, tk.y, accs[q].y);
          }
        }
        if ((dm >> k) & 1u)
          for (int e = d_start[ii]; e < d_start[ii + 1]; ++e)
            if (direct[e].k == k) {
              const double w = direct[e].w;
              slots[(int64_t)direct[e].slot * nbn + bo + o] = make_double2(w * tk.x, w * tk.y);
            }
      }
    }
  }
};

// T_KK x at o: the band row against the window (positions of KK's parity within +-KK)
template <int K, int KK>
__device__ __forceinline__ double2 lv_band(const double (&R)[K + 1][2 * K + 1], const double2 (&xw)[2 * K + 1]) {
  double2 t = make_double2(0.0, 0.0);
  if (KK == 0) t = xw[K];
#pragma unroll
  for (int p = 0; p < 2 * K + 1; ++p) {
    const int d = p - K;
    if (KK == 0 || d < -KK || d > KK || ((d + KK) & 1)) continue;
    t.x = fma(R[KK][p], xw[p].x, t.x);
    t.y = fma(R[KK][p], xw[p].y, t.y);
  }
  return t;
}

// Pieces of a runtime-specialised level (hp_level_jit.cu writes LvGen::inputs() as a sequence of
// these with literal arguments; `w` is the level's weight array, a kernel parameter):
//   LV_GEN_IN(ptr) LV_GEN_LOAD(p).. { LV_GEN_T(k) LV_GEN_ACC(q, wi).. LV_GEN_DIRECT(slot, wi).. LV_GEN_T_END }.. LV_GEN_IN_END
#define LV_GEN_IN(ptr)                                                                       \
  {                                                                                          \
    const double2* x_ = (ptr);                                                               \
    asm volatile("" : "+l"(x_)); /* formed once per input, not rematerialised at every load */ \
    double2 xw_[2 * K + 1];
#define LV_GEN_LOAD(p) xw_[p] = seg[p] >= 0 ? __ldg(x_ + lv_uidx(seg[p])) : make_double2(0.0, 0.0);
#define LV_GEN_T(k) \
  {                 \
    const double2 t_ = lv_band<K, k>(R, xw_);
#define LV_GEN_ACC(q, wi)                    \
  accs[q].x = fma(w[wi], t_.x, accs[q].x); \
  accs[q].y = fma(w[wi], t_.y, accs[q].y);
#define LV_GEN_DIRECT(slot, wi) \
  slots[(int64_t)(slot) * nbn + bo + o] = make_double2(w[wi] * t_.x, w[wi] * t_.y);
#define LV_GEN_T_END }
#define LV_GEN_IN_END }

#ifndef LV_MINB
// minimum resident 256-thread blocks per SM handed to ptxas: 4 (<= 64 registers).  Occupancy beats
// spill traffic on these gather kernels (profiles/r2/sweep_level.txt, dense-weight kernels: cfg3
// 6.00 ms uncapped (76 registers), 5.13 at 4 blocks, 6.04 at 5, 7.11 at 6; cfg5 654 / 511 / 699 /
// 874 ms)
#define LV_MINB 4
#endif
// PROG is the level as the kernel reads it: LvLevel (the interpreted form compiled into the library)
// or a runtime-specialised LvGen whose inputs() is straight-line code (hp_level_jit.cu).
template <int K, int TGN, class AX, class AXS, class PROG>
__device__ __forceinline__ void lv_body(int64_t n, int64_t batch, const AX& ax, const AXS& axs, int dim, const PROG& lv,
                                               double inv_L, double two_L, const double2* __restrict__ v,
                                               double2* __restrict__ slots, double2* __restrict__ y, int first,
                                               int osc, double2* __restrict__ dotp,
                                               const int32_t* __restrict__ perm,
                                               const double* __restrict__ sqtab) {
  constexpr int S = 2 * K + 1;
  double2 dacc = make_double2(0.0, 0.0);
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // perm (outer axes of tabled sets): line-blocked order (line_order below), so the +-K
  // windows of neighbouring warps overlap in L1/L2 (ordinal order puts the window positions
  // one sub-block apart, far beyond L2 reuse)
  int64_t o_next = t < n ? (perm ? (int64_t)__ldg(perm + t) : t) : 0;
  typename AX::Pre pre_next = ax.pre(o_next);
  for (; t < n; t += gstride) {
    const int64_t o = o_next;
    const typename AX::Pre pre_o = pre_next;
    if (t + gstride < n) {  // the next ordinal's first walk hop, in flight during this one
      o_next = perm ? (int64_t)__ldg(perm + t + gstride) : t + gstride;
      pre_next = ax.pre(o_next);
    }
    // the axis line through o: seg[K + d] = ordinal of j + d e_a, or -1
    typename AX::Idx seg[S];  // int32 on tabled sets
    int jo;
    ax.template segment_pre<K>(pre_o, o, jo, seg);
    // links of the window: lk[p] = sqrt(j_p / 2) couples positions p - 1 and p (cd at p = cu at
    // p - 1); a link with an absent end is 0, which is the restriction of the ladder to the set
    double lk[S + 1];
#pragma unroll
    for (int p = 1; p < S; ++p) {
      const int j = jo + p - K;
      lk[p] = (seg[p - 1] >= 0 && seg[p] >= 0) ? (sqtab ? __ldg(sqtab + j) : sqrt(j * 0.5)) : 0.0;
    }
    // band rows R_k[p] = [T_k(X_a / L)]_{o, o + (p - K) e_a} of the restricted operator, by the
    // three-term recurrence on the row vector (the operator is symmetric); T_k couples only
    // offsets d = p - K with |d| <= k and d = k mod 2.  Formed once per ordinal and shared by
    // every input vector and batch member: an input costs k + 1 complex FMAs per degree.
    double R[K + 1][S];
#pragma unroll
    for (int k = 1; k <= K; ++k) {
      const double sc = k == 1 ? inv_L : two_L;
#pragma unroll
      for (int p = 0; p < S; ++p) {
        const int d = p - K;
        if (d < -k || d > k || ((d + k) & 1)) continue;
        double a = 0.0;
        // (R_{k-1} J)[p] = R_{k-1}[p-1] lk[p] + R_{k-1}[p+1] lk[p+1]
        if (d - 1 >= -(k - 1)) a = (k == 1 ? 1.0 : R[k - 1][p - 1]) * lk[p];
        if (d + 1 <= k - 1) a = (d - 1 >= -(k - 1)) ? fma(k == 1 ? 1.0 : R[k - 1][p + 1], lk[p + 1], a)
                                                    : (k == 1 ? 1.0 : R[k - 1][p + 1]) * lk[p + 1];
        a *= sc;
        if (k >= 2 && d >= -(k - 2) && d <= k - 2) a -= (k == 2 ? 1.0 : R[k - 2][p]);
        R[k][p] = a;
      }
    }
    const double lev = osc ? axs.level(dim, o) : 0.0;  // oscillator level sum_l (j_l + 1/2)
    for (int64_t b = 0; b < batch; ++b) {
      const int64_t bo = b * n;
      double2 accs[TGN];
#pragma unroll
      for (int q = 0; q < TGN; ++q) accs[q] = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < S; ++p) HP_DCHECK(seg[p] < n);
      lv.template inputs<K, TGN>(R, seg, v, slots, n * batch, bo, o, accs);
#pragma unroll
      for (int tgi = 0; tgi < TGN; ++tgi) {
        if (tgi >= lv.ntg_()) break;
        double2 acc = accs[tgi];
        const int tb = lv.tg_buf_(tgi);
        if (tb >= 0) {
          slots[(int64_t)tb * n * batch + bo + o] = acc;
        } else {
          if (osc) {
            double2 x = __ldg(v + bo + o);
            acc.x = fma(lev, x.x, acc.x);
            acc.y = fma(lev, x.y, acc.y);
          }
          if (!first) {
            double2 old = y[bo + o];
            acc.x += old.x;
            acc.y += old.y;
          }
          y[bo + o] = acc;
          if (dotp) cdot_acc(__ldg(v + bo + o), acc, dacc);
        }
      }
    }
  }
  if (dotp) {
    dacc = block_sum2(dacc);
    if (threadIdx.x == 0) dotp[blockIdx.x] = dacc;
  }
}

template <int K, int TGN, class AX, class AXS, class PROG>
__global__ void __launch_bounds__(256, LV_MINB) k_level(int64_t n, int64_t batch, AX ax, AXS axs, int dim, PROG lv,
                                               double inv_L, double two_L, const double2* __restrict__ v,
                                               double2* __restrict__ slots, double2* __restrict__ y, int first,
                                               int osc, double2* __restrict__ dotp,
                                               const int32_t* __restrict__ perm,
                                               const double* __restrict__ sqtab) {
  lv_body<K, TGN>(n, batch, ax, axs, dim, lv, inv_L, two_L, v, slots, y, first, osc, dotp, perm, sqtab);
}

struct LvAllBox {
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::LvAllBox"; }  // type name in runtime-compiled source
#endif
  AxBox ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return ax[a].jloc(o) + ax[a].joff; }
  __device__ __forceinline__ double level(int dim, int64_t o) const {
    double lev = 0.0;
    for (int a = 0; a < dim; ++a) lev += (double)j(a, o) + 0.5;
    return lev;
  }
};
struct LvAllTab {
#ifndef __CUDACC_RTC__
  static const char* name() { return "hp::LvAllTab"; }  // type name in runtime-compiled source
#endif
  AxTab ax[HP_MAXDIM];
  const int32_t* jsum;  // sum_l j_l per ordinal (hp_level.cu level_sums), or null
  __device__ __forceinline__ int j(int a, int64_t o) const { return __ldg(ax[a].jv + o); }
  // sum_l (j_l + 1/2): exact in double either way; one 4-byte load instead of one per axis
  __device__ __forceinline__ double level(int dim, int64_t o) const {
    if (jsum) return (double)__ldg(jsum + o) + 0.5 * dim;
    double lev = 0.0;
    for (int a = 0; a < dim; ++a) lev += (double)j(a, o) + 0.5;
    return lev;
  }
};


}  // namespace hp
