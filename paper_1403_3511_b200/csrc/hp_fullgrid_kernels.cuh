// Pass A / pass B kernels of the fused full-cube evaluator (see hp_fullgrid.cu).
//
// Both kernels march one axis with a register window whose slots rotate by
// compile-time index (the march loop is unrolled by lcm of the window
// lengths), so no register moves are spent shifting windows.  Planes/rows
// stream through a zero-padded cp.async (LDGSTS) ring in shared memory; the
// neighbours along the second axis of each pass are read straight from the
// ring row, and the pads make those reads branch-free.  Band masks are
// template parameters: the cfg4 potential only populates even diagonals
// (plus +-1 for the x1*x2 coupling), and unused diagonals cost nothing.
#pragma once

#include <utility>

namespace hp {

template <int I>
using IC = std::integral_constant<int, I>;
template <class F, int... I>
__device__ __forceinline__ void unroll_seq(F&& f, std::integer_sequence<int, I...>) {
  (f(IC<I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void unroll(F&& f) {
  unroll_seq(f, std::make_integer_sequence<int, N>{});
}
constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
constexpr int clcm(int a, int b) { return a / cgcd(a, b) * b; }

__device__ __forceinline__ double2 zz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ void fma2(double c, double2 x, double2& acc) {
  acc.x = fma(c, x.x, acc.x);
  acc.y = fma(c, x.y, acc.y);
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr unsigned FG_MASK_ALL = (1u << FG_W) - 1;
constexpr unsigned FG_MASK_EVEN = 0x155;             // diagonals -4,-2,0,2,4
constexpr unsigned FG_MASK_EVEN_PM1 = 0x155 | 0x28;  // plus -1,+1

// ---------------------------------------------------------------- pass B
// u = (P_3 (x) I + I (x) P_4) v on every (j1, j2) block of n2 x n3 elements.
// CTA = one block, one thread per j4 column, marching j3.
constexpr int FGB_D = 6;                  // rows in flight
constexpr int FGB_NS = 16;                // ring rows (>= FG_K + FGB_D + 2, power of 2)

template <unsigned M2, unsigned M3>
__global__ void __launch_bounds__(128) k_fg_inner2(const double2* __restrict__ v, double2* __restrict__ u,
                                                   const double* __restrict__ P2, const double* __restrict__ P3,
                                                   int n2, int n3) {
  extern __shared__ double2 ring[];  // [FGB_NS][n3 + 2K], pads zero
  const int t = threadIdx.x;
  const int RW = n3 + 2 * FG_K;
  const bool act = t < n3;
  const int64_t base = (int64_t)blockIdx.x * n2 * n3;
  const double2* vb = v + base;
  double2* ub = u + base;
  for (int i = t; i < FGB_NS * 2 * FG_K; i += blockDim.x) {
    int slot = i / (2 * FG_K), k = i % (2 * FG_K);
    ring[slot * RW + (k < FG_K ? k : n3 + k)] = zz();
  }
  double p3[FG_W];
#pragma unroll
  for (int d = 0; d < FG_W; ++d) p3[d] = ((M3 >> d) & 1) && act ? __ldg(P3 + t * FG_W + d) : 0.0;
  auto issue = [&](int r) {
    if (!act) return;
    bool ok = r < n2;
    cp_async16(ring + (r & (FGB_NS - 1)) * RW + FG_K + t, ok ? (const void*)(vb + (int64_t)r * n3 + t) : (const void*)vb,
               ok ? 16 : 0);
  };
  // prologue: group 0 = rows 0..K, then one group per row K+1 .. K+D-1
  for (int r = 0; r <= FG_K; ++r) issue(r);
  cp_commit();
#pragma unroll
  for (int r = 1; r < FGB_D; ++r) {
    issue(FG_K + r);
    cp_commit();
  }
  cp_wait<FGB_D - 1>();
  __syncthreads();
  // window slot of row q is (q + K) mod W; before step 0 it holds rows -K-1 .. K-1
  double2 V[FG_W];
#pragma unroll
  for (int q = -FG_K - 1; q <= FG_K - 1; ++q) {
    const int s = ((q + FG_K) % FG_W + FG_W) % FG_W;
    V[s] = (act && q >= 0 && q < n2) ? ring[(q & (FGB_NS - 1)) * RW + FG_K + t] : zz();
  }
  for (int i0 = 0; i0 < n2; i0 += FG_W) {
    unroll<FG_W>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const int i = i0 + k;
      if (i >= n2) return;
      // this row's j3 band (uniform), loaded before the barrier so its latency hides behind it
      double p2[FG_W];
      const double* p2r = P2 + (size_t)i * FG_W;
#pragma unroll
      for (int d = 0; d < FG_W; ++d) p2[d] = ((M2 >> d) & 1) ? __ldg(p2r + d) : 0.0;
      issue(i + FG_K + FGB_D);
      cp_commit();
      cp_wait<FGB_D>();
      __syncthreads();
      constexpr int snew = (k + 2 * FG_K) % FG_W;  // row i + K
      V[snew] = act ? ring[((i + FG_K) & (FGB_NS - 1)) * RW + FG_K + t] : zz();
      if (act) {
        const double2* row = ring + (i & (FGB_NS - 1)) * RW + t;  // row[d] = element j4 + d - K
        double2 acc = zz(), acc2 = zz();
#pragma unroll
        for (int d = 0; d < FG_W; ++d) {
          if ((M2 >> d) & 1) fma2(p2[d], V[(k + d) % FG_W], acc);  // row i + d - K
          if (d != FG_K && ((M3 >> d) & 1)) fma2(p3[d], row[d], acc2);
        }
        fma2(p3[FG_K], V[(k + FG_K) % FG_W], acc2);
        ub[(int64_t)i * n3 + t] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
      }
    });
  }
  cp_wait<0>();
}

// ---------------------------------------------------------------- pass A
// y = u + P_1 v + P_2 v + sum_m B_{1,r0_m} (G_m v): one CTA per FG_C-element
// inner chunk, one thread per (j2, inner element), marching j1.
constexpr int FGA_D = 6;    // planes in flight
constexpr int FGA_NS = 16;  // v ring (>= FG_K + FGA_D + 2, power of 2)
constexpr int FGA_NU = 8;   // u ring (>= FGA_D + 2, power of 2)

template <int RM, int NMIX, unsigned M0, unsigned M1>
__global__ void __launch_bounds__(512, 1) k_fg_outer2(const double2* __restrict__ v, const double2* __restrict__ u,
                                                      double2* __restrict__ y, const double* __restrict__ P0,
                                                      const double* __restrict__ P1, const double* __restrict__ G,
                                                      const double* __restrict__ B0, int n0, int n1, int64_t S0,
                                                      int64_t S1, int r0a, int r0b, double2* __restrict__ dotp) {
  constexpr int WS = RM + 1, WG = 2 * RM + 1;
  double2 dacc = zz();  // <v, y> partial (Lanczos alpha), only if dotp
  constexpr int U = clcm(FG_W, clcm(WS, WG));
  constexpr int NM = NMIX > 0 ? NMIX : 1;
  extern __shared__ double2 sm[];
  const int tile = n1 * FG_C;
  const int SL = (n1 + 2 * FG_K) * FG_C;  // ring slot with K zero rows above and below
  double2* ring = sm;
  double2* uring = sm + FGA_NS * SL;
  const int t = threadIdx.x;
  const bool act = t < tile;
  const int j1 = t / FG_C, e = t % FG_C;
  const int64_t off = (int64_t)j1 * S1 + (int64_t)blockIdx.x * FG_C + e;
  const int me = (FG_K + j1) * FG_C + e;  // my element inside a ring slot
  for (int i = t; i < FGA_NS * 2 * FG_K * FG_C; i += blockDim.x) {
    int slot = i / (2 * FG_K * FG_C), k = i % (2 * FG_K * FG_C);
    sm[slot * SL + (k < FG_K * FG_C ? k : tile + k)] = zz();
  }
  double p1[FG_W];
  double g[NM][FG_W];
#pragma unroll
  for (int d = 0; d < FG_W; ++d) {
    p1[d] = act && ((M1 >> d) & 1) ? __ldg(P1 + j1 * FG_W + d) : 0.0;
#pragma unroll
    for (int m = 0; m < NM; ++m)
      g[m][d] = act && m < NMIX && ((M1 >> d) & 1) ? __ldg(G + (size_t)m * FG_MAXN * FG_W + j1 * FG_W + d) : 0.0;
  }
  const int r0s[2] = {r0a, r0b};
  auto issue_v = [&](int p) {
    if (!act) return;
    bool ok = p < n0;
    cp_async16(ring + (p & (FGA_NS - 1)) * SL + me, ok ? (const void*)(v + (int64_t)p * S0 + off) : (const void*)v,
               ok ? 16 : 0);
  };
  auto issue_u = [&](int p) {
    if (!act) return;
    bool ok = p < n0;
    cp_async16(uring + (p & (FGA_NU - 1)) * tile + t, ok ? (const void*)(u + (int64_t)p * S0 + off) : (const void*)u,
               ok ? 16 : 0);
  };
  for (int p = 0; p <= FG_K; ++p) issue_v(p);
  issue_u(0);
  cp_commit();
#pragma unroll
  for (int k = 1; k < FGA_D; ++k) {
    issue_v(FG_K + k);
    issue_u(k);
    cp_commit();
  }
  cp_wait<FGA_D - 1>();
  __syncthreads();

  // j2 bands of plane q read from the ring: s1 = P_1 v(q), gm = G_m v(q)
  auto exchange = [&](int q, double2& s1, double2 (&gm)[NM]) {
    s1 = zz();
#pragma unroll
    for (int m = 0; m < NM; ++m) gm[m] = zz();
    if (q >= n0 || !act) return;
    const double2* pl = ring + (q & (FGA_NS - 1)) * SL + me;
#pragma unroll
    for (int d = 0; d < FG_W; ++d) {
      if (!((M1 >> d) & 1)) continue;
      double2 x = pl[(d - FG_K) * FG_C];
      fma2(p1[d], x, s1);
#pragma unroll
      for (int m = 0; m < NMIX; ++m) fma2(g[m][d], x, gm[m]);
    }
  };

  // windows before step 0: V slot (q + K) mod W holds plane q in [-K-1, K-1];
  // S1W slot q mod WS holds s1(q), q in [-1, RM-1]; GW slot (q + RM) mod WG holds g(q)
  double2 V[FG_W], S1W[WS], GW[NM][WG];
#pragma unroll
  for (int q = -FG_K - 1; q <= FG_K - 1; ++q) {
    const int s = ((q + FG_K) % FG_W + FG_W) % FG_W;
    V[s] = (act && q >= 0 && q < n0) ? ring[(q & (FGA_NS - 1)) * SL + me] : zz();
  }
#pragma unroll
  for (int q = -1; q <= RM - 1; ++q) {
    double2 s1, gm[NM];
    exchange(q < 0 ? n0 : q, s1, gm);  // q < 0: zeros
    S1W[((q % WS) + WS) % WS] = s1;
#pragma unroll
    for (int m = 0; m < NM; ++m) GW[m][(((q + RM) % WG) + WG) % WG] = gm[m];
  }
#pragma unroll
  for (int q = -RM - 1; q < -1; ++q)
#pragma unroll
    for (int m = 0; m < NM; ++m) GW[m][(((q + RM) % WG) + WG) % WG] = zz();

  for (int p0 = 0; p0 < n0; p0 += U) {
    unroll<U>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const int p = p0 + k;
      if (p >= n0) return;
      // this plane's j1 bands (uniform), loaded before the barrier so their latency hides behind it
      double t0[FG_W], tb[NM][WG];
      const double* p0r = P0 + (size_t)p * FG_W;
#pragma unroll
      for (int d = 0; d < FG_W; ++d) t0[d] = ((M0 >> d) & 1) ? __ldg(p0r + d) : 0.0;
#pragma unroll
      for (int m = 0; m < NMIX; ++m) {
        const double* b0 = B0 + ((size_t)r0s[m] * n0 + p) * FG_W + FG_K;
#pragma unroll
        for (int d = -RM; d <= RM; ++d) tb[m][d + RM] = __ldg(b0 + d);
      }
      issue_v(p + FG_K + FGA_D);
      issue_u(p + FGA_D);
      cp_commit();
      cp_wait<FGA_D>();
      __syncthreads();
      V[(k + 2 * FG_K) % FG_W] = (act && p + FG_K < n0) ? ring[((p + FG_K) & (FGA_NS - 1)) * SL + me] : zz();
      {
        double2 s1, gm[NM];
        exchange(p + RM, s1, gm);
        S1W[(k + RM) % WS] = s1;
#pragma unroll
        for (int m = 0; m < NM; ++m) GW[m][(k + 2 * RM) % WG] = gm[m];
      }
      if (!act) return;
      double2 acc = uring[(p & (FGA_NU - 1)) * tile + t];
      double2 acc2 = S1W[k % WS];
#pragma unroll
      for (int d = 0; d < FG_W; ++d)
        if ((M0 >> d) & 1) fma2(t0[d], V[(k + d) % FG_W], (d & 1) ? acc : acc2);  // plane p + d - K
#pragma unroll
      for (int m = 0; m < NMIX; ++m) {
#pragma unroll
        for (int d = -RM; d <= RM; ++d) fma2(tb[m][d + RM], GW[m][(k + d + RM) % WG], acc);
      }
      const double2 out = make_double2(acc.x + acc2.x, acc.y + acc2.y);
      y[(int64_t)p * S0 + off] = out;
      if (dotp) cdot_acc(V[(k + FG_K) % FG_W], out, dacc);
    });
  }
  cp_wait<0>();
  if (dotp) {
    dacc = block_sum2(dacc);
    if (t == 0) dotp[blockIdx.x] = dacc;
  }
}

// ---------------------------------------------------------------- v3 kernels
// The march loop is unrolled by FG3_U = 18 = lcm(9, 2, 3) and the smem rings
// have FG3_U (v / rows) and FG3_NU (u) slots, both dividing the unroll, so
// every ring slot, window slot and band offset is a compile-time constant;
// global addresses advance by pointer increments.  This removes most of the
// integer work per point that bounded the v2 kernels (ncu: IMAD ~ DFMA).
constexpr int FG3_U = 18;
constexpr int FG3_DA = 4;   // planes in flight, pass A
constexpr int FG3_NU = 6;   // u ring slots, pass A (divides FG3_U, >= FG3_DA + 2)
constexpr int FG3_DB = 8;   // rows in flight, pass B
constexpr unsigned FG_MASK_PM1 = 0x28;  // diagonals -1, +1

template <unsigned M2, unsigned M3>
__global__ void __launch_bounds__(128) k_fg_inner3(const double2* __restrict__ v, double2* __restrict__ u,
                                                   const double* __restrict__ P2, const double* __restrict__ P3,
                                                   int n2, int n3) {
  constexpr int U = FG3_U, D = FG3_DB, K = FG_K, W = FG_W;
  static_assert(U % W == 0 && U >= K + D + 2, "ring / unroll mismatch");
  extern __shared__ double2 ring[];  // [U][n3 + 2K], pads zero
  const int t = threadIdx.x;
  const int RW = n3 + 2 * K;
  const bool act = t < n3;
  const int64_t base = (int64_t)blockIdx.x * n2 * n3;
  const double2* vb = v + base;
  double2* dst = u + base + t;
  for (int i = t; i < U * 2 * K; i += blockDim.x) {
    int slot = i / (2 * K), k = i % (2 * K);
    ring[slot * RW + (k < K ? k : n3 + k)] = zz();
  }
  double p3[W];
#pragma unroll
  for (int d = 0; d < W; ++d) p3[d] = ((M3 >> d) & 1) && act ? __ldg(P3 + t * W + d) : 0.0;
  double2* myring = ring + K + t;
  auto issue = [&](int slot, const double2* src, bool ok) {
    if (act) cp_async16(myring + slot * RW, ok ? (const void*)src : (const void*)vb, ok ? 16 : 0);
  };
  const double2* src = vb + t;
#pragma unroll
  for (int r = 0; r <= K; ++r) issue(r, src + (int64_t)r * n3, r < n2);
  cp_commit();
#pragma unroll
  for (int r = K + 1; r < K + D; ++r) {
    issue(r, src + (int64_t)r * n3, r < n2);
    cp_commit();
  }
  cp_wait<D - 1>();
  __syncthreads();
  double2 V[W];  // slot (q + K) mod W holds row q
#pragma unroll
  for (int q = -K - 1; q <= K - 1; ++q) V[((q + K) % W + W) % W] = (act && q >= 0 && q < n2) ? myring[q * RW] : zz();
  src += (int64_t)(K + D) * n3;
  const double* p2r = P2;
  for (int i0 = 0; i0 < n2; i0 += U) {
    unroll<U>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const int i = i0 + k;
      if (i >= n2) return;
      double p2[W];
#pragma unroll
      for (int d = 0; d < W; ++d) p2[d] = ((M2 >> d) & 1) ? __ldg(p2r + d) : 0.0;
      p2r += W;
      issue((k + K + D) % U, src, i + K + D < n2);
      src += n3;
      cp_commit();
      cp_wait<D>();
      __syncthreads();
      V[(k + 2 * K) % W] = act ? myring[((k + K) % U) * RW] : zz();
      if (act) {
        const double2* row = myring + (k % U) * RW - K;  // row[d] = element j4 + d - K of row i
        double2 acc = zz(), acc2 = zz();
#pragma unroll
        for (int d = 0; d < W; ++d) {
          if ((M2 >> d) & 1) fma2(p2[d], V[(k + d) % W], acc);
          if (d != K && ((M3 >> d) & 1)) fma2(p3[d], row[d], acc2);
        }
        fma2(p3[K], V[(k + K) % W], acc2);
        *dst = make_double2(acc.x + acc2.x, acc.y + acc2.y);
      }
      dst += n3;
    });
  }
  cp_wait<0>();
}

template <int RM, int NMIX, unsigned M0, unsigned M1P, unsigned M1G, int C = FG_C>
__global__ void __launch_bounds__(512, 1) k_fg_outer3(const double2* __restrict__ v, const double2* __restrict__ u,
                                                      double2* __restrict__ y, const double* __restrict__ P0,
                                                      const double* __restrict__ P1, const double* __restrict__ G,
                                                      const double* __restrict__ B0, int n0, int n1, int64_t S0,
                                                      int64_t S1, int r0a, int r0b, double2* __restrict__ dotp) {
  constexpr int U = FG3_U, D = FG3_DA, NU = FG3_NU, K = FG_K, W = FG_W;
  constexpr int WS = RM + 1, WG = 2 * RM + 1;
  constexpr int NM = NMIX > 0 ? NMIX : 1;
  static_assert(U % W == 0 && U % WS == 0 && U % WG == 0 && U % NU == 0, "unroll must cover every ring");
  static_assert(U >= K + D + 2 && NU >= D + 2, "ring too short for the prefetch distance");
  extern __shared__ double2 sm[];
  const int tile = n1 * C;
  const int SL = (n1 + 2 * K) * C;
  const int t = threadIdx.x;
  const bool act = t < tile;
  const int j1 = t / C, e = t % C;
  const int64_t off = (int64_t)j1 * S1 + (int64_t)blockIdx.x * C + e;
  double2* myring = sm + (K + j1) * C + e;  // my element in ring slot 0
  double2* myu = sm + U * SL + t;              // my element in u-ring slot 0
  for (int i = t; i < U * 2 * K * C; i += blockDim.x) {
    int slot = i / (2 * K * C), k = i % (2 * K * C);
    sm[slot * SL + (k < K * C ? k : tile + k)] = zz();
  }
  double p1[W], g[NM][W];
#pragma unroll
  for (int d = 0; d < W; ++d) {
    p1[d] = act && ((M1P >> d) & 1) ? __ldg(P1 + j1 * W + d) : 0.0;
#pragma unroll
    for (int m = 0; m < NM; ++m)
      g[m][d] = act && m < NMIX && ((M1G >> d) & 1) ? __ldg(G + (size_t)m * FG_MAXN * W + j1 * W + d) : 0.0;
  }
  const double2* vs = v + off;
  const double2* us = u + off;
  auto issue_v = [&](int slot, const double2* src, bool ok) {
    if (act) cp_async16(myring + slot * SL, ok ? (const void*)src : (const void*)v, ok ? 16 : 0);
  };
  auto issue_u = [&](int slot, const double2* src, bool ok) {
    if (act) cp_async16(myu + slot * tile, ok ? (const void*)src : (const void*)u, ok ? 16 : 0);
  };
#pragma unroll
  for (int p = 0; p <= K; ++p) issue_v(p, vs + (int64_t)p * S0, p < n0);
  issue_u(0, us, 0 < n0);
  cp_commit();
#pragma unroll
  for (int k = 1; k < D; ++k) {
    issue_v(K + k, vs + (int64_t)(K + k) * S0, K + k < n0);
    issue_u(k, us + (int64_t)k * S0, k < n0);
    cp_commit();
  }
  cp_wait<D - 1>();
  __syncthreads();

  // j2 bands of the ring plane in `slot`: s1 = P_1 v(q), gm = G_m v(q)
  auto exchange = [&](int slot, bool valid, double2& s1, double2 (&gm)[NM]) {
    s1 = zz();
#pragma unroll
    for (int m = 0; m < NM; ++m) gm[m] = zz();
    if (!valid || !act) return;
    const double2* pl = myring + slot * SL;
#pragma unroll
    for (int d = 0; d < W; ++d) {
      constexpr unsigned any = M1P | M1G;
      if (!((any >> d) & 1)) continue;
      double2 x = pl[(d - K) * C];
      if ((M1P >> d) & 1) fma2(p1[d], x, s1);
      if ((M1G >> d) & 1)
#pragma unroll
        for (int m = 0; m < NMIX; ++m) fma2(g[m][d], x, gm[m]);
    }
  };

  double2 V[W], S1W[WS], GW[NM][WG];
#pragma unroll
  for (int q = -K - 1; q <= K - 1; ++q)
    V[((q + K) % W + W) % W] = (act && q >= 0 && q < n0) ? myring[q * SL] : zz();
#pragma unroll
  for (int q = -RM - 1; q <= RM - 1; ++q) {
    double2 s1, gm[NM];
    exchange(q < 0 ? 0 : q, q >= 0 && q < n0, s1, gm);
    if (q >= -1) S1W[((q % WS) + WS) % WS] = s1;
#pragma unroll
    for (int m = 0; m < NM; ++m) GW[m][(((q + RM) % WG) + WG) % WG] = gm[m];
  }
  double2 dacc = zz();
  const double2* vnext = vs + (int64_t)(K + D) * S0;
  const double2* unext = us + (int64_t)D * S0;
  double2* yp = y + off;
  const double* p0r = P0;
  const double* b0r[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) b0r[m] = B0 + (size_t)(m == 0 ? r0a : r0b) * n0 * W + K;
  for (int p0 = 0; p0 < n0; p0 += U) {
    unroll<U>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const int p = p0 + k;
      if (p >= n0) return;
      double t0[W], tb[NM][WG];
#pragma unroll
      for (int d = 0; d < W; ++d) t0[d] = ((M0 >> d) & 1) ? __ldg(p0r + d) : 0.0;
      p0r += W;
#pragma unroll
      for (int m = 0; m < NMIX; ++m) {
#pragma unroll
        for (int d = -RM; d <= RM; ++d) tb[m][d + RM] = __ldg(b0r[m] + d);
        b0r[m] += W;
      }
      issue_v((k + K + D) % U, vnext, p + K + D < n0);
      issue_u((k + D) % NU, unext, p + D < n0);
      vnext += S0;
      unext += S0;
      cp_commit();
      cp_wait<D>();
      __syncthreads();
      V[(k + 2 * K) % W] = (act && p + K < n0) ? myring[((k + K) % U) * SL] : zz();
      {
        double2 s1, gm[NM];
        exchange((k + RM) % U, p + RM < n0, s1, gm);
        S1W[(k + RM) % WS] = s1;
#pragma unroll
        for (int m = 0; m < NM; ++m) GW[m][(k + 2 * RM) % WG] = gm[m];
      }
      if (act) {
        double2 acc = myu[(k % NU) * tile];
        double2 acc2 = S1W[k % WS];
#pragma unroll
        for (int d = 0; d < W; ++d)
          if ((M0 >> d) & 1) fma2(t0[d], V[(k + d) % W], (d & 2) ? acc : acc2);
#pragma unroll
        for (int m = 0; m < NMIX; ++m)
#pragma unroll
          for (int d = -RM; d <= RM; ++d) fma2(tb[m][d + RM], GW[m][(k + d + RM) % WG], acc);
        const double2 out = make_double2(acc.x + acc2.x, acc.y + acc2.y);
        *yp = out;
        if (dotp) cdot_acc(V[(k + K) % W], out, dacc);
      }
      yp += S0;
    });
  }
  cp_wait<0>();
  if (dotp) {
    dacc = block_sum2(dacc);
    if (t == 0) dotp[blockIdx.x] = dacc;
  }
}

}  // namespace hp
