// Single-pass fused full-cube evaluator (cfg4 class): TMA-staged planes + register scatter ring.
//
// y = [c0 + sum_a P_a(X_a) + T_r0(X_0) G(X_1)] v on a 4-D box, ONE read of v and
// ONE write of y per coefficient (32 B algorithmic), instead of the two HBM
// passes of k_fg_inner2 / k_fg_outer3 (80 B).  (Axes 0-based here: axis 0 is
// DESIGN.md's j1.)
//
// Work decomposition.  The cross-section (j1, j2, j3) is cut into 8x4x16
// tiles (512 points); one persistent 256-thread CTA per SM takes tiles in a
// blocked order (ensure_tiles) and marches axis 0 through the n0 planes of its
// tile.  For every plane p one elected thread issues three TMA boxes into one
// of F1_S pipeline stages (40 KB): the tile with its +-4 rows along j1 (axis-1
// stencil and the G coupling) and +-4 columns along j3 (384 B rows: 64 B halo
// rows cost the TMA unit twice as much per byte), and the +-4 rows along j2.
// Boxes that run off the cube are zero-filled by the TMA unit -- exactly the
// truncation of the ladder operators at the box faces.  Halo rows of the
// neighbouring tiles were fetched from HBM by the CTAs that own them at about
// the same time, so they mostly come from L2.  Each stage has a "full"
// mbarrier (transaction bytes) and an "empty" one (one arrival per warp).
//
// Axis 0 is the march axis: instead of a 9-plane window of v, each thread
// keeps a 9-slot ring of PARTIAL OUTPUTS y(p-4 .. p+4) in registers.  When
// plane p arrives it scatters c = v(p) into y(p + d) with the band weight
// P_0(p + d, -d) (a per-plane row staged in smem, uniform over the CTA), adds
// the in-plane stencil of axes 1-3 and scatters g = G v(p) through T_r0(X_0);
// y(p-4) is then complete and is stored.  Ring slots are compile-time (march
// unrolled by 9).  With NP = 2 a thread owns rows j1 and j1 + 2 of the tile,
// whose axis-1 and coupling taps overlap (9 shared loads instead of 14).
//
// Bounds: the shared-memory port (TMA fills + stencil reads)
// and L2->SM traffic; the kernel runs at 62-66% of the smem-port floor.  A
// plane range [plo, phi) restricts the output planes (streamed host vectors,
// overlapped slab shards).  `exp` bits are timing instrumentation only
// (HP_FG_EXP: 1 skip halo boxes, 2 pipeline only, 8 compute only, 16-48 L2
// policy), all off in production.
#pragma once

#include <cuda.h>

// compiler fence between the stage's load groups (bounds registers held by in-flight loads)
#ifndef F1_FENCES
#define F1_FENCES 0
#endif
#if F1_FENCES
#define F1_FENCE() asm volatile("" ::: "memory")
#else
#define F1_FENCE() \
  do {             \
  } while (0)
#endif

#ifndef F1_TILE_J2
#define F1_TILE_J2 4
#endif

namespace hp {

// tile extents along axes 1, 2, 3 (T1 must be 8: the NP = 2 row pairing assumes it)
constexpr int F1_T1 = 8;
constexpr int F1_T2 = F1_TILE_J2;
constexpr int F1_T3 = 64 / F1_TILE_J2;
constexpr int F1_H = FG_K;              // halo (band radius)
constexpr int F1_S = 5;                 // pipeline stages
constexpr int F1_POINTS = F1_T1 * F1_T2 * F1_T3;  // tile points (512)
// stage layout in double2 units: A1 = [j1 +-4][j2][j3 +-4] (256 B rows: the j3 halos ride in the
// tile rows -- 64 B halo rows cost the TMA unit twice as much per byte) | j2 halos lo, hi
constexpr int F1_RW = F1_T3 + 2 * F1_H;                    // A1 row (j3) length
constexpr int F1_A1 = (F1_T1 + 2 * F1_H) * F1_T2 * F1_RW;  // [j1 +-4][j2][j3 +-4]
constexpr int F1_B2 = F1_T1 * F1_H * F1_T3;                // [j1][4][j3]
constexpr int F1_OFF_B2LO = F1_A1;
constexpr int F1_OFF_B2HI = F1_A1 + F1_B2;
constexpr int F1_STAGE = F1_A1 + 2 * F1_B2;  // 2560 double2 = 40 KB
constexpr unsigned F1_STAGE_BYTES = F1_STAGE * 16u;
constexpr int F1_WROW = 8;  // per-plane scatter weights (doubles), see k_fg_single
constexpr size_t F1_WOFF = (size_t)F1_S * F1_STAGE_BYTES;
constexpr size_t F1_BOFF = F1_WOFF + (size_t)FG_MAXN * F1_WROW * sizeof(double);
constexpr size_t F1_SMEM = F1_BOFF + 2 * F1_S * sizeof(uint64_t) + 8 * sizeof(int);

__device__ __forceinline__ unsigned f1_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void f1_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(f1_saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void f1_mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(f1_saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void f1_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(f1_saddr(bar)) : "memory");
}
__device__ __forceinline__ bool f1_mbar_try(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(f1_saddr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded wait: a TMA that never lands traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void f1_mbar_wait(uint64_t* bar, unsigned parity) {
  if (f1_mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!f1_mbar_try(bar, parity))
    if (clock64() - t0 > (1ll << 33)) __trap();
}
__device__ __forceinline__ void f1_tma4_hint(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                             uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3, %4, %5}], [%6], %7;\n" ::"r"(f1_saddr(dst)),
      "l"((unsigned long long)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(f1_saddr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t f1_policy(int hint) {
  uint64_t pol = 0;
  if (hint == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  else if (hint == 2)
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void f1_tma4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];\n" ::"r"(f1_saddr(dst)),
      "l"((unsigned long long)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(f1_saddr(bar))
      : "memory");
}


// NMIX = 0: no coupling term; NMIX = 1: one T_1(X_0) G(X_1) class with G on diagonals +-1.
// Single-axis bands on all four axes are even (diagonals 0, +-2, +-4).
//
// NP points per thread (512 / NP threads): with NP = 2 a thread owns tile rows j1 and j1 + 2
// (rows {0,2}, {1,3}, {4,6}, {5,7}), whose axis-1 and G taps overlap: 9 shared-memory loads
// serve both points' axis-1 + coupling + centre terms instead of 14, which is what bounds
// this kernel (the shared-memory pipe), at the price of a second register ring.
//
// Pipeline: thread 0 is the producer.  Stage s carries a "full" mbarrier (TMA
// transaction bytes) and an "empty" mbarrier (one arrival per warp once the
// warp has read the stage); the producer refills a stage only after its empty
// phase completes, so warps drift freely up to F1_S - 2 planes apart.
template <int NMIX, bool DOT, int NP>
__global__ void __launch_bounds__(F1_POINTS / NP, 1)
    k_fg_single(const __grid_constant__ CUtensorMap mA1, const __grid_constant__ CUtensorMap mB2,
                const double2* __restrict__ v, double2* __restrict__ y, const double* __restrict__ P,
                const double* __restrict__ G, const double* __restrict__ B0, const int* __restrict__ tiles,
                int ntiles, int n0, int n1, int n2, int n3, double2* __restrict__ dotp, int exp, int plo,
                int phi) {
  constexpr int NT = F1_POINTS / NP;
  extern __shared__ __align__(128) unsigned char f1_smem[];
  double2* stg = (double2*)f1_smem;
  double* W = (double*)(f1_smem + F1_WOFF);
  uint64_t* full = (uint64_t*)(f1_smem + F1_BOFF);
  uint64_t* empty = full + F1_S;
  const int tid = threadIdx.x, lane = tid & 31;
  const int j3 = tid % F1_T3, j2 = (tid / F1_T3) % F1_T2;
  const int j1 = NP == 1 ? (tid >> 6) : (((tid >> 6) >> 1) * 4 + ((tid >> 6) & 1));  // first row
  const double* P0 = P;
  const double* P1 = P + FG_MAXN * FG_W;
  const double* P2 = P + 2 * FG_MAXN * FG_W;
  const double* P3 = P + 3 * FG_MAXN * FG_W;
  if (tid == 0) {
    for (int s = 0; s < F1_S; ++s) {
      f1_mbar_init(&full[s], 1);
      f1_mbar_init(&empty[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // per-plane scatter weights: row p = {P0(p,0), P0(p+2,-2), P0(p-2,2), P0(p+4,-4), P0(p-4,4),
  //                                     B0(p+1,-1), B0(p-1,1), 0}
  for (int q = tid; q < n0; q += NT) {
    auto p0 = [&](int r, int e) { return (r >= 0 && r < n0) ? P0[r * FG_W + e + FG_K] : 0.0; };
    auto b0 = [&](int r, int e) { return (NMIX && r >= 0 && r < n0) ? B0[r * FG_W + e + FG_K] : 0.0; };
    double* w = W + q * F1_WROW;
    w[0] = p0(q, 0);
    w[1] = p0(q + 2, -2);
    w[2] = p0(q - 2, 2);
    w[3] = p0(q + 4, -4);
    w[4] = p0(q - 4, 4);
    w[5] = b0(q + 1, -1);
    w[6] = b0(q - 1, 1);
    w[7] = 0.0;
  }
  __syncthreads();

  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // output planes [plo, phi) (the whole cube, or one chunk of a streamed matvec): the march
  // consumes input planes [ps0, pe), the band radius around them
  const int ps0 = max(plo - F1_H, 0), pe = min(phi + F1_H, n0), nper = pe - ps0;
  const int nitems = my_tiles * nper;
  // producer state (thread 0 only; kept in shared memory so that it costs the consumer
  // threads no registers): next item, its tile / plane / stage / stage-use count, tile origin
  int* ps_ = (int*)(empty + F1_S);
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) ps_[i] = 0;
    ps_[2] = ps0;
  }
  auto issue_next = [&]() {
    int pk = ps_[0], pti = ps_[1], pp = ps_[2], ps = ps_[3], pu = ps_[4];
    if (pk >= nitems || (exp & 8)) return;
    if (pu > 0) f1_mbar_wait(&empty[ps], (unsigned)((pu - 1) & 1));
    if (pp == ps0) {
      const int code = __ldg(tiles + blockIdx.x + pti * gridDim.x);
      ps_[5] = (code & 1023) * F1_T1;
      ps_[6] = ((code >> 10) & 1023) * F1_T2;
      ps_[7] = (code >> 20) * F1_T3;
    }
    const int T1 = ps_[5], T2 = ps_[6], T3 = ps_[7];
    double2* dst = stg + (size_t)ps * F1_STAGE;
    uint64_t* bar = &full[ps];
    f1_mbar_expect(bar, (exp & 1) ? F1_A1 * 16u : F1_STAGE_BYTES);
    // L2 policy of the tile loads: explicit evict_normal (HP_FG_EXP bits 4-5: 1 evict_last,
    // 2 evict_normal, 3 evict_first, 0 no hint).  Measured on the Lanczos (dot) variant: no hint
    // 18.1 GB HBM reads / 4.30 ms, evict_normal 15.5 GB / 3.95 ms, evict_first 28.1 GB / 5.65 ms.
    const int hint = (exp >> 4) & 3 ? (exp >> 4) & 3 : 2;
    if (hint) {
      const uint64_t pol = f1_policy(hint);
      f1_tma4_hint(dst, &mA1, 2 * (T3 - F1_H), T2, T1 - F1_H, pp, bar, pol);
      f1_tma4_hint(dst + F1_OFF_B2LO, &mB2, 2 * T3, T2 - F1_H, T1, pp, bar, pol);
      f1_tma4_hint(dst + F1_OFF_B2HI, &mB2, 2 * T3, T2 + F1_T2, T1, pp, bar, pol);
    } else {
      f1_tma4(dst, &mA1, 2 * (T3 - F1_H), T2, T1 - F1_H, pp, bar);
      if (!(exp & 1)) {
        f1_tma4(dst + F1_OFF_B2LO, &mB2, 2 * T3, T2 - F1_H, T1, pp, bar);
        f1_tma4(dst + F1_OFF_B2HI, &mB2, 2 * T3, T2 + F1_T2, T1, pp, bar);
      }
    }
    ++pk;
    if (++pp == pe) {
      pp = ps0;
      ++pti;
    }
    if (++ps == F1_S) {
      ps = 0;
      ++pu;
    }
    ps_[0] = pk;
    ps_[1] = pti;
    ps_[2] = pp;
    ps_[3] = ps;
    ps_[4] = pu;
  };
  if (tid == 0)
    for (int k = 0; k < F1_S - 1; ++k) issue_next();

  constexpr int R1 = F1_T2 * F1_RW;  // A1 j1-row stride (double2)
  // centre of point 0 in A1; point 1 (NP = 2) sits two j1 rows below
  const int oc = (j1 + F1_H) * R1 + j2 * F1_RW + j3 + F1_H;
  // axis-2 taps: inside the tile they are A1 rows, outside they live in the j2 halo boxes
  // (computed on the fly so they hold no registers across the march)
  auto o2 = [&](int row, int d) {
    const int a = j2 + d;
    return a < 0 ? F1_OFF_B2LO + row * (F1_H * F1_T3) + (a + F1_H) * F1_T3 + j3
                 : (a >= F1_T2 ? F1_OFF_B2HI + row * (F1_H * F1_T3) + (a - F1_T2) * F1_T3 + j3
                              : (row + F1_H) * R1 + a * F1_RW + j3 + F1_H);
  };

  double2 dacc = make_double2(0.0, 0.0);
  int cs = 0, cu = 0;  // consumer stage / stage-use count
  const int64_t plane = (int64_t)n1 * n2 * n3;
  for (int ti = 0; ti < my_tiles; ++ti) {
    const int code = __ldg(tiles + blockIdx.x + ti * gridDim.x);
    const int J1 = (code & 1023) * F1_T1 + j1, J2 = ((code >> 10) & 1023) * F1_T2 + j2,
              J3 = (code >> 20) * F1_T3 + j3;
    const bool in0 = J1 < n1 && J2 < n2 && J3 < n3;
    const bool in1 = NP == 2 && J1 + 2 < n1 && J2 < n2 && J3 < n3;
    const int c1a = min(J1, FG_MAXN - 1), c1b = min(J1 + 2, FG_MAXN - 1);
    const int c2 = min(J2, FG_MAXN - 1), c3 = min(J3, FG_MAXN - 1);
    double w1a[4], w1b[4], w2[4], w3[4];
    double wga0 = 0.0, wga1 = 0.0, wgb0 = 0.0, wgb1 = 0.0;
    {
      const int ds[4] = {-4, -2, 2, 4};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        w1a[i] = __ldg(P1 + c1a * FG_W + ds[i] + FG_K);
        w1b[i] = NP == 2 ? __ldg(P1 + c1b * FG_W + ds[i] + FG_K) : 0.0;
        w2[i] = __ldg(P2 + c2 * FG_W + ds[i] + FG_K);
        w3[i] = __ldg(P3 + c3 * FG_W + ds[i] + FG_K);
      }
      if (NMIX) {
        wga0 = __ldg(G + c1a * FG_W + FG_K - 1);
        wga1 = __ldg(G + c1a * FG_W + FG_K + 1);
        if (NP == 2) {
          wgb0 = __ldg(G + c1b * FG_W + FG_K - 1);
          wgb1 = __ldg(G + c1b * FG_W + FG_K + 1);
        }
      }
    }
    const double c23 = __ldg(P2 + c2 * FG_W + FG_K) + __ldg(P3 + c3 * FG_W + FG_K);
    const double cca = __ldg(P1 + c1a * FG_W + FG_K) + c23;
    const double ccb = NP == 2 ? __ldg(P1 + c1b * FG_W + FG_K) + c23 : 0.0;
    const int col = (J1 * n2 + J2) * n3 + J3;  // n1 n2 n3 <= 2^24
    const int colb = col + 2 * n2 * n3;

    double2 RA[9], RB[NP == 2 ? 9 : 1];
#pragma unroll
    for (int i = 0; i < 9; ++i) RA[i] = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < (NP == 2 ? 9 : 1); ++i) RB[i] = make_double2(0.0, 0.0);

    for (int pb = ps0 - ps0 % 9; pb < phi + F1_H; pb += 9) {  // ring slot = plane mod 9
      unroll<9>([&](auto UU) {
        constexpr int U = decltype(UU)::value;
        const int p = pb + U;
        if (p < ps0 || p >= phi + F1_H) return;
        // DOT: v at the plane completed by this step is re-read from L2 (it was staged 4 planes
        // ago); the load is issued here, ahead of the stage wait and the step's work, so its
        // latency is hidden (the wait's memory clobber keeps the compiler from sinking it)
        double2 vqa = make_double2(0.0, 0.0), vqb = make_double2(0.0, 0.0);
        if (DOT && p - F1_H >= plo) {
          const int64_t base = (int64_t)(p - F1_H) * plane;
          if (in0) vqa = __ldg(v + base + col);
          if (NP == 2 && in1) vqb = __ldg(v + base + colb);
        }
        if (p < pe) {
          if (tid == 0) issue_next();
          if (!(exp & 8)) f1_mbar_wait(&full[cs], (unsigned)(cu & 1));  // bit 3: compute only
          if (exp & 2) {  // timing experiment: pipeline only
            __syncwarp();
            if (lane == 0) f1_mbar_arrive(&empty[cs]);
            if (++cs == F1_S) {
              cs = 0;
              ++cu;
            }
            return;
          }
          const double2* st = stg + (size_t)cs * F1_STAGE;
          // load groups separated by compiler fences: bounds the registers held by in-flight
          // shared loads (rings + weights already take most of the budget)
          double2 ua, ub = make_double2(0.0, 0.0), ga = make_double2(0.0, 0.0), gb = make_double2(0.0, 0.0);
          double2 ca, cb = make_double2(0.0, 0.0);
          {
            const double2 m4 = st[oc - 4 * R1], m2 = st[oc - 2 * R1], z0 = st[oc], p2 = st[oc + 2 * R1],
                          p4 = st[oc + 4 * R1];
            ca = z0;
            ua = make_double2(cca * z0.x, cca * z0.y);
            fma2(w1a[0], m4, ua);
            fma2(w1a[1], m2, ua);
            fma2(w1a[2], p2, ua);
            fma2(w1a[3], p4, ua);
            if (NP == 2) {
              const double2 p6 = st[oc + 6 * R1];
              cb = p2;
              ub = make_double2(ccb * p2.x, ccb * p2.y);
              fma2(w1b[0], m2, ub);
              fma2(w1b[1], z0, ub);
              fma2(w1b[2], p4, ub);
              fma2(w1b[3], p6, ub);
            }
          }
          if (NMIX) {
            F1_FENCE();
            const double2 m1 = st[oc - R1], p1 = st[oc + R1];
            ga = make_double2(wga0 * m1.x, wga0 * m1.y);
            fma2(wga1, p1, ga);
            if (NP == 2) {
              const double2 p3 = st[oc + 3 * R1];
              gb = make_double2(wgb0 * p1.x, wgb0 * p1.y);
              fma2(wgb1, p3, gb);
            }
          }
          F1_FENCE();
          {
            const double2 a = st[o2(j1, -4)], b = st[o2(j1, -2)], c = st[o2(j1, 2)], d = st[o2(j1, 4)];
            fma2(w2[0], a, ua);
            fma2(w2[1], b, ua);
            fma2(w2[2], c, ua);
            fma2(w2[3], d, ua);
          }
          F1_FENCE();
          {
            const double2 a = st[oc - 4], b = st[oc - 2], c = st[oc + 2], d = st[oc + 4];
            fma2(w3[0], a, ua);
            fma2(w3[1], b, ua);
            fma2(w3[2], c, ua);
            fma2(w3[3], d, ua);
          }
          if (NP == 2) {
            F1_FENCE();
            {
              const double2 a = st[o2(j1 + 2, -4)], b = st[o2(j1 + 2, -2)], c = st[o2(j1 + 2, 2)],
                            d = st[o2(j1 + 2, 4)];
              fma2(w2[0], a, ub);
              fma2(w2[1], b, ub);
              fma2(w2[2], c, ub);
              fma2(w2[3], d, ub);
            }
            F1_FENCE();
            {
              const int ob = oc + 2 * R1;
              const double2 a = st[ob - 4], b = st[ob - 2], c = st[ob + 2], d = st[ob + 4];
              fma2(w3[0], a, ub);
              fma2(w3[1], b, ub);
              fma2(w3[2], c, ub);
              fma2(w3[3], d, ub);
            }
          }
          __syncwarp();
          if (lane == 0) f1_mbar_arrive(&empty[cs]);
          if (++cs == F1_S) {
            cs = 0;
            ++cu;
          }
          const double2 wa = *(const double2*)(W + p * F1_WROW);
          const double2 wb = *(const double2*)(W + p * F1_WROW + 2);
          const double2 wc = *(const double2*)(W + p * F1_WROW + 4);
          const double2 wd = *(const double2*)(W + p * F1_WROW + 6);
          auto scatter = [&](double2* R, double2 c, double2 u, double2 g) {
            fma2(wa.x, c, u);
            R[U].x += u.x;
            R[U].y += u.y;
            fma2(wa.y, c, R[(U + 2) % 9]);
            fma2(wb.x, c, R[(U + 7) % 9]);
            fma2(wb.y, c, R[(U + 4) % 9]);
            fma2(wc.x, c, R[(U + 5) % 9]);
            if (NMIX) {
              fma2(wc.y, g, R[(U + 1) % 9]);
              fma2(wd.x, g, R[(U + 8) % 9]);
            }
          };
          scatter(RA, ca, ua, ga);
          if (NP == 2) scatter(RB, cb, ub, gb);
        }
        // y(p - 4) has received its last contribution
        constexpr int SQ = (U + 5) % 9;
        if (p - F1_H >= plo) {
          const int64_t base = (int64_t)(p - F1_H) * plane;
          if (in0) {
            __stcs(y + base + col, RA[SQ]);  // streaming store: keep L2 for v halos
            if (DOT) cdot_acc(vqa, RA[SQ], dacc);
          }
          if (NP == 2 && in1) {
            __stcs(y + base + colb, RB[SQ % (NP == 2 ? 9 : 1)]);
            if (DOT) cdot_acc(vqb, RB[SQ % (NP == 2 ? 9 : 1)], dacc);
          }
        }
        RA[SQ] = make_double2(0.0, 0.0);
        if (NP == 2) RB[SQ % (NP == 2 ? 9 : 1)] = make_double2(0.0, 0.0);
      });
    }
  }
  if (DOT) {
    dacc = block_sum2(dacc);
    if (tid == 0) dotp[blockIdx.x] = dacc;
  }
}

}  // namespace hp
