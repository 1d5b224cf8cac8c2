// Single-pass fused full-cube evaluator, quad variant: 1024-point tiles, four points per thread.
//
// Same operator and march as k_fg_single (hp_fg1.cuh):
//   y = [c0 + sum_a P_a(X_a) + T_r0(X_0) G(X_1)] v  on a 4-D box (axes 0-based, axis 0 = j1),
// one read of v and one write of y per coefficient.  MIX selects the couplings: bit 0 the
// (0,1) class above; bit 1 adds c02 T_1(X_0) T_1(X_2) (x1 x3: its axis-2 taps b +- 1 come from
// A1 / the B2 boxes and join the same march-axis scatter); bit 2 adds c03 T_1(X_0) T_1(X_3) (x1 x4:
// taps c +- 1 of the same rows, same scatter); bit 3 adds c13 T_1(X_1) T_1(X_3)
// (x2 x4: an in-plane term whose corner taps (a +- 1, c +- 1) lie inside box A1).  The other
// pairs' corners are not staged.  What changes against k_fg_single is the per-SM working set:
//
// * Tiles are 8 x 8 x 16 (axes 1, 2, 3) = 1024 points instead of 512, so the halo staged per
//   plane falls from 5x to 4x the tile (64 B/coef of TMA fills instead of 80): box A1 =
//   [axis 1 +-4][axis 2][axis 3 +-4] (384 B rows), boxes B2 = the +-4 rows along axis 2.
// * Each thread owns the 2 x 2 points {a, a+2} x {b, b+2} (axes 1, 2) of one axis-3 column.
//   Even-offset taps of the pair overlap along both axes: 42 shared-memory loads serve the four
//   points' 84 taps (10.5 per point instead of 12.5).
// * The march-axis ring of partial outputs has 8 slots instead of 9: at step p the slot of
//   y(p-4) receives its last term (from v(p)), is stored, and is reused for y(p+4).  Every
//   in-plane term goes straight into a ring slot (no per-point accumulators): 128 of the 255
//   registers are the ring.
// * Band weights are read per plane from shared tables indexed by global coordinate (a warp
//   owns one axis-1 row pair: broadcast loads); holding them in registers spills.
// * 3 stages of 64 KB; the LAST warp to release a stage refills it (no producer warp, no warp
//   waiting to act as producer).
// * Global addresses advance by one plane per step (64-bit index math per step cost ~40
//   registers and spilled the first version).
//
// Measured: 2.26-2.45 ms per cfg4 matvec (0.54-0.58 of the HBM roofline), bound
// by the TMA fills (64 B/coef, 1.55 ms alone) and the LSU shared wavefronts (80% busy), which
// overlap only in part at 8 warps/SM.
#pragma once

#ifndef Q_FENCES
#define Q_FENCES 0  // compiler fences between load phases: off measured 0.8% faster (2.416 vs 2.434 ms)
#endif
// (the instantiation with all three couplings keeps them: its live ranges spill otherwise)
#define Q_FENCE()                                                   \
  do {                                                              \
    if (Q_FENCES || MIX == 11 || MIX == 15) asm volatile("" ::: "memory"); \
  } while (0)

namespace hp {

constexpr int Q_T1 = 8, Q_T2 = 8, Q_T3 = 16;
constexpr int Q_MAXN = 128;  // largest side the weight tables are sized for (larger cubes: k_fg_single)
constexpr int Q_H = FG_K;
constexpr int Q_NT = 256;
constexpr int Q_POINTS = Q_T1 * Q_T2 * Q_T3;
constexpr int Q_RW = Q_T3 + 2 * Q_H;                 // A1 row (axis 3) length: 24
constexpr int Q_R1 = Q_T2 * Q_RW;                    // A1 axis-1 stride: 192
constexpr int Q_A1 = (Q_T1 + 2 * Q_H) * Q_R1;        // 3072
constexpr int Q_B2R1 = Q_H * Q_T3;                   // B2 axis-1 stride: 64
constexpr int Q_B2 = Q_T1 * Q_B2R1;                  // 512
constexpr int Q_OFF_LO = Q_A1, Q_OFF_HI = Q_A1 + Q_B2;
constexpr int Q_STAGE = Q_A1 + 2 * Q_B2;             // 4096 double2 = 64 KB
constexpr unsigned Q_STAGE_BYTES = Q_STAGE * 16u;
#ifndef Q_STAGES
#define Q_STAGES 3
#endif
constexpr int Q_S = Q_STAGES;
constexpr size_t Q_WOFF = (size_t)Q_S * Q_STAGE_BYTES;
constexpr int Q_T1W = 8;  // doubles per axis-1 weight row
constexpr size_t Q_TOFF = Q_WOFF + (size_t)Q_MAXN * F1_WROW * sizeof(double);
constexpr size_t Q_T2OFF = Q_TOFF + (size_t)(Q_MAXN + 8) * Q_T1W * sizeof(double);
constexpr size_t Q_T3OFF = Q_T2OFF + (size_t)(Q_MAXN + 8) * Q_T1W * sizeof(double);
constexpr int Q_T3N = Q_MAXN;  // axis-3 table: [Q_T3ROWS][Q_T3N], transposed (16 lanes read 128 B); J3 < ceil(n3 / 16) * 16 <= Q_MAXN
constexpr int Q_T3ROWS = 9;  // P3(-4, -2, 2, 4, 0), B_{3,1}(-1, +1) (MIX & 8), c03 B_{3,1}(-1, +1) (MIX & 4)
constexpr size_t Q_BOFF = Q_T3OFF + (size_t)Q_T3ROWS * Q_T3N * sizeof(double);
constexpr int Q_TC = 64;  // tile codes cached in shared memory
constexpr size_t Q_SMEM = Q_BOFF + 2 * Q_S * sizeof(uint64_t) + (Q_S + Q_TC) * sizeof(int);

__device__ __forceinline__ void q_prefetch4(const CUtensorMap* m, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];\n" ::"l"(
                   (unsigned long long)m),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

template <int MIX, bool DOT>
__global__ void __launch_bounds__(Q_NT, 1)
    k_fg_quad(const __grid_constant__ CUtensorMap mA1, const __grid_constant__ CUtensorMap mB2,
              const double2* __restrict__ v, double2* __restrict__ y, const double* __restrict__ P,
              const double* __restrict__ G, const double* __restrict__ B0, const int* __restrict__ tiles, int ntiles,
              int n0, int n1, int n2, int n3, double2* __restrict__ dotp, int exp, int plo, int phi) {
  extern __shared__ __align__(128) unsigned char q_smem[];
  double2* stg = (double2*)q_smem;
  double* W = (double*)(q_smem + Q_WOFF);
  double* T1w = (double*)(q_smem + Q_TOFF);
  double* T2w = (double*)(q_smem + Q_T2OFF);
  double* T3w = (double*)(q_smem + Q_T3OFF);
  uint64_t* full = (uint64_t*)(q_smem + Q_BOFF);
  uint64_t* empty = full + Q_S;
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = tid & 15, bq = (tid >> 4) & 3, aq = tid >> 6;
  const int a = (aq >> 1) * 4 + (aq & 1), b = (bq >> 1) * 4 + (bq & 1);
  const double* P0 = P;
  const double* P1 = P + FG_MAXN * FG_W;
  const double* P2 = P + 2 * FG_MAXN * FG_W;
  const double* P3 = P + 3 * FG_MAXN * FG_W;
  if (tid == 0) {
    for (int s = 0; s < Q_S; ++s) {
      f1_mbar_init(&full[s], 1);
      f1_mbar_init(&empty[s], Q_NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // per-plane scatter weights (k_fg_single's row layout):
  // {P0(p,0), P0(p+2,-2), P0(p-2,2), P0(p+4,-4), P0(p-4,4), B0(p+1,-1), B0(p-1,1), 0}
  for (int q = tid; q < n0; q += Q_NT) {
    auto p0 = [&](int r, int e) { return (r >= 0 && r < n0) ? P0[r * FG_W + e + FG_K] : 0.0; };
    auto b0 = [&](int r, int e) { return (MIX && r >= 0 && r < n0) ? B0[r * FG_W + e + FG_K] : 0.0; };
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
  // axis-1 rows r = 0 .. n1+7: {P1(r,-4), P1(r,-2), P1(r,2), P1(r,4), G(r,-1), G(r,+1), P1(r,0), 0}
  // (rows past the cube are zeros: their points are never stored)
  for (int r = tid; r < n1 + 8; r += Q_NT) {
    double* w = T1w + r * Q_T1W;
    const bool ok = r < n1;
    w[0] = ok ? P1[r * FG_W + FG_K - 4] : 0.0;
    w[1] = ok ? P1[r * FG_W + FG_K - 2] : 0.0;
    w[2] = ok ? P1[r * FG_W + FG_K + 2] : 0.0;
    w[3] = ok ? P1[r * FG_W + FG_K + 4] : 0.0;
    w[4] = ok && (MIX & 1) ? G[r * FG_W + FG_K - 1] : 0.0;
    w[5] = ok && (MIX & 1) ? G[r * FG_W + FG_K + 1] : 0.0;
    w[6] = ok ? P1[r * FG_W + FG_K] : 0.0;
    // c13 B_{1,1}(r, -1): the band is symmetric, so B_{1,1}(r, +1) is the entry of row r + 1
    w[7] = ok && (MIX & 8) ? G[(size_t)3 * FG_MAXN * FG_W + r * FG_W + FG_K - 1] : 0.0;
  }
  // axis-2 rows: {P2(r,-4), P2(r,-2), P2(r,2), P2(r,4), P2(r,0), 0, 0, 0}
  for (int r = tid; r < n2 + 8; r += Q_NT) {
    double* w = T2w + r * Q_T1W;
    const bool ok = r < n2;
    w[0] = ok ? P2[r * FG_W + FG_K - 4] : 0.0;
    w[1] = ok ? P2[r * FG_W + FG_K - 2] : 0.0;
    w[2] = ok ? P2[r * FG_W + FG_K + 2] : 0.0;
    w[3] = ok ? P2[r * FG_W + FG_K + 4] : 0.0;
    w[4] = ok ? P2[r * FG_W + FG_K] : 0.0;
    w[5] = ok && (MIX & 2) ? G[(size_t)2 * FG_MAXN * FG_W + r * FG_W + FG_K - 1] : 0.0;  // c02 B_{2,1}(r, -1)
    w[6] = ok && (MIX & 2) ? G[(size_t)2 * FG_MAXN * FG_W + r * FG_W + FG_K + 1] : 0.0;  // c02 B_{2,1}(r, +1)
    w[7] = 0.0;
  }
  // axis-3 columns, transposed: T3w[i][r] = P3(r, -4, -2, 2, 4, 0 for i = 0..4)
  for (int r = tid; r < Q_T3N; r += Q_NT) {
    const bool ok = r < n3;
    T3w[0 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K - 4] : 0.0;
    T3w[1 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K - 2] : 0.0;
    T3w[2 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K + 2] : 0.0;
    T3w[3 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K + 4] : 0.0;
    T3w[4 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K] : 0.0;
    if (MIX & 8) {
      T3w[5 * Q_T3N + r] = ok ? G[(size_t)4 * FG_MAXN * FG_W + r * FG_W + FG_K - 1] : 0.0;  // B_{3,1}(r, -1)
      T3w[6 * Q_T3N + r] = ok ? G[(size_t)4 * FG_MAXN * FG_W + r * FG_W + FG_K + 1] : 0.0;  // B_{3,1}(r, +1)
    }
    if (MIX & 4) {
      T3w[7 * Q_T3N + r] = ok ? G[(size_t)5 * FG_MAXN * FG_W + r * FG_W + FG_K - 1] : 0.0;  // c03 B_{3,1}(r, -1)
      T3w[8 * Q_T3N + r] = ok ? G[(size_t)5 * FG_MAXN * FG_W + r * FG_W + FG_K + 1] : 0.0;  // c03 B_{3,1}(r, +1)
    }
  }
  __syncthreads();

  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int ps0 = max(plo - Q_H, 0), pe = min(phi + Q_H, n0), nper = pe - ps0;
  const int nitems = my_tiles * nper;
  // Stage refills: the LAST warp to release a stage (smem counter per stage) refills it with the
  // item S steps later, so no warp ever waits for the slowest one before issuing, and a fill is
  // issued the moment its stage is free.  Item k = (tile k / nper, plane ps0 + k % nper).
  int* cnt = (int*)(empty + Q_S);  // [Q_S] release counters
  int* tcode = cnt + Q_S;          // this CTA's tile codes (first Q_TC)
  for (int i = tid; i < Q_S; i += Q_NT) cnt[i] = 0;
  for (int i = tid; i < min(my_tiles, Q_TC); i += Q_NT) tcode[i] = __ldg(tiles + blockIdx.x + i * gridDim.x);
  __syncthreads();
  auto issue_item = [&](int k, int ps) {
    const int ti = k / nper, pp = ps0 + k % nper;
    const int code = ti < Q_TC ? tcode[ti] : __ldg(tiles + blockIdx.x + ti * gridDim.x);
    const int T1 = (code & 1023) * Q_T1, T2 = ((code >> 10) & 1023) * Q_T2, T3 = (code >> 20) * Q_T3;
    double2* dst = stg + (size_t)ps * Q_STAGE;
    uint64_t* bar = &full[ps];
    f1_mbar_expect(bar, Q_STAGE_BYTES);
    const uint64_t pol = f1_policy((exp >> 4) & 3 ? (exp >> 4) & 3 : 2);  // HP_FG_EXP bits 4-5: L2 policy experiments
    f1_tma4_hint(dst, &mA1, 2 * (T3 - Q_H), T2, T1 - Q_H, pp, bar, pol);
    f1_tma4_hint(dst + Q_OFF_LO, &mB2, 2 * T3, T2 - Q_H, T1, pp, bar, pol);
    f1_tma4_hint(dst + Q_OFF_HI, &mB2, 2 * T3, T2 + Q_T2, T1, pp, bar, pol);
  };
  if (tid == 0)
    for (int k = 0; k < min(Q_S, nitems); ++k) issue_item(k, k);
  int kk = 0;  // this thread's item index

  // centre of point (a, b) in A1; the other three points are +2 rows along axes 1 / 2
  const int oc = (a + Q_H) * Q_R1 + b * Q_RW + c + Q_H;
  // axis-2 taps of row r (= a or a + 2) at axis-2 index t: A1 inside the tile, B2 boxes outside
  auto o2 = [&](int r, int t) {
    return t < 0 ? Q_OFF_LO + r * Q_B2R1 + (t + Q_H) * Q_T3 + c
                 : (t >= Q_T2 ? Q_OFF_HI + r * Q_B2R1 + (t - Q_T2) * Q_T3 + c : (r + Q_H) * Q_R1 + t * Q_RW + c + Q_H);
  };
  // per thread, fixed over the whole run: t = b-4, b-2, b+4, b+6 for rows a and a+2
  // (row a + 2 = row a + 2 axis-1 strides: 2 Q_R1 in A1, 2 Q_B2R1 in the B2 boxes)
  int o2a[4];
  {
    const int ts[4] = {b - 4, b - 2, b + 4, b + 6};
#pragma unroll
    for (int i = 0; i < 4; ++i) o2a[i] = o2(a, ts[i]);
  }
  const int dlo = b < Q_H ? 2 * Q_B2R1 : 2 * Q_R1;  // taps b-4, b-2: B2 box iff b < 4
  const int dhi = b < Q_H ? 2 * Q_R1 : 2 * Q_B2R1;  // taps b+4, b+6: B2 box iff b >= 4

  double2 dacc = make_double2(0.0, 0.0), dT = make_double2(0.0, 0.0), dL = make_double2(0.0, 0.0);
  int cs = 0, cu = 0;
  const int64_t plane = (int64_t)n1 * n2 * n3;
  const int s1 = 2 * n2 * n3, s2 = 2 * n3;  // global offsets of the +2 rows along axes 1, 2
  for (int ti = 0; ti < my_tiles; ++ti) {
    const int code = __ldg(tiles + blockIdx.x + ti * gridDim.x);
    const int J1 = (code & 1023) * Q_T1 + a, J2 = ((code >> 10) & 1023) * Q_T2 + b, J3 = (code >> 20) * Q_T3 + c;
    const bool okc = J3 < n3;
    const bool in00 = okc && J1 < n1 && J2 < n2, in10 = okc && J1 + 2 < n1 && J2 < n2;
    const bool in01 = okc && J1 < n1 && J2 + 2 < n2, in11 = okc && J1 + 2 < n1 && J2 + 2 < n2;
    const int col = (J1 * n2 + J2) * n3 + J3;  // n1 n2 n3 <= 2^24
    // y at plane p - 4 of the step about to run, advanced by one plane per step
    double2* yq = y + col + (int64_t)(ps0 - Q_H) * plane;

    // ring of partial outputs, slot = plane mod 8; index [point][slot], points 00, 10, 01, 11
    double2 R[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) R[k][i] = make_double2(0.0, 0.0);

    for (int pb = ps0 - ps0 % 8; pb < phi + Q_H; pb += 8) {
      unroll<8>([&](auto UU) {
        constexpr int U = decltype(UU)::value;
        const int p = pb + U;
        if (p < ps0 || p >= phi + Q_H) return;
        constexpr int SQ = (U + 4) & 7;  // slot of y(p-4), then of y(p+4)
        // DOT (row p of v^H A v, by the symmetry of A): L_p = conj(v_p) . [y_p so far: the terms
        // of planes < p] before this plane's own terms, T_p = conj(v_p) . [y_p after them]; then
        // v^H A v = sum (T_p + conj(L_p)) -- no re-read of v (the former scheme re-read the
        // completed plane from L2: +4.3 GB of L2->SM traffic per matvec)
        const bool dotrow = DOT && p >= plo && p < phi;
        if (p < pe) {
          f1_mbar_wait(&full[cs], (unsigned)(cu & 1));
          const double2* st = stg + (size_t)cs * Q_STAGE;
          HP_DCHECK(oc - 4 * Q_R1 >= 0 && oc + 6 * Q_R1 + 2 * Q_RW + 4 < Q_A1 && o2a[0] + dlo >= 0 &&
                    o2a[3] + dhi < Q_STAGE && cs < Q_S);
          // march-axis weights of plane p (uniform over the CTA)
#define Q3(i) A3[(i) * Q_T3N]
#define QW(i) W[p * F1_WROW + (i)]
#define QT1A(i) T1w[J1 * Q_T1W + (i)]
#define QT1B(i) T1w[J1 * Q_T1W + 2 * Q_T1W + (i)]
#define QT2A(i) T2w[J2 * Q_T1W + (i)]
#define QT2B(i) T2w[J2 * Q_T1W + 2 * Q_T1W + (i)]
          const double2 wa = make_double2(QW(0), QW(1));
          const double2 wc = make_double2(QW(4), QW(5));
          const double wd = QW(6);
          // axis-1 weights of rows a, a+2 (uniform over the warp: broadcast loads, no registers
          // held across the march)
          const double* A3 = T3w + J3;
          double2 z[4];
          // phase A: axis-1 band + diagonal at axis-2 rows b and b + 2, into the slots of y(p)
          {
            const double2 wa01 = make_double2(QT1A(0), QT1A(1)), wa23 = make_double2(QT1A(2), QT1A(3));
            const double2 wb01 = make_double2(QT1B(0), QT1B(1)), wb23 = make_double2(QT1B(2), QT1B(3));
            const double dg = Q3(4) + wa.x;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int o = oc + h * 2 * Q_RW;
              const double2 m4 = st[o - 4 * Q_R1], m2 = st[o - 2 * Q_R1], z0 = st[o], p2 = st[o + 2 * Q_R1],
                            p4 = st[o + 4 * Q_R1], p6 = st[o + 6 * Q_R1];
              const double d2 = (h ? QT2B(4) : QT2A(4)) + dg;
              const double da = QT1A(6) + d2, db = QT1B(6) + d2;
              double2& ra = R[2 * h][U];
              double2& rb = R[2 * h + 1][U];
              z[2 * h] = z0;
              z[2 * h + 1] = p2;
              if (dotrow) {
                cdot_acc(z0, ra, dL);
                cdot_acc(p2, rb, dL);
              }
              fma2(da, z0, ra);
              fma2(wa01.x, m4, ra);
              fma2(wa01.y, m2, ra);
              fma2(wa23.x, p2, ra);
              fma2(wa23.y, p4, ra);
              fma2(db, p2, rb);
              fma2(wb01.x, m2, rb);
              fma2(wb01.y, z0, rb);
              fma2(wb23.x, p4, rb);
              fma2(wb23.y, p6, rb);
            }
          }
          // phase E (needs only the centres): march-axis band terms of the centres; y(p-4) receives its last term
          {
            const double2 wb = make_double2(QW(2), QW(3));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              fma2(wa.y, z[k], R[k][(U + 2) & 7]);
              fma2(wb.x, z[k], R[k][(U + 6) & 7]);
              fma2(wc.x, z[k], R[k][SQ]);
            }
            if (p - Q_H >= plo) {
              double2* yb = yq;
              HP_DCHECK(yb - y >= 0 && yb - y + (in11 ? s1 + s2 : 0) < (int64_t)n0 * plane);
              if (in00) __stcs(yb, R[0][SQ]);
              if (in10) __stcs(yb + s1, R[1][SQ]);
              if (in01) __stcs(yb + s2, R[2][SQ]);
              if (in11) __stcs(yb + s1 + s2, R[3][SQ]);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) R[k][SQ] = make_double2(wb.y * z[k].x, wb.y * z[k].y);  // y(p+4)
          }
          Q_FENCE();
          // axis-2 taps: point b uses t = b-4, b-2, (b+2 = centre of point b+2), b+4;
          //              point b+2 uses b-2, (b = centre of point b), b+4, b+6
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int el = h ? dlo : 0, eh = h ? dhi : 0;
            const double2 t0 = st[o2a[0] + el], t1 = st[o2a[1] + el], t2 = st[o2a[2] + eh], t3 = st[o2a[3] + eh];
            const double2 wa01 = make_double2(QT2A(0), QT2A(1)), wa23 = make_double2(QT2A(2), QT2A(3));
            const double2 wb01 = make_double2(QT2B(0), QT2B(1)), wb23 = make_double2(QT2B(2), QT2B(3));
            double2& ra = R[h][U];      // (row a or a+2, b)
            double2& rb = R[h + 2][U];  // (row a or a+2, b+2)
            fma2(wa01.x, t0, ra);
            fma2(wa01.y, t1, ra);
            fma2(wa23.x, z[h + 2], ra);
            fma2(wa23.y, t2, ra);
            fma2(wb01.x, t1, rb);
            fma2(wb01.y, z[h], rb);
            fma2(wb23.x, t2, rb);
            fma2(wb23.y, t3, rb);
            Q_FENCE();
          }
          // phase C: couplings through the march axis, g = [G(X_1) + c02 T_1(X_2) + c03 T_1(X_3)] v at rows a, a+2,
          // scattered through T_r0(X_0) to y(p +- 1)
          if (MIX & 7) {
            const double2 ga = make_double2(QT1A(4), QT1A(5)), gb = make_double2(QT1B(4), QT1B(5));
            const double2 wcd = make_double2(wc.y, wd);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int o = oc + h * 2 * Q_RW;
              double2* Ra = R[2 * h];
              double2* Rb = R[2 * h + 1];
              double2 g = make_double2(0.0, 0.0), g2 = make_double2(0.0, 0.0);
              if (MIX & 1) {
                const double2 m1 = st[o - Q_R1], p1 = st[o + Q_R1], p3 = st[o + 3 * Q_R1];
                g = make_double2(ga.x * m1.x, ga.x * m1.y);
                fma2(ga.y, p1, g);
                g2 = make_double2(gb.x * p1.x, gb.x * p1.y);
                fma2(gb.y, p3, g2);
              }
              if ((MIX & 3) == 3) Q_FENCE();
              if (MIX & 2) {
                // axis-2 taps t = (b + 2h) -+ 1 of rows a and a + 2 (A1 inside the tile, B2 boxes outside)
                const int tm = b + 2 * h - 1, tp = b + 2 * h + 1;
                const int om = o2(a, tm), op = o2(a, tp);
                const int dm = (tm < 0 || tm >= Q_T2) ? 2 * Q_B2R1 : 2 * Q_R1, dp = (tp < 0 || tp >= Q_T2) ? 2 * Q_B2R1 : 2 * Q_R1;
                const double cm = h ? QT2B(5) : QT2A(5), cp = h ? QT2B(6) : QT2A(6);
                fma2(cm, st[om], g);
                fma2(cp, st[op], g);
                fma2(cm, st[om + dm], g2);
                fma2(cp, st[op + dp], g2);
              }
              if (MIX & 4) {  // axis-3 taps c -+ 1 of the same rows
                const double em = Q3(7), ep = Q3(8);
                fma2(em, st[o - 1], g);
                fma2(ep, st[o + 1], g);
                fma2(em, st[o + 2 * Q_R1 - 1], g2);
                fma2(ep, st[o + 2 * Q_R1 + 1], g2);
              }
              fma2(wcd.x, g, Ra[(U + 1) & 7]);
              fma2(wcd.y, g, Ra[(U + 7) & 7]);
              fma2(wcd.x, g2, Rb[(U + 1) & 7]);
              fma2(wcd.y, g2, Rb[(U + 7) & 7]);
            }
            Q_FENCE();
          }
          // in-plane coupling c13 T_1(X_1) T_1(X_3) v: corner taps (a +- 1, c +- 1) and (a + 1 | a + 3, c +- 1)
          if (MIX & 8) {
            const double w3m = Q3(5), w3p = Q3(6);
            const double s0 = QT1A(7), s1 = T1w[(J1 + 1) * Q_T1W + 7], s2 = QT1B(7), s3 = T1w[(J1 + 3) * Q_T1W + 7];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int o = oc + h * 2 * Q_RW;
              double2 hm = make_double2(0.0, 0.0), h1 = hm, h3 = hm;
              fma2(w3m, st[o - Q_R1 - 1], hm);
              fma2(w3p, st[o - Q_R1 + 1], hm);
              fma2(w3m, st[o + Q_R1 - 1], h1);
              fma2(w3p, st[o + Q_R1 + 1], h1);
              fma2(w3m, st[o + 3 * Q_R1 - 1], h3);
              fma2(w3p, st[o + 3 * Q_R1 + 1], h3);
              fma2(s0, hm, R[2 * h][U]);
              fma2(s1, h1, R[2 * h][U]);
              fma2(s2, h1, R[2 * h + 1][U]);
              fma2(s3, h3, R[2 * h + 1][U]);
            }
            Q_FENCE();
          }
          // axis-3 taps (contiguous rows of A1)
          const double w3[4] = {Q3(0), Q3(1), Q3(2), Q3(3)};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int o = oc + (k & 1) * 2 * Q_R1 + (k >> 1) * 2 * Q_RW;
            const double2 t0 = st[o - 4], t1 = st[o - 2], t2 = st[o + 2], t3 = st[o + 4];
            fma2(w3[0], t0, R[k][U]);
            fma2(w3[1], t1, R[k][U]);
            fma2(w3[2], t2, R[k][U]);
            fma2(w3[3], t3, R[k][U]);
            if (k & 1) Q_FENCE();
          }
          if (dotrow) {  // T_p: y_p now holds every term of planes <= p; centres re-read from the stage
#pragma unroll
            for (int k = 0; k < 4; ++k) cdot_acc(st[oc + (k & 1) * 2 * Q_R1 + (k >> 1) * 2 * Q_RW], R[k][U], dT);
          }
          __syncwarp();
          if (lane == 0) {
            f1_mbar_arrive(&empty[cs]);
            if (atomicAdd(&cnt[cs], 1) == Q_NT / 32 - 1) {
              cnt[cs] = 0;
              f1_mbar_wait(&empty[cs], (unsigned)(cu & 1));  // all releases landed (acquire)
              if (kk + Q_S < nitems) issue_item(kk + Q_S, cs);
            }
          }
          ++kk;
          if (++cs == Q_S) {
            cs = 0;
            ++cu;
          }
        } else {
          // past the last input plane: y(p-4) only drains
          if (p - Q_H >= plo) {
            double2* yb = yq;
            if (in00) __stcs(yb, R[0][SQ]);
            if (in10) __stcs(yb + s1, R[1][SQ]);
            if (in01) __stcs(yb + s2, R[2][SQ]);
            if (in11) __stcs(yb + s1 + s2, R[3][SQ]);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) R[k][SQ] = make_double2(0.0, 0.0);
        }
        yq += plane;
      });
    }
  }
  if (DOT) {
    dacc = block_sum2(make_double2(dT.x + dL.x, dT.y - dL.y));
    if (tid == 0) dotp[blockIdx.x] = dacc;
  }
}

}  // namespace hp
