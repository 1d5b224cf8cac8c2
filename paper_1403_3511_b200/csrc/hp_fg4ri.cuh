// Single-pass fused full-cube evaluator, split-component variant of k_fg_quad (hp_fg4.cuh).
//
// The operator is real, so the real and imaginary parts of y = W v are two independent
// real problems.  k_fg_quad_ri gives each thread ONE component of its four points: lanes
// 2c and 2c+1 of a warp hold the real and imaginary parts of j4 column c (16 columns).  Per thread the march-axis ring is 4 points x 8 slots x 8 B =
// 64 registers instead of 128, so a CTA runs 512 threads (16 warps per SM instead of 8) on the
// same 8 x 8 x 16 tile, TMA boxes and 3-stage pipeline -- twice the warps to hide the
// shared-memory latency that bounds k_fg_quad.  Shared loads become 64-bit: a warp reads the
// 256 contiguous bytes of 16 complex values (2 wavefronts), the same bytes per point as before.
// A warp owns one (j2 pair, j3 pair), so the j1-row, j2 and j3 band weights are warp-uniform
// and come from the constant bank (k_fg_qtables); the j4 weights from a shared table.
#pragma once

namespace hp {

constexpr int QR_NT = 512;
constexpr size_t QR_T3OFF = (size_t)Q_S * Q_STAGE_BYTES;
constexpr size_t QR_BOFF = QR_T3OFF + (size_t)5 * Q_T3N * sizeof(double);
constexpr size_t QR_SMEM = QR_BOFF + 2 * Q_S * sizeof(uint64_t) + (Q_S + Q_TC) * sizeof(int);

template <int NMIX, bool DOT>
__global__ void __launch_bounds__(QR_NT, 1)
    k_fg_quad_ri(const __grid_constant__ CUtensorMap mA1, const __grid_constant__ CUtensorMap mB2,
                 const double2* __restrict__ v, double2* __restrict__ y, const double* __restrict__ P,
                 const int* __restrict__ tiles, int ntiles, int n0, int n1, int n2, int n3,
                 double2* __restrict__ dotp, int plo, int phi) {
  extern __shared__ __align__(128) unsigned char qr_smem[];
  double2* stg = (double2*)qr_smem;
  double* T3w = (double*)(qr_smem + QR_T3OFF);
  uint64_t* full = (uint64_t*)(qr_smem + QR_BOFF);
  uint64_t* empty = full + Q_S;
  int* cnt = (int*)(empty + Q_S);
  int* tcode = cnt + Q_S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // lanes 2c, 2c+1: real / imaginary part of column c (a half-warp reads 128 contiguous bytes)
  const int c = lane >> 1, comp = lane & 1;
  const int aq = warp >> 2, bq = warp & 3;
  const int a = (aq >> 1) * 4 + (aq & 1), b = (bq >> 1) * 4 + (bq & 1);
  const double* P3 = P + 3 * FG_MAXN * FG_W;
  constexpr int NW = QR_NT / 32;
  if (tid == 0) {
    for (int s = 0; s < Q_S; ++s) {
      f1_mbar_init(&full[s], 1);
      f1_mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int r = tid; r < Q_T3N; r += QR_NT) {
    const bool ok = r < n3;
    T3w[0 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K - 4] : 0.0;
    T3w[1 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K - 2] : 0.0;
    T3w[2 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K + 2] : 0.0;
    T3w[3 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K + 4] : 0.0;
    T3w[4 * Q_T3N + r] = ok ? P3[r * FG_W + FG_K] : 0.0;
  }
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int ps0 = max(plo - Q_H, 0), pe = min(phi + Q_H, n0), nper = pe - ps0;
  const int nitems = my_tiles * nper;
  for (int i = tid; i < Q_S; i += QR_NT) cnt[i] = 0;
  for (int i = tid; i < min(my_tiles, Q_TC); i += QR_NT) tcode[i] = __ldg(tiles + blockIdx.x + i * gridDim.x);
  __syncthreads();
  auto issue_item = [&](int k, int ps) {
    const int ti = k / nper, pp = ps0 + k % nper;
    const int code = ti < Q_TC ? tcode[ti] : __ldg(tiles + blockIdx.x + ti * gridDim.x);
    const int T1 = (code & 1023) * Q_T1, T2 = ((code >> 10) & 1023) * Q_T2, T3 = (code >> 20) * Q_T3;
    double2* dst = stg + (size_t)ps * Q_STAGE;
    uint64_t* bar = &full[ps];
    f1_mbar_expect(bar, Q_STAGE_BYTES);
    const uint64_t pol = f1_policy(2);
    f1_tma4_hint(dst, &mA1, 2 * (T3 - Q_H), T2, T1 - Q_H, pp, bar, pol);
    f1_tma4_hint(dst + Q_OFF_LO, &mB2, 2 * T3, T2 - Q_H, T1, pp, bar, pol);
    f1_tma4_hint(dst + Q_OFF_HI, &mB2, 2 * T3, T2 + Q_T2, T1, pp, bar, pol);
  };
  if (tid == 0)
    for (int k = 0; k < min(Q_S, nitems); ++k) issue_item(k, k);
  int kk = 0;

  // stage offsets in complex (double2) units, as in k_fg_quad; loads read component `comp`
  const int oc = (a + Q_H) * Q_R1 + b * Q_RW + c + Q_H;
  auto o2 = [&](int r, int t) {
    return t < 0 ? Q_OFF_LO + r * Q_B2R1 + (t + Q_H) * Q_T3 + c
                 : (t >= Q_T2 ? Q_OFF_HI + r * Q_B2R1 + (t - Q_T2) * Q_T3 + c : (r + Q_H) * Q_R1 + t * Q_RW + c + Q_H);
  };
  int o2a[4];
  {
    const int ts[4] = {b - 4, b - 2, b + 4, b + 6};
#pragma unroll
    for (int i = 0; i < 4; ++i) o2a[i] = o2(a, ts[i]);
  }
  const int dlo = b < Q_H ? 2 * Q_B2R1 : 2 * Q_R1;
  const int dhi = b < Q_H ? 2 * Q_R1 : 2 * Q_B2R1;

  double dr = 0.0, di = 0.0;  // DOT partials: Re and Im of v^H y
  int cs = 0, cu = 0;
  const int64_t plane = (int64_t)n1 * n2 * n3;
  const int s1 = 2 * n2 * n3, s2 = 2 * n3;  // +2 rows along axes 1, 2 (complex units)
  for (int ti = 0; ti < my_tiles; ++ti) {
    const int code = __ldg(tiles + blockIdx.x + ti * gridDim.x);
    const int J1 = (code & 1023) * Q_T1 + a, J2 = ((code >> 10) & 1023) * Q_T2 + b, J3 = (code >> 20) * Q_T3 + c;
    const bool okc = J3 < n3;
    const bool in00 = okc && J1 < n1 && J2 < n2, in10 = okc && J1 + 2 < n1 && J2 < n2;
    const bool in01 = okc && J1 < n1 && J2 + 2 < n2, in11 = okc && J1 + 2 < n1 && J2 + 2 < n2;
    const int col = (J1 * n2 + J2) * n3 + J3;
    // component pointers of y (and v) at plane p - 4 of the next step
    double* yq = (double*)y + 2 * ((int64_t)col + (int64_t)(ps0 - Q_H) * plane) + comp;
    const double* vqp = (const double*)v + 2 * ((int64_t)col + (int64_t)(ps0 - Q_H) * plane) + comp;
    const double* A3 = T3w + J3;

    double R[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) R[k][i] = 0.0;

    for (int pb = ps0 - ps0 % 8; pb < phi + Q_H; pb += 8) {
      unroll<8>([&](auto UU) {
        constexpr int U = decltype(UU)::value;
        const int p = pb + U;
        if (p < ps0 || p >= phi + Q_H) return;
        constexpr int SQ = (U + 4) & 7;
        double vq[4] = {0.0, 0.0, 0.0, 0.0};
        if (DOT && p - Q_H >= plo) {
          if (in00) vq[0] = __ldg(vqp);
          if (in10) vq[1] = __ldg(vqp + 2 * s1);
          if (in01) vq[2] = __ldg(vqp + 2 * s2);
          if (in11) vq[3] = __ldg(vqp + 2 * (s1 + s2));
        }
        auto finish = [&]() {  // y(p-4) is complete: store, dot, free the slot
          if (p - Q_H >= plo) {
            if (in00) __stcs(yq, R[0][SQ]);
            if (in10) __stcs(yq + 2 * s1, R[1][SQ]);
            if (in01) __stcs(yq + 2 * s2, R[2][SQ]);
            if (in11) __stcs(yq + 2 * (s1 + s2), R[3][SQ]);
            if (DOT) {
              // v^H y = sum vr yr + vi yi + i (vr yi - vi yr): the partner lane (other component of
              // the same point) supplies the cross term
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const double yo = __shfl_xor_sync(0xffffffffu, R[k][SQ], 1);
                dr = fma(vq[k], R[k][SQ], dr);
                di = fma(comp ? -vq[k] : vq[k], yo, di);
              }
            }
          }
        };
        if (p < pe) {
          f1_mbar_wait(&full[cs], (unsigned)(cu & 1));
          const double* st = (const double*)(stg + (size_t)cs * Q_STAGE) + comp;
          auto ld = [&](int idx) { return st[2 * idx]; };
          const double* W = q_cw + Q_CW_W + p * 8;
          const double* T1a = q_cw + Q_CW_T1 + J1 * 8;
          const double* T1b = T1a + 16;
          const double* T2a = q_cw + Q_CW_T2 + J2 * 8;
          const double* T2b = T2a + 16;
          const double w0 = W[0];
          double z[4];
          // phase A: axis-1 band + diagonal at axis-2 rows b, b + 2
          {
            const double dg = A3[4 * Q_T3N] + w0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int o = oc + h * 2 * Q_RW;
              const double m4 = ld(o - 4 * Q_R1), m2 = ld(o - 2 * Q_R1), z0 = ld(o), p2 = ld(o + 2 * Q_R1),
                           p4 = ld(o + 4 * Q_R1), p6 = ld(o + 6 * Q_R1);
              const double d2 = (h ? T2b[4] : T2a[4]) + dg;
              double& ra = R[2 * h][U];
              double& rb = R[2 * h + 1][U];
              z[2 * h] = z0;
              z[2 * h + 1] = p2;
              ra = fma(T1a[6] + d2, z0, ra);
              ra = fma(T1a[0], m4, ra);
              ra = fma(T1a[1], m2, ra);
              ra = fma(T1a[2], p2, ra);
              ra = fma(T1a[3], p4, ra);
              rb = fma(T1b[6] + d2, p2, rb);
              rb = fma(T1b[0], m2, rb);
              rb = fma(T1b[1], z0, rb);
              rb = fma(T1b[2], p4, rb);
              rb = fma(T1b[3], p6, rb);
            }
          }
          Q_FENCE();
          // phase E: march-axis band terms of the centres; y(p-4) receives its last term
          {
            const double w1 = W[1], w2 = W[2], w3 = W[3], w4 = W[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              R[k][(U + 2) & 7] = fma(w1, z[k], R[k][(U + 2) & 7]);
              R[k][(U + 6) & 7] = fma(w2, z[k], R[k][(U + 6) & 7]);
              R[k][SQ] = fma(w4, z[k], R[k][SQ]);
            }
            finish();
#pragma unroll
            for (int k = 0; k < 4; ++k) R[k][SQ] = w3 * z[k];  // y(p+4)
          }
          Q_FENCE();
          // phase B: axis-2 taps
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int el = h ? dlo : 0, eh = h ? dhi : 0;
            const double t0 = ld(o2a[0] + el), t1 = ld(o2a[1] + el), t2 = ld(o2a[2] + eh), t3 = ld(o2a[3] + eh);
            double& ra = R[h][U];
            double& rb = R[h + 2][U];
            ra = fma(T2a[0], t0, ra);
            ra = fma(T2a[1], t1, ra);
            ra = fma(T2a[2], z[h + 2], ra);
            ra = fma(T2a[3], t2, ra);
            rb = fma(T2b[0], t1, rb);
            rb = fma(T2b[1], z[h], rb);
            rb = fma(T2b[2], t2, rb);
            rb = fma(T2b[3], t3, rb);
            Q_FENCE();
          }
          // phase C: coupling g = G(X_1) v at rows a, a+2 -> y(p +- 1) through T_r0(X_0)
          if (NMIX) {
            const double wc = W[5], wd = W[6];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int o = oc + h * 2 * Q_RW;
              const double m1 = ld(o - Q_R1), p1 = ld(o + Q_R1), p3 = ld(o + 3 * Q_R1);
              double* Ra = R[2 * h];
              double* Rb = R[2 * h + 1];
              double g = T1a[4] * m1;
              g = fma(T1a[5], p1, g);
              Ra[(U + 1) & 7] = fma(wc, g, Ra[(U + 1) & 7]);
              Ra[(U + 7) & 7] = fma(wd, g, Ra[(U + 7) & 7]);
              g = T1b[4] * p1;
              g = fma(T1b[5], p3, g);
              Rb[(U + 1) & 7] = fma(wc, g, Rb[(U + 1) & 7]);
              Rb[(U + 7) & 7] = fma(wd, g, Rb[(U + 7) & 7]);
            }
            Q_FENCE();
          }
          // phase D: axis-3 taps (contiguous rows of A1)
          {
            const double w30 = A3[0], w31 = A3[Q_T3N], w32 = A3[2 * Q_T3N], w33 = A3[3 * Q_T3N];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int o = oc + (k & 1) * 2 * Q_R1 + (k >> 1) * 2 * Q_RW;
              const double t0 = ld(o - 4), t1 = ld(o - 2), t2 = ld(o + 2), t3 = ld(o + 4);
              R[k][U] = fma(w30, t0, R[k][U]);
              R[k][U] = fma(w31, t1, R[k][U]);
              R[k][U] = fma(w32, t2, R[k][U]);
              R[k][U] = fma(w33, t3, R[k][U]);
              if (k & 1) Q_FENCE();
            }
          }
          __syncwarp();
          if (lane == 0) {
            f1_mbar_arrive(&empty[cs]);
            if (atomicAdd(&cnt[cs], 1) == NW - 1) {
              cnt[cs] = 0;
              f1_mbar_wait(&empty[cs], (unsigned)(cu & 1));
              if (kk + Q_S < nitems) issue_item(kk + Q_S, cs);
            }
          }
          ++kk;
          if (++cs == Q_S) {
            cs = 0;
            ++cu;
          }
        } else {
          finish();
#pragma unroll
          for (int k = 0; k < 4; ++k) R[k][SQ] = 0.0;
        }
        yq += 2 * plane;
        if (DOT) vqp += 2 * plane;
      });
    }
  }
  if (DOT) {
    double2 dacc = block_sum2(make_double2(dr, di));
    if (tid == 0) dotp[blockIdx.x] = dacc;
  }
}

}  // namespace hp
