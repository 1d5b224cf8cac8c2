// Fused full-cube evaluator for N = 4 boxes (cfg4 class).
//
// The even-band class (all single-axis bands even, at most one r1 = 1 coupling on axes
// (1, 2)) runs the single-pass TMA kernel of hp_fg1.cuh (one HBM read of v, one write of y);
// every other covered structure runs the two-pass split below.  Both share the band tables
// and the term classification.
//
// On a full cube (or a j1-slab of one) the restricted ladders of different
// axes commute, so every term alpha_r prod_l T_{r_l}(X_l/L) is a tensor
// product of 1-D banded matrices B_{l,k} = T_k(J_l/L), J_l the truncated
// Jacobi (ladder) matrix of axis l.  Those bands are tabulated once per set
// (host matrix recurrence, identical polynomial to the reference's vector
// recurrence fast_apply.py:69-92) and the whole surrogate becomes a
// stencil with per-index weights.  A 4-D radius-4 stencil does not fit on
// chip in one pass (a 9-plane window of a 128^3 plane is 302 MB), so the
// operator is split by axes:
//
//   pass B  (inner axes 3,4; one CTA per (j1, j2) block, marching j3 with a
//            9-row register window per j4 column, j4 neighbours via a smem row)
//              u = [c0 + P_3(X_3) + P_4(X_4) (+ their oscillator levels)] v
//   pass A  (outer axes 1,2; one CTA per 4-element inner chunk, all j2 rows,
//            marching j1 with a 9-plane register window; planes stream through
//            a cp.async (LDGSTS) ring, the j2 neighbours are read from the ring)
//              y = u + P_1(X_1) v + P_2(X_2) v + sum_m T_{r0_m}(X_1/L) G_m(X_2) v
//
// HBM traffic: 32 B/coefficient (pass B) + 48 B/coefficient (pass A).
// Supported term structure (else the generic program of hp_apply.cu runs):
// constant, single-axis terms on any axis (degree <= 4), and mixed terms on
// axes (1, 2) only with r1 <= 2 (at most two distinct r1).  This is cfg4.
#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "hp_common.cuh"
#include "hp_program.h"

namespace hp {

constexpr int FG_K = 4;
constexpr int FG_W = 2 * FG_K + 1;
constexpr int FG_C = 4;  // inner chunk of pass A (4 x 16 B = 64 B per row segment)
constexpr int FG_D = 4;  // cp.async prefetch distance (planes)
constexpr int FG_MAXN = 256;
constexpr int FG_DOTP = 512;  // per-CTA dot partials (grid <= SM count) at the end of the workspace
constexpr size_t FG_DOTP_BYTES = FG_DOTP * 16;

// ---------------------------------------------------------------- host tables

// B_k = T_k(J/L) for k = 0..FG_K as bands [k][i][FG_W] (diagonal d at index d + FG_K)
static void basis_1d(int n, int joff, double L, double* out) {
  std::vector<double> X(n * 3, 0.0);  // tridiagonal: [i][0] = below, [i][2] = above
  for (int i = 0; i < n; ++i) {
    double j = (double)(joff + i);
    X[i * 3 + 0] = i > 0 ? std::sqrt(j / 2.0) / L : 0.0;
    X[i * 3 + 2] = i < n - 1 ? std::sqrt((j + 1.0) / 2.0) / L : 0.0;
  }
  // dense banded storage of T_{k-1}, T_k
  std::vector<double> Tm(n * FG_W, 0.0), Tc(n * FG_W, 0.0), Tn(n * FG_W, 0.0);
  auto at = [&](std::vector<double>& T, int i, int c) -> double& { return T[i * FG_W + (c - i) + FG_K]; };
  for (int i = 0; i < n; ++i) at(Tm, i, i) = 1.0;
  for (int i = 0; i < n; ++i) {
    if (i > 0) at(Tc, i, i - 1) = X[i * 3 + 0];
    if (i < n - 1) at(Tc, i, i + 1) = X[i * 3 + 2];
  }
  std::copy(Tm.begin(), Tm.end(), out);
  std::copy(Tc.begin(), Tc.end(), out + (size_t)n * FG_W);
  for (int k = 2; k <= FG_K; ++k) {
    std::fill(Tn.begin(), Tn.end(), 0.0);
    for (int i = 0; i < n; ++i)
      for (int c = std::max(0, i - k); c <= std::min(n - 1, i + k); ++c) {
        double s = 0.0;
        if (i > 0 && std::abs(c - (i - 1)) <= k - 1) s += X[i * 3 + 0] * at(Tc, i - 1, c);
        if (i < n - 1 && std::abs(c - (i + 1)) <= k - 1) s += X[i * 3 + 2] * at(Tc, i + 1, c);
        double prev = std::abs(c - i) <= k - 2 ? at(Tm, i, c) : 0.0;
        at(Tn, i, c) = 2.0 * s - prev;
      }
    std::copy(Tn.begin(), Tn.end(), out + (size_t)k * n * FG_W);
    std::swap(Tm, Tc);
    std::swap(Tc, Tn);
  }
}

// basis layout on the device: axis a at offset a * (FG_K+1) * FG_MAXN * FG_W
static size_t basis_axis_stride() { return (size_t)(FG_K + 1) * FG_MAXN * FG_W; }

static hp_status ensure_basis(const hp_set_s* s, double L, cudaStream_t st) {
  std::lock_guard<std::mutex> g(s->fg_mtx);
  if (s->fg_basis && s->fg_L == L) return HP_OK;
  std::vector<double> host(4 * basis_axis_stride(), 0.0);
  for (int a = 0; a < 4; ++a) basis_1d(s->side[a], a == 0 ? s->lo : 0, L, host.data() + a * basis_axis_stride());
  if (!s->fg_basis) HP_CUDA(cudaMalloc(&s->fg_basis, host.size() * sizeof(double)));
  HP_CUDA(cudaMemcpyAsync(s->fg_basis, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  HP_CUDA(cudaStreamSynchronize(st));
  s->fg_L = L;
  return HP_OK;
}

// ---------------------------------------------------------------- term classification

struct FgPlan {
  bool ok = false;
  double c0 = 0.0;
  double ws[4][FG_K + 1] = {{0}};  // single-axis weights per axis/degree
  int nmix = 0;
  int r0[2] = {0, 0};              // axis-1 degree of each mixed class
  double wm[2][FG_K + 1] = {{0}};  // axis-2 weights per mixed class
  int rm = 0;
  unsigned mask[4] = {0, 0, 0, 0}; // nonzero diagonals of the combined single-axis bands
  unsigned maskG = 0;              // nonzero diagonals of the mixed-term axis-2 bands G_m
  bool twopass = true;             // the cube fits the two-pass kernels' chunking (single pass: any side)
  // further T_1 (x) T_1 couplings of the single-pass quad kernel: axes (0,2), (0,3) and (1,3), i.e.
  // x1 x3, x1 x4 and x2 x4 (the halo boxes of k_fg_quad hold their taps; (1,2) and (2,3) corners are not staged)
  double cx02 = 0.0, cx03 = 0.0, cx13 = 0.0;
  bool extra() const { return cx02 != 0.0 || cx03 != 0.0 || cx13 != 0.0; }
  // the other T_1 (x) T_1 pairs -- (1,2), (2,3) -- are added by a second, streaming pass
  // (k_fg_pairs) after the fused evaluator: y += sum c_ab T_1(X_a) T_1(X_b) v
  double cres[3] = {0.0, 0.0, 0.0};
  bool residual() const { return cres[0] != 0.0 || cres[1] != 0.0 || cres[2] != 0.0; }
};
constexpr int FG_RES_A[3] = {-1, 1, 2}, FG_RES_B[3] = {-1, 2, 3};  // (slot 0: x1 x4, now inside k_fg_quad)

static FgPlan classify(const hp_set_s* s, const std::vector<Term>& terms, int dtype, int64_t batch, int flags) {
  FgPlan P;
  if (!s->boxed || s->dim != 4 || dtype != HP_C128 || batch < 1) return P;
  for (int a = 0; a < 4; ++a) if (s->side[a] > FG_MAXN) return P;
  if (((int64_t)s->side[2] * s->side[3]) % FG_C != 0 || s->side[1] * FG_C > 512 || s->side[3] > 128)
    P.twopass = false;
  for (const Term& t : terms) {
    int act[4], na = 0;
    for (int a = 0; a < 4; ++a) if (t.r[a] > 0) act[na++] = a;
    if (na == 0) { P.c0 += t.alpha; continue; }
    if (na == 1) {
      if (t.r[act[0]] > FG_K) return P;
      P.ws[act[0]][t.r[act[0]]] += t.alpha;
      continue;
    }
    if (na == 2 && act[0] == 0 && act[1] == 1 && t.r[0] <= 2 && t.r[1] <= FG_K) {
      int m = -1;
      for (int i = 0; i < P.nmix; ++i) if (P.r0[i] == t.r[0]) m = i;
      if (m < 0) {
        if (P.nmix == 2) return P;
        m = P.nmix++;
        P.r0[m] = t.r[0];
      }
      P.wm[m][t.r[1]] += t.alpha;
      continue;
    }
    if (na == 2 && t.r[act[0]] == 1 && t.r[act[1]] == 1 && act[0] == 0 && act[1] == 2) {
      P.cx02 += t.alpha;
      continue;
    }
    if (na == 2 && t.r[act[0]] == 1 && t.r[act[1]] == 1 && act[0] == 1 && act[1] == 3) {
      P.cx13 += t.alpha;
      continue;
    }
    if (na == 2 && t.r[act[0]] == 1 && t.r[act[1]] == 1 && act[0] == 0 && act[1] == 3) {
      P.cx03 += t.alpha;
      continue;
    }
    if (na == 2 && t.r[act[0]] == 1 && t.r[act[1]] == 1) {
      bool placed = false;
      for (int i = 0; i < 3; ++i)
        if (act[0] == FG_RES_A[i] && act[1] == FG_RES_B[i]) {
          P.cres[i] += t.alpha;
          placed = true;
        }
      if (placed) continue;
    }
    return P;
  }
  for (int m = 0; m < P.nmix; ++m) P.rm = std::max(P.rm, P.r0[m]);
  for (int a = 0; a < 4; ++a) {
    unsigned mk = 1u << FG_K;  // centre always (c0 / oscillator levels)
    for (int k = 1; k <= FG_K; ++k)
      if (P.ws[a][k] != 0.0)
        for (int d = -k; d <= k; d += 2) mk |= 1u << (d + FG_K);
    P.mask[a] = mk;
  }
  if (P.nmix) {
    unsigned mk = 0;
    for (int m = 0; m < P.nmix; ++m)
      for (int k = 0; k <= FG_K; ++k)
        if (P.wm[m][k] != 0.0) for (int d = -k; d <= k; d += 2) mk |= 1u << (d + FG_K);
    P.maskG = mk;
  }
  P.ok = true;
  (void)flags;
  return P;
}

// ---------------------------------------------------------------- kernels

// band tables in the workspace: P[4] | G[2] (mixed classes of axes (0,1)) | cx02 B_{2,1} | cx13 B_{1,1} | B_{3,1} | cx03 B_{3,1}
constexpr int FG_NTAB = 10;

struct CombineArgs {
  double ws[4][FG_K + 1];
  double wm[2][FG_K + 1];
  double cx02, cx03, cx13;
  int side[4];
  int joff0;
  int nmix;
  double c0;
  int osc;
  double sq;  // harmonic part q: q * sum_l x_l^2 folded into the single-axis bands (fast_apply.py:229-245)
};

// combined bands: P[a][j][d] = sum_k ws[a][k] B_{a,k}[j][d] (+ levels, + c0 on axis 4)
//                 G[m][j][d] = sum_k wm[m][k] B_{2,k}[j][d]
__global__ void k_fg_combine(const double* __restrict__ basis, double* __restrict__ P, double* __restrict__ G,
                             CombineArgs A) {
  const size_t bs = (size_t)(FG_K + 1) * FG_MAXN * FG_W;
  int total = FG_NTAB * FG_MAXN * FG_W;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    int tab = idx / (FG_MAXN * FG_W);
    int rem = idx % (FG_MAXN * FG_W);
    int j = rem / FG_W, d = rem % FG_W;
    if (tab < 4) {
      int a = tab;
      int n = A.side[a];
      double acc = 0.0;
      if (j < n) {
        for (int k = 1; k <= FG_K; ++k)
          if (A.ws[a][k] != 0.0) acc += A.ws[a][k] * basis[a * bs + ((size_t)k * n + j) * FG_W + d];
        if (d == FG_K) {
          acc += A.ws[a][0];
          if (A.osc) acc += (double)(j + (a == 0 ? A.joff0 : 0)) + 0.5;
          if (a == 3) acc += A.c0;
        }
        if (A.sq != 0.0) {
          const double jg = (double)(j + (a == 0 ? A.joff0 : 0));
          if (d == FG_K) acc += A.sq * (jg + 0.5);
          if (d == FG_K + 2 && j + 2 < n) acc += A.sq * 0.5 * sqrt((jg + 1.0) * (jg + 2.0));
          if (d == FG_K - 2 && j >= 2) acc += A.sq * 0.5 * sqrt(jg * (jg - 1.0));
        }
      }
      P[(size_t)a * FG_MAXN * FG_W + rem] = acc;
    } else if (tab < 6) {
      int m = tab - 4;
      int n = A.side[1];
      double acc = 0.0;
      if (m < A.nmix && j < n)
        for (int k = 0; k <= FG_K; ++k)
          if (A.wm[m][k] != 0.0) acc += A.wm[m][k] * basis[1 * bs + ((size_t)k * n + j) * FG_W + d];
      G[(size_t)m * FG_MAXN * FG_W + rem] = acc;
    } else {
      // T_1 bands of the further couplings: cx02 B_{2,1}, cx13 B_{1,1}, B_{3,1}
      const int a = tab == 6 ? 2 : (tab == 7 ? 1 : 3);
      const double c = tab == 6 ? A.cx02 : (tab == 7 ? A.cx13 : (tab == 8 ? 1.0 : A.cx03));
      const int n = A.side[a];
      G[(size_t)(tab - 4) * FG_MAXN * FG_W + rem] = (j < n && c != 0.0) ? c * basis[a * bs + ((size_t)1 * n + j) * FG_W + d] : 0.0;
    }
  }
}

}  // namespace hp

#include "hp_fullgrid_kernels.cuh"
#include "hp_fg1.cuh"
#include "hp_fg4.cuh"

#include <cudaTypedefs.h>

namespace hp {

// ---------------------------------------------------------------- single pass (TMA)

static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

// 4-D map over a complex box viewed as f64 [n0][n1][n2][2 n3]; box (b0 doubles, b1, b2, 1)
static bool tma_map(CUtensorMap* m, const void* base, const int side[4], unsigned b0, unsigned b1, unsigned b2) {
  auto enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {2ull * side[3], (cuuint64_t)side[2], (cuuint64_t)side[1], (cuuint64_t)side[0]};
  cuuint64_t strides[3] = {16ull * side[3], 16ull * side[2] * side[3], 16ull * side[1] * side[2] * side[3]};
  cuuint32_t box[4] = {b0, b1, b2, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// tile order: 3x3 blocks of (i1, i2) columns, i3 fastest, so that the ~148 tiles in
// flight form a compact block whose halos are shared through L2
static hp_status make_tiles(const hp_set_s* s, int T1, int T2, int T3, int** out, int* nout) {
  std::lock_guard<std::mutex> g(s->fg_mtx);
  if (*out) return HP_OK;
  const int t1 = (s->side[1] + T1 - 1) / T1, t2 = (s->side[2] + T2 - 1) / T2, t3 = (s->side[3] + T3 - 1) / T3;
  // blocks of E1 x E2 x E3 tiles (axis 3 fastest inside a block); HP_FG_BLOCK = "e" or "e1,e2,e3"
  int E[3] = {3, 3, t3};
  if (const char* e = getenv("HP_FG_BLOCK")) {
    int a = 0, b = 0, c = 0;
    const int k = sscanf(e, "%d,%d,%d", &a, &b, &c);
    if (k == 1) E[0] = E[1] = std::max(1, a);
    if (k == 3) E[0] = std::max(1, a), E[1] = std::max(1, b), E[2] = std::max(1, c);
  }
  std::vector<int> codes;
  codes.reserve((size_t)t1 * t2 * t3);
  for (int b1 = 0; b1 < t1; b1 += E[0])
    for (int b2 = 0; b2 < t2; b2 += E[1])
      for (int b3 = 0; b3 < t3; b3 += E[2])
        for (int i1 = b1; i1 < std::min(t1, b1 + E[0]); ++i1)
          for (int i2 = b2; i2 < std::min(t2, b2 + E[1]); ++i2)
            for (int i3 = b3; i3 < std::min(t3, b3 + E[2]); ++i3) codes.push_back(i1 | (i2 << 10) | (i3 << 20));
  int* d = nullptr;
  HP_CUDA(cudaMalloc(&d, codes.size() * sizeof(int)));
  HP_CUDA(cudaMemcpy(d, codes.data(), codes.size() * sizeof(int), cudaMemcpyHostToDevice));
  *nout = (int)codes.size();
  *out = d;
  return HP_OK;
}
static hp_status ensure_tiles(const hp_set_s* s) {
  return make_tiles(s, F1_T1, F1_T2, F1_T3, &s->fg_tiles, &s->fg_ntiles);
}

static bool fg_single_enabled() {
  static int v = [] {
    const char* e = getenv("HP_FG_SINGLE");
    return e && atoi(e) == 0 ? 0 : 1;
  }();
  return v == 1;
}

static int fg_quad() {  // HP_FG_QUAD=0 selects the 512-point k_fg_single instead of k_fg_quad
  static int v = [] {
    const char* e = getenv("HP_FG_QUAD");
    return e && atoi(e) == 0 ? 0 : 1;
  }();
  return v;
}

static int fg_np() {  // points per thread of k_fg_single (HP_FG_NP = 1 or 2)
  static int v = [] {
    const char* e = getenv("HP_FG_NP");
    return e && atoi(e) == 1 ? 1 : 2;
  }();
  return v;
}
static int fg_exp() {  // timing experiments only (HP_FG_EXP bit 0: skip halo boxes, bit 1: skip
                       // compute -> wrong results)
  static int v = [] {
    const char* e = getenv("HP_FG_EXP");
    return e ? atoi(e) : 0;
  }();
  return v;
}

static int sm_count() {
  static int n = [] {
    int dev = 0, c = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c;
  }();
  return n;
}

// k_fg_quad: 8 x 8 x 16 tiles, sides <= Q_MAXN
// MIX: bit 0 = the (0,1) coupling class, bit 1 = (0,2), bit 2 = (0,3), bit 3 = (1,3) (hp_fg4.cuh)
constexpr int FG_MIX_ALL = 1 | 2 | 8;
template <int NMIX>
static hp_status launch_quad(const hp_set_s* s, const double2* v, double2* y, const double* P, const double* G,
                             const FgPlan& F, cudaStream_t st, DotOut* dot, bool* launched, int plo, int phi) {
  CUtensorMap mA1, mB2;
  if (!tma_map(&mA1, v, s->side, 2 * Q_RW, Q_T2, Q_T1 + 2 * Q_H) || !tma_map(&mB2, v, s->side, 2 * Q_T3, Q_H, Q_T1))
    return HP_OK;  // no driver entry point: the two-pass kernels run
  hp_status rc = make_tiles(s, Q_T1, Q_T2, Q_T3, &s->fg_tiles4, &s->fg_ntiles4);
  if (rc) return rc;
  const int n0 = s->side[0];
  // axis 0 band that carries the march-axis couplings: degree r0 of the (0,1) class, T_1 otherwise
  const double* B0 = s->fg_basis + (size_t)(NMIX ? (F.nmix ? F.r0[0] : 1) : 0) * n0 * FG_W;
  const int grid = std::min(s->fg_ntiles4, sm_count());
  const bool use_dot = dot && dot->partial && grid <= dot->capacity;
  double2* dotp = use_dot ? dot->partial : nullptr;
  auto kern = use_dot ? k_fg_quad<NMIX, true> : k_fg_quad<NMIX, false>;
  if ((NMIX == 7 || NMIX == FG_MIX_ALL || NMIX == 15) && !use_dot && grid <= FG_DOTP) {
    // three or more couplings: ptxas spills the plain instantiation inside the march (152 bytes of
    // reloads per step, 4.9 ms on the cfg4 cube) but not the one with the fused dot, so that one
    // runs, its partials going to the workspace's dot region (behind the tables and the u vector)
    kern = k_fg_quad<NMIX, true>;
    dotp = (double2*)((char*)P + (size_t)FG_NTAB * FG_MAXN * FG_W * sizeof(double) + 256 + (size_t)s->n * sizeof(double2));
  }
  HP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q_SMEM));
  // exp = 0: k_fg_quad keeps the experiment slot of k_fg_single's signature (dropping it moves
  // ptxas to a spilling allocation of the 255-register kernel)
  kern<<<grid, Q_NT, Q_SMEM, st>>>(mA1, mB2, v, y, P, G, B0, s->fg_tiles4, s->fg_ntiles4, n0, s->side[1],
                                   s->side[2], s->side[3], dotp, fg_exp(), plo, phi);
  HP_LAUNCH_CHECK("k_fg_quad");
  if (use_dot) dot->n = grid;
  *launched = true;
  return HP_OK;
}

// the single-pass evaluator of the cfg4 class (output planes [plo, phi)): k_fg_quad, or
// k_fg_single on cubes with a side > Q_MAXN (HP_FG_QUAD=0 forces it); *launched stays false
// when TMA descriptors are unavailable (the caller then runs the two-pass kernels)
template <int NMIX>
static hp_status launch_single(const hp_set_s* s, const double2* v, double2* y, const double* P, const double* G,
                               const FgPlan& F, cudaStream_t st, DotOut* dot, bool* launched, int plo = 0,
                               int phi = -1) {
  if (phi < 0) phi = s->side[0];
  *launched = false;
  if (fg_quad() && s->side[0] <= Q_MAXN && s->side[1] <= Q_MAXN)
    return launch_quad<NMIX>(s, v, y, P, G, F, st, dot, launched, plo, phi);
  if constexpr (NMIX > 1) return HP_OK;  // the further couplings exist in k_fg_quad only
  CUtensorMap mA1, mB2;
  if (!tma_map(&mA1, v, s->side, 2 * F1_RW, F1_T2, F1_T1 + 2 * F1_H) ||
      !tma_map(&mB2, v, s->side, 2 * F1_T3, F1_H, F1_T1))
    return HP_OK;  // no driver entry point: the two-pass kernels run
  hp_status rc = ensure_tiles(s);
  if (rc) return rc;
  const int n0 = s->side[0];
  const double* B0 = s->fg_basis + (size_t)(NMIX ? F.r0[0] : 0) * n0 * FG_W;  // axis 0, degree r0
  const int grid = std::min(s->fg_ntiles, sm_count());
  const bool use_dot = dot && dot->partial && grid <= dot->capacity;
  const int np = fg_np();
  constexpr int NM1 = NMIX & 1;
  auto kern = np == 1 ? (use_dot ? k_fg_single<NM1, true, 1> : k_fg_single<NM1, false, 1>)
                      : (use_dot ? k_fg_single<NM1, true, 2> : k_fg_single<NM1, false, 2>);
  HP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F1_SMEM));
  kern<<<grid, F1_POINTS / np, F1_SMEM, st>>>(mA1, mB2, v, y, P, G, B0, s->fg_tiles, s->fg_ntiles, n0, s->side[1],
                                              s->side[2], s->side[3], use_dot ? dot->partial : nullptr, fg_exp(),
                                              plo, phi);
  HP_LAUNCH_CHECK("k_fg_single");
  if (use_dot) dot->n = grid;
  *launched = true;
  return HP_OK;
}

static hp_status launch_single_for(const FgPlan& F, const hp_set_s* s, const double2* v, double2* y, const double* P,
                                   const double* G, cudaStream_t st, DotOut* dot, bool* launched, int plo = 0,
                                   int phi = -1) {
  // one instantiation per set of couplings present (an absent coupling costs no shared-memory taps)
  int mix = (F.nmix ? 1 : 0) | (F.cx02 != 0.0 ? 2 : 0) | (F.cx13 != 0.0 ? 8 : 0);
  if (F.cx03 != 0.0) mix |= 7;  // x1 x4 comes with the whole march-axis family (two more instantiations, not eight)
  switch (mix) {
    case 0: return launch_single<0>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 1: return launch_single<1>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 2: return launch_single<2>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 3: return launch_single<3>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 8: return launch_single<8>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 9: return launch_single<9>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 10: return launch_single<10>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 7: return launch_single<7>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    case 15: return launch_single<15>(s, v, y, P, G, F, st, dot, launched, plo, phi);
    default: return launch_single<FG_MIX_ALL>(s, v, y, P, G, F, st, dot, launched, plo, phi);
  }
}

template <unsigned M2, unsigned M3>
static hp_status launch_inner(const hp_set_s* s, const double2* v, double2* u, const double* P, cudaStream_t st) {
  int n2 = s->side[2], n3 = s->side[3];
  int threads = (n3 + 31) / 32 * 32;
  // v2 pass B measured faster than the unrolled v3 (ncu: 1.59 vs 1.77 ms, more CTAs/SM)
  size_t smem = (size_t)FGB_NS * (n3 + 2 * FG_K) * sizeof(double2);
  auto kern = k_fg_inner2<M2, M3>;
  HP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t blocks = (int64_t)s->side[0] * s->side[1];
  kern<<<(unsigned)blocks, threads, smem, st>>>(v, u, P + 2 * FG_MAXN * FG_W, P + 3 * FG_MAXN * FG_W, n2, n3);
  HP_LAUNCH_CHECK("k_fg_inner2");
  return HP_OK;
}

// v2 pass A (runtime ring slots): used for r1 = 2 mixed terms
template <int RM, int NMIX, unsigned M0, unsigned M1>
static hp_status launch_outer(const hp_set_s* s, const double2* v, const double2* u, double2* y, const double* P,
                              const double* G, const FgPlan& F, cudaStream_t st, DotOut* dot) {
  int n0 = s->side[0], n1 = s->side[1];
  int tile = n1 * FG_C;
  const int64_t nblk = (int64_t)s->side[2] * s->side[3] / FG_C;
  const bool use_dot = dot && dot->partial && nblk <= dot->capacity;
  size_t smem = ((size_t)FGA_NS * (n1 + 2 * FG_K) * FG_C + (size_t)FGA_NU * tile) * sizeof(double2);
  auto kern = k_fg_outer2<RM, NMIX, M0, M1>;
  HP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int threads = (tile + 31) / 32 * 32;
  kern<<<(unsigned)nblk, threads, smem, st>>>(v, u, y, P, P + FG_MAXN * FG_W, G, s->fg_basis, n0, n1, s->stride[0],
                                             s->stride[1], F.r0[0], F.r0[1], use_dot ? dot->partial : nullptr);
  if (use_dot) dot->n = (int)nblk;
  HP_LAUNCH_CHECK("k_fg_outer2");
  return HP_OK;
}

// v3 pass A (compile-time ring slots): r1 <= 1.  C = inner chunk; C = 2 (256-thread CTAs,
// two per SM) measured no faster than C = 4 on cfg4 (4.90 vs 4.87 ms), so C = FG_C is used.
template <int RM, int NMIX, unsigned M0, unsigned M1P, unsigned M1G, int C = FG_C>
static hp_status launch_outer3(const hp_set_s* s, const double2* v, const double2* u, double2* y, const double* P,
                               const double* G, const FgPlan& F, cudaStream_t st, DotOut* dot) {
  int n0 = s->side[0], n1 = s->side[1];
  int tile = n1 * C;
  const int64_t nblk = (int64_t)s->side[2] * s->side[3] / C;
  const bool use_dot = dot && dot->partial && nblk <= dot->capacity;
  size_t smem = ((size_t)FG3_U * (n1 + 2 * FG_K) * C + (size_t)FG3_NU * tile) * sizeof(double2);
  auto kern = k_fg_outer3<RM, NMIX, M0, M1P, M1G, C>;
  HP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int threads = (tile + 31) / 32 * 32;
  kern<<<(unsigned)nblk, threads, smem, st>>>(v, u, y, P, P + FG_MAXN * FG_W, G, s->fg_basis, n0, n1, s->stride[0],
                                             s->stride[1], F.r0[0], F.r0[1], use_dot ? dot->partial : nullptr);
  if (use_dot) dot->n = (int)nblk;
  HP_LAUNCH_CHECK("k_fg_outer3");
  return HP_OK;
}

// the terms the fused evaluators take from any polynomial on an N = 4 box (constants, even
// single-axis degrees, T_1 x T_1 pairs) and the rest, for fullgrid_apply_split
static void split_fused_terms(const std::vector<Term>& terms, std::vector<Term>* fused, std::vector<Term>* rest) {
  for (const Term& t : terms) {
    int act[4], na = 0;
    for (int a = 0; a < 4; ++a)
      if (t.r[a] > 0) act[na++] = a;
    const bool in_class = na == 0 || (na == 1 && t.r[act[0]] <= FG_K && t.r[act[0]] % 2 == 0) ||
                          (na == 2 && t.r[act[0]] == 1 && t.r[act[1]] == 1);
    (in_class ? fused : rest)->push_back(t);
  }
}

size_t fullgrid_workspace_bytes(const hp_set_s* s, const std::vector<Term>& terms, int dtype, int64_t batch,
                                int flags) {
  FgPlan F = classify(s, terms, dtype, batch, flags);
  if (!F.ok && s->boxed && s->dim == 4) {  // room for the fused part of a split evaluation
    std::vector<Term> fused, rest;
    split_fused_terms(terms, &fused, &rest);
    if (!fused.empty() && !rest.empty()) F = classify(s, fused, dtype, batch, flags);
  }
  if (!F.ok) return 0;
  // bands | u (two-pass kernels) | per-CTA dot partials of the plane-range entry point
  return (size_t)FG_NTAB * FG_MAXN * FG_W * sizeof(double) + 256 + (size_t)s->n * sizeof(double2) + FG_DOTP_BYTES;
}

// classification + band tables; *ok = false when the fused evaluator does not cover the call
static hp_status fg_prepare(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                            int64_t batch, int flags, void* ws, size_t ws_bytes, cudaStream_t st, FgPlan* Fo,
                            bool* ok, double sq = 0.0) {
  *ok = false;
  FgPlan& F = *Fo;
  F = classify(s, terms, dtype, batch, flags);
  if (!F.ok) return HP_OK;
  if (sq != 0.0)
    for (int a = 0; a < 4; ++a) F.mask[a] |= (1u << (FG_K - 2)) | (1u << FG_K) | (1u << (FG_K + 2));
  size_t need = fullgrid_workspace_bytes(s, terms, dtype, batch, flags);
  if (ws_bytes < need) return HP_OK;  // caller sized for the generic program only
  hp_status rc = ensure_basis(s, halfwidth, st);
  if (rc) return rc;
  double* P = (double*)ws;
  double* G = P + 4 * FG_MAXN * FG_W;
  CombineArgs A;
  for (int a = 0; a < 4; ++a) {
    for (int k = 0; k <= FG_K; ++k) A.ws[a][k] = F.ws[a][k];
    A.side[a] = s->side[a];
  }
  for (int m = 0; m < 2; ++m)
    for (int k = 0; k <= FG_K; ++k) A.wm[m][k] = F.wm[m][k];
  A.joff0 = s->lo;
  A.nmix = F.nmix;
  A.cx02 = F.cx02;
  A.cx03 = F.cx03;
  A.cx13 = F.cx13;
  A.c0 = F.c0;
  A.osc = (flags & HP_ADD_OSC) ? 1 : 0;
  A.sq = sq;
  k_fg_combine<<<64, 256, 0, st>>>(s->fg_basis, P, G, A);
  HP_LAUNCH_CHECK("k_fg_combine");
  *ok = true;
  return HP_OK;
}

// the single-pass kernel covers even single-axis bands and at most one r1 = 1 coupling class
static bool fg_single_class(const FgPlan& F) {
  const bool even = F.mask[0] == FG_MASK_EVEN && F.mask[1] == FG_MASK_EVEN && F.mask[2] == FG_MASK_EVEN &&
                    F.mask[3] == FG_MASK_EVEN;
  return fg_single_enabled() && even &&
         (F.nmix == 0 || (F.nmix == 1 && F.rm == 1 && (F.maskG & ~FG_MASK_PM1) == 0));
}
// the (0,2) / (1,3) couplings exist in k_fg_quad only (sides <= Q_MAXN)
static bool fg_extra_ok(const hp_set_s* s, const FgPlan& F) {
  return !F.extra() || (fg_quad() && s->side[0] <= Q_MAXN && s->side[1] <= Q_MAXN && fg_single_class(F));
}

static hp_status launch_pairs(const hp_set_s* s, const FgPlan& F, const double2* v, double2* y, cudaStream_t st,
                              int plo = 0, int phi = -1);

hp_status fullgrid_apply(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                         const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                         cudaStream_t st, bool* done, DotOut* dot, double sq) {
  if (dot) dot->n = 0;
  *done = false;
  FgPlan F;
  bool ok = false;
  hp_status rc = fg_prepare(s, terms, halfwidth, dtype, batch, flags, ws, ws_bytes, st, &F, &ok, sq);
  if (rc || !ok) return rc;
  double* P = (double*)ws;
  double* G = P + 4 * FG_MAXN * FG_W;
  double2* u = (double2*)((char*)ws + (((size_t)FG_NTAB * FG_MAXN * FG_W * sizeof(double) + 255) & ~(size_t)255));
  const double2* v = (const double2*)in;
  double2* y = (double2*)out;
  const bool even = F.mask[0] == FG_MASK_EVEN && F.mask[2] == FG_MASK_EVEN && F.mask[3] == FG_MASK_EVEN;
  if (F.residual()) dot = nullptr;  // <v, y> would miss the second pass: the caller forms it
  // single pass for the even-band class (cfg4); a batch runs one launch per vector
  if (fg_single_class(F) && fg_extra_ok(s, F)) {
    bool launched = false;
    for (int64_t b = 0; b < batch; ++b) {
      const int64_t off = b * s->n;
      rc = launch_single_for(F, s, v + off, y + off, P, G, st, batch == 1 ? dot : nullptr, &launched);
      if (rc) return rc;
      if (!launched) break;
      if ((rc = launch_pairs(s, F, v + off, y + off, st))) return rc;
    }
    if (launched) {
      *done = true;
      return HP_OK;
    }
  }
  // the two-pass kernels take one vector and need their chunking: otherwise the level evaluator
  if (batch != 1 || !F.twopass || F.extra()) return HP_OK;
  // pass B
  rc = even ? launch_inner<FG_MASK_EVEN, FG_MASK_EVEN>(s, v, u, P, st)
            : launch_inner<FG_MASK_ALL, FG_MASK_ALL>(s, v, u, P, st);
  if (rc) return rc;
  // pass A
  const unsigned m1 = F.mask[1], mg = F.maskG;
  if (F.nmix == 0 && even && m1 == FG_MASK_EVEN)
    rc = launch_outer3<0, 0, FG_MASK_EVEN, FG_MASK_EVEN, 0>(s, v, u, y, P, G, F, st, dot);
  else if (F.nmix == 1 && F.rm == 1 && even && m1 == FG_MASK_EVEN && mg == FG_MASK_PM1)
    rc = launch_outer3<1, 1, FG_MASK_EVEN, FG_MASK_EVEN, FG_MASK_PM1>(s, v, u, y, P, G, F, st, dot);
  else if (F.nmix == 0)
    rc = launch_outer3<0, 0, FG_MASK_ALL, FG_MASK_ALL, 0>(s, v, u, y, P, G, F, st, dot);
  else if (F.rm == 1)
    rc = launch_outer3<1, 1, FG_MASK_ALL, FG_MASK_ALL, FG_MASK_ALL>(s, v, u, y, P, G, F, st, dot);
  else if (F.nmix == 1)
    rc = launch_outer<2, 1, FG_MASK_ALL, FG_MASK_ALL>(s, v, u, y, P, G, F, st, dot);
  else
    rc = launch_outer<2, 2, FG_MASK_ALL, FG_MASK_ALL>(s, v, u, y, P, G, F, st, dot);
  if (rc) return rc;
  if ((rc = launch_pairs(s, F, v, y, st))) return rc;
  *done = true;
  return HP_OK;
}


// ---------------------------------------------------------------- fused part + level remainder

hp_status fullgrid_apply_split(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                               const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                               cudaStream_t st, bool* done, DotOut* dot, double sq) {
  hp_status rc = fullgrid_apply(s, terms, halfwidth, dtype, in, out, batch, flags, ws, ws_bytes, st, done, dot, sq);
  if (rc || *done) return rc;
  if (!s->boxed || s->dim != 4 || dtype != HP_C128 || !fg_single_enabled()) return HP_OK;
  std::vector<Term> fused, rest;
  split_fused_terms(terms, &fused, &rest);
  if (fused.empty() || rest.empty()) return HP_OK;
  // the remainder must be cheaper in level passes than the whole polynomial by more than the fused launch
  const double c_all = level_plan_cost(s->dim, terms), c_rest = level_plan_cost(s->dim, rest);
  if (c_rest < 0.0 || (c_all >= 0.0 && c_rest + 2.0 > c_all)) return HP_OK;
  if (level_workspace_bytes(s, rest, dtype, 1) > ws_bytes || fullgrid_workspace_bytes(s, fused, dtype, batch, flags) > ws_bytes ||
      fullgrid_workspace_bytes(s, fused, dtype, batch, flags) == 0)
    return HP_OK;
  bool done_a = false, done_b = false;
  rc = fullgrid_apply(s, fused, halfwidth, dtype, in, out, batch, flags, ws, ws_bytes, st, &done_a, nullptr, sq);
  if (rc || !done_a) return rc;
  // y += (remaining terms) v; the oscillator and the harmonic part went with the fused part
  rc = level_apply(s, rest, halfwidth, dtype, in, out, batch, (flags & ~HP_ADD_OSC) | HP_LV_ACCUMULATE, ws, ws_bytes, st,
                   &done_b, nullptr);
  if (rc) return rc;
  if (dot) dot->n = 0;  // <v, y> is left to the caller
  *done = done_b;       // (not done: the caller's evaluator overwrites y with the whole polynomial)
  return HP_OK;
}

// ---------------------------------------------------------------- residual pair couplings

struct PairArgs {
  int side[4];
  double c[3];  // coefficients of the pairs (0,3), (1,2), (2,3)
};

// y += sum_pairs c_ab T_1(X_a / L) T_1(X_b / L) v on a 4-D box: the four corner neighbours
// (j_a +- 1, j_b +- 1) weighted by the T_1 bands (zero across the faces, global j on a slab's axis 0).
// A streaming pass behind the fused evaluator for the pairs whose corners its halo boxes do not
// hold (MASK: bit i = pair i present).  blockIdx.y = j0; a block owns 256 consecutive points of
// the (j2, j3) cross-section and marches j1, so its j2 / j3 weights are formed once and the rows
// (j1 + 1, j2 +- 1) it loads at one step are the rows (j1' - 1, ..) of the step after next
// (L1 / L2 hits); consecutive threads run along the last axis.
template <int MASK>
__global__ void __launch_bounds__(256) k_fg_pairs(const double2* __restrict__ v, double2* __restrict__ y,
                                                  const double* __restrict__ basis, PairArgs A, int plo) {
  constexpr size_t bs = (size_t)(FG_K + 1) * FG_MAXN * FG_W;
  const unsigned n1 = A.side[1], n2 = A.side[2], n3 = A.side[3], cross = n2 * n3;
  const unsigned q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cross) return;
  const int j0 = plo + (int)blockIdx.y, j2 = (int)(q / n3), j3 = (int)(q % n3);  // output planes [plo, plo + gridDim.y)
  const int64_t plane = (int64_t)n1 * cross;
  // T_1 band of axis a at row j: entries (j, j - 1) and (j, j + 1), zero across the faces
  auto band = [&](int a, int j, double& wm, double& wp) {
    const double* B = basis + a * bs + ((size_t)A.side[a] + j) * FG_W + FG_K;  // degree 1, row j, centre
    wm = j > 0 ? __ldg(B - 1) : 0.0;
    wp = j + 1 < A.side[a] ? __ldg(B + 1) : 0.0;
  };
  // c . sum over the corners (j_a +- 1, j_b +- 1); sa, sb = element strides of the two axes
  auto corners = [&](const double2* x, int64_t sa, int64_t sb, double wam, double wap, double wbm, double wbp, double c,
                     double2& acc) {
    auto row = [&](const double2* xr, double wa) {
      if (wa == 0.0) return;
      double2 h = make_double2(0.0, 0.0);
      if (wbm != 0.0) {
        const double2 t = __ldg(xr - sb);
        h.x = wbm * t.x;
        h.y = wbm * t.y;
      }
      if (wbp != 0.0) {
        const double2 t = __ldg(xr + sb);
        h.x = fma(wbp, t.x, h.x);
        h.y = fma(wbp, t.y, h.y);
      }
      acc.x = fma(c * wa, h.x, acc.x);
      acc.y = fma(c * wa, h.y, acc.y);
    };
    row(x - sa, wam);
    row(x + sa, wap);
  };
  double w0m = 0.0, w0p = 0.0, w3m = 0.0, w3p = 0.0, w2m = 0.0, w2p = 0.0;
  if (MASK & 1) band(0, j0, w0m, w0p);
  if (MASK & 5) band(3, j3, w3m, w3p);
  if (MASK & 6) band(2, j2, w2m, w2p);
  const double2* x = v + (int64_t)j0 * plane + q;
  double2* yo = y + (int64_t)j0 * plane + q;
  for (unsigned j1 = 0; j1 < n1; ++j1, x += cross, yo += cross) {
    double2 acc = make_double2(0.0, 0.0);
    if (MASK & 1) corners(x, plane, 1, w0m, w0p, w3m, w3p, A.c[0], acc);
    if (MASK & 2) {
      double w1m, w1p;
      band(1, (int)j1, w1m, w1p);
      corners(x, cross, n3, w1m, w1p, w2m, w2p, A.c[1], acc);
    }
    if (MASK & 4) corners(x, n3, 1, w2m, w2p, w3m, w3p, A.c[2], acc);
    double2 out = *yo;
    out.x += acc.x;
    out.y += acc.y;
    *yo = out;
  }
}

static hp_status launch_pairs(const hp_set_s* s, const FgPlan& F, const double2* v, double2* y, cudaStream_t st,
                              int plo, int phi) {
  if (phi < 0) phi = s->side[0];
  if (!F.residual() || phi <= plo) return HP_OK;
  PairArgs A;
  for (int a = 0; a < 4; ++a) A.side[a] = s->side[a];
  int mask = 0;
  for (int i = 0; i < 3; ++i) {
    A.c[i] = F.cres[i];
    if (F.cres[i] != 0.0) mask |= 1 << i;
  }
  const dim3 grid((unsigned)(((int64_t)s->side[2] * s->side[3] + 255) / 256), (unsigned)(phi - plo));
  switch (mask) {
    case 1: k_fg_pairs<1><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
    case 2: k_fg_pairs<2><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
    case 3: k_fg_pairs<3><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
    case 4: k_fg_pairs<4><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
    case 5: k_fg_pairs<5><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
    case 6: k_fg_pairs<6><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
    default: k_fg_pairs<7><<<grid, 256, 0, st>>>(v, y, s->fg_basis, A, plo); break;
  }
  HP_LAUNCH_CHECK("k_fg_pairs");
  return HP_OK;
}

// ---------------------------------------------------------------- plane ranges

// y on output j1-planes [plo, phi) only (reads input planes [plo - 4, phi + 4)); *done = false
// when the set / terms are outside the single-pass class
// dot_accum[0..1] += sum of the per-CTA partials, in CTA order (one block)
__global__ void k_fg_dot_accum(const double2* __restrict__ partial, int n, double* __restrict__ acc) {
  __shared__ double2 sh[256];
  double2 a = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    a.x += partial[i].x;
    a.y += partial[i].y;
  }
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sh[threadIdx.x].x += sh[threadIdx.x + w].x;
      sh[threadIdx.x].y += sh[threadIdx.x + w].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    acc[0] += sh[0].x;
    acc[1] += sh[0].y;
  }
}

hp_status fullgrid_apply_planes(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                                const void* in, void* out, int plo, int phi, int flags, void* ws, size_t ws_bytes,
                                cudaStream_t st, bool* done, double* dot_accum, double sq) {
  *done = false;
  FgPlan F = classify(s, terms, dtype, 1, flags);
  // (with second-pass couplings the rows of x^H A x are not formed in-kernel: the caller's other route)
  if (!F.ok || !fg_single_class(F) || !fg_extra_ok(s, F) || (F.residual() && dot_accum)) return HP_OK;
  if (plo == phi) {  // support query: nothing to compute
    *done = ws_bytes >= fullgrid_workspace_bytes(s, terms, dtype, 1, flags);
    return HP_OK;
  }
  bool ok = false;
  hp_status rc = fg_prepare(s, terms, halfwidth, dtype, 1, flags, ws, ws_bytes, st, &F, &ok, sq);
  if (rc || !ok) return rc;
  const double* P = (const double*)ws;
  const double* G = P + 4 * FG_MAXN * FG_W;
  bool launched = false;
  DotOut d;
  if (dot_accum) {
    d.partial = (double2*)((char*)ws + fullgrid_workspace_bytes(s, terms, dtype, 1, flags) - FG_DOTP_BYTES);
    d.capacity = FG_DOTP;
  }
  DotOut* dp = dot_accum ? &d : nullptr;
  rc = launch_single_for(F, s, (const double2*)in, (double2*)out, P, G, st, dp, &launched, plo, phi);
  if (rc) return rc;
  if (launched && dot_accum) {
    if (d.n == 0) return fail(HP_ERR_RUNTIME, "plane-range matvec: fused dot unavailable");
    k_fg_dot_accum<<<1, 256, 0, st>>>(d.partial, d.n, dot_accum);
    HP_LAUNCH_CHECK("k_fg_dot_accum");
  }
  if (launched && (rc = launch_pairs(s, F, (const double2*)in, (double2*)out, st, plo, phi))) return rc;
  *done = launched;
  return HP_OK;
}

// ---------------------------------------------------------------- streamed (host-resident vectors)

// copy streams of the streamed matvec, one pair per device
hp_status copy_streams(cudaStream_t* in, cudaStream_t* out) {
  static std::mutex mtx;
  static std::map<int, std::pair<cudaStream_t, cudaStream_t>> per_dev;
  int dev = 0;
  HP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mtx);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    cudaStream_t a, b;
    HP_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    HP_CUDA(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
    it = per_dev.emplace(dev, std::make_pair(a, b)).first;
  }
  *in = it->second.first;
  *out = it->second.second;
  return HP_OK;
}

// y = W v for host-resident v / y on a full cube of the single-pass class.  The cube is cut
// into chunks of j1 planes (~64 MB); chunk k is copied in on one stream, its output planes are
// computed on `st` once the chunks holding its band halo (4 planes) have landed, and copied out
// on a third stream, so PCIe traffic in both directions overlaps the kernels.  cfg4 measures
// 92 ms for 4.3 GB each way (46.5 GB/s per direction, the duplex limit of the link: chunk sizes
// of 1-8 planes all land within 3%).  *done = false when
// the set / terms are not covered (the caller then copies whole vectors).
hp_status fullgrid_apply_streamed(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                                  const void* in_host, void* out_host, void* in_dev, void* out_dev, int flags,
                                  void* ws, size_t ws_bytes, cudaStream_t st, bool* done) {
  *done = false;
  FgPlan F = classify(s, terms, dtype, 1, flags);
  if (!F.ok || !fg_single_class(F) || !fg_extra_ok(s, F)) return HP_OK;
  bool ok = false;
  hp_status rc = fg_prepare(s, terms, halfwidth, dtype, 1, flags, ws, ws_bytes, st, &F, &ok);
  if (rc || !ok) return rc;
  const double* P = (const double*)ws;
  const double* G = P + 4 * FG_MAXN * FG_W;
  const int n0 = s->side[0];
  const size_t plane = (size_t)(s->n / n0) * sizeof(double2);
  int C = (int)std::min<size_t>(n0, ((size_t)64 << 20) / std::max<size_t>(plane, 1));
  if (const char* e = getenv("HP_STREAM_CHUNK")) C = atoi(e);  // planes per chunk (tests)
  C = std::max(C, 1);
  const int ahead = (F1_H + C - 1) / C;  // chunks k+1 .. k+ahead hold the band halo of chunk k
  const int nch = (n0 + C - 1) / C;
  cudaStream_t sin, sout;
  if ((rc = copy_streams(&sin, &sout))) return rc;
  StreamedEvents ev;
  if ((rc = ev.create(2 * nch + 2))) return rc;
  ev.drain[0] = sin;
  ev.drain[1] = sout;
  cudaEvent_t ev0 = ev[2 * nch], evend = ev[2 * nch + 1];
  HP_CUDA(cudaEventRecord(ev0, st));  // orders the copies after the caller's prior work
  HP_CUDA(cudaStreamWaitEvent(sin, ev0, 0));
  HP_CUDA(cudaStreamWaitEvent(sout, ev0, 0));
  for (int k = 0; k < nch; ++k) {
    const int p0 = k * C, p1 = std::min(n0, p0 + C);
    HP_CUDA(cudaMemcpyAsync((char*)in_dev + p0 * plane, (const char*)in_host + p0 * plane, (p1 - p0) * plane,
                            cudaMemcpyHostToDevice, sin));
    HP_CUDA(cudaEventRecord(ev[k], sin));
  }
  for (int k = 0; k < nch; ++k) {
    const int p0 = k * C, p1 = std::min(n0, p0 + C);
    HP_CUDA(cudaStreamWaitEvent(st, ev[std::min(k + ahead, nch - 1)], 0));
    bool launched = false;
    rc = launch_single_for(F, s, (const double2*)in_dev, (double2*)out_dev, P, G, st, nullptr, &launched, p0, p1);
    if (rc) return rc;
    if (!launched) return fail(HP_ERR_RUNTIME, "streamed matvec: TMA descriptors unavailable");
    // second-pass couplings of these planes: their corner rows (planes p0 - 1 .. p1) have arrived
    if ((rc = launch_pairs(s, F, (const double2*)in_dev, (double2*)out_dev, st, p0, p1))) return rc;
    HP_CUDA(cudaEventRecord(ev[nch + k], st));
    HP_CUDA(cudaStreamWaitEvent(sout, ev[nch + k], 0));
    HP_CUDA(cudaMemcpyAsync((char*)out_host + p0 * plane, (const char*)out_dev + p0 * plane, (p1 - p0) * plane,
                            cudaMemcpyDeviceToHost, sout));
  }
  HP_CUDA(cudaEventRecord(evend, sout));
  HP_CUDA(cudaStreamWaitEvent(st, evend, 0));
  ev.committed = true;
  *done = true;
  return HP_OK;
}

}  // namespace hp
