// Lanczos / Magnus time stepping on the device (reference:
// krylov_propagator.py:58-263, error_lab.py:154-185).
//
// One exponential step runs without any host synchronisation: the Lanczos
// recurrence scalars (alpha_k, beta_k, breakdown state) live in a small
// device struct, every reduction is a fixed-shape two-stage tree (so results
// are bitwise reproducible run to run), breakdown (beta_k <= 1e-14,
// krylov_propagator.py:29, 90-93) truncates the factorisation on the device,
// and the tridiagonal eigenproblem (implicit-shift QL, :107-170) plus
// exp(-i tau T) e_1 (:173-177) run in one device thread.  The whole step is
// therefore a pure launch sequence (CUDA-graph capturable).
#include <algorithm>
#include <string>
#include <vector>

#include "hp_common.cuh"
#include "hp_program.h"

#define HP_MAXM 48
#define HP_RED_BLOCKS 592
#define HP_RED_THREADS 256

namespace hp {

// Scaled Lanczos: the basis is stored unnormalised (row k holds w_k with
// v_k = scale[k] * w_k), so no separate normalisation pass is needed; the
// scales enter the next update and the final combine as scalars.
struct LzState {
  double alpha[HP_MAXM];
  double beta[HP_MAXM];
  double scale[HP_MAXM];
  double2 col[HP_MAXM];
  double2 reo[HP_MAXM];
  double nrm0;
  double defect;
  double scratch;
  int m_eff;
  int broken;
  int breakdown_at;
  int ql_fail;
};

// ---------------------------------------------------------------- reductions

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

template <int MODE>  // 0: sum conj(a)*b (complex); 1: sum |a|^2 (re in .x)
__global__ void __launch_bounds__(HP_RED_THREADS) k_red_partial(int64_t n, const double2* __restrict__ a,
                                                                const double2* __restrict__ b,
                                                                double2* __restrict__ partial) {
  __shared__ double2 sh[HP_RED_THREADS];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = __ldg(a + i);
    if (MODE == 0) {
      double2 y = __ldg(b + i);
      acc.x = fma(x.x, y.x, fma(x.y, y.y, acc.x));
      acc.y = fma(x.x, y.y, fma(-x.y, y.x, acc.y));
    } else {
      acc.x = fma(x.x, x.x, fma(x.y, x.y, acc.x));
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = HP_RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__device__ double2 block_sum_partials(const double2* partial, int np) {
  __shared__ double2 sh[HP_RED_THREADS];
  double2 acc = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc = cadd(acc, partial[i]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = HP_RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  return sh[0];
}

// what: 1 nrm0 and scale_0 (norm), 4 write dot to out[0..1], 5 write norm to out[0],
//       6 alpha_k (scaled dot), 7 beta_k / scale_{k+1} / breakdown (norm), 8 reorth coefficient
__device__ void lz_scalar(double2 s, LzState* st, int k, int what, double tol, double* out);

__global__ void __launch_bounds__(HP_RED_THREADS) k_red_final(const double2* partial, int np, LzState* st,
                                                              int k, int what, double tol, double* out) {
  double2 s = block_sum_partials(partial, np);
  if (threadIdx.x != 0) return;
  lz_scalar(s, st, k, what, tol, out);
}

// one already-reduced scalar into the Lanczos state (the sharded path: the per-rank partials are
// summed across ranks in rank order before this)
__global__ void k_lz_set(const double* value, LzState* st, int k, int what, double tol) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  lz_scalar(make_double2(value[0], value[1]), st, k, what, tol, nullptr);
}

__device__ void lz_scalar(double2 s, LzState* st, int k, int what, double tol, double* out) {
  if (what == 4) { out[0] = s.x; out[1] = s.y; return; }
  if (what == 5) { out[0] = sqrt(s.x); return; }
  if (st->broken && k >= st->m_eff) return;
  if (what == 6) {  // alpha_k = s_k^2 <w_k, A w_k>
    double s2 = st->scale[k] * st->scale[k];
    st->alpha[k] = s2 * s.x;
    st->defect = fmax(st->defect, fabs(s2 * s.y));
  } else if (what == 7) {  // beta_k = ||w_{k+1}||, scale_{k+1} = 1 / beta_k
    double bk = sqrt(s.x);
    if (bk <= tol) {
      st->broken = 1;
      st->m_eff = k + 1;
      st->breakdown_at = k + 1;
    } else {
      st->beta[k] = bk;
      st->scale[k + 1] = 1.0 / bk;
    }
  } else if (what == 8) {  // reorthogonalisation coefficient c_k = s_k <w_k, w'>
    st->reo[k] = make_double2(st->scale[k] * s.x, st->scale[k] * s.y);
  } else if (what == 1) {
    st->nrm0 = sqrt(s.x);
    st->scale[0] = 1.0 / st->nrm0;
  }
}

static hp_status reduce(int mode, int64_t n, const double2* a, const double2* b, double2* partial, LzState* st,
                        int k, int what, double tol, double* out, cudaStream_t s) {
  if (mode == 0) k_red_partial<0><<<HP_RED_BLOCKS, HP_RED_THREADS, 0, s>>>(n, a, b, partial);
  else k_red_partial<1><<<HP_RED_BLOCKS, HP_RED_THREADS, 0, s>>>(n, a, nullptr, partial);
  HP_LAUNCH_CHECK("k_red_partial");
  k_red_final<<<1, HP_RED_THREADS, 0, s>>>(partial, HP_RED_BLOCKS, st, k, what, tol, out);
  HP_LAUNCH_CHECK("k_red_final");
  return HP_OK;
}

// ---------------------------------------------------------------- vector kernels

// gl2 operator average: out = 0.5 (y1 + y2) - i gamma (z2 - z1)  (krylov_propagator.py:226-231).
// With `v` and `dotp`, the block partials of v^H out (the Lanczos alpha of this Krylov matvec) are
// formed in the same pass -- one extra vector read instead of a separate two-vector dot pass.
__global__ void __launch_bounds__(256) k_gl2_combine(int64_t n, const double2* __restrict__ y1,
                                                     const double2* __restrict__ y2,
                                                     const double2* __restrict__ z2y1,
                                                     const double2* __restrict__ z1y2, double gamma,
                                                     double2* __restrict__ out, const double2* __restrict__ v,
                                                     double2* __restrict__ dotp) {
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 c = ssub(__ldg(z2y1 + i), __ldg(z1y2 + i));
    double2 h = smul(0.5, sadd(__ldg(y1 + i), __ldg(y2 + i)));
    double2 ic = make_double2(__dsub_rn(__dmul_rn(0.0, c.x), __dmul_rn(gamma, c.y)),
                              __dadd_rn(__dmul_rn(0.0, c.y), __dmul_rn(gamma, c.x)));
    const double2 o = ssub(h, ic);
    out[i] = o;
    if (dotp) cdot_acc(__ldg(v + i), o, acc);
  }
  if (dotp) {
    acc = block_sum2(acc);
    if (threadIdx.x == 0) dotp[blockIdx.x] = acc;
  }
}

// scaled update w_{k+1} = s_k z - alpha_k s_k w_k - beta_{k-1} s_{k-1} w_{k-1}
// (= A v_k - alpha_k v_k - beta_{k-1} v_{k-1}, krylov_propagator.py:86) fused with
// the partial sums of ||w_{k+1}||^2 (:89)
__global__ void __launch_bounds__(HP_RED_THREADS) k_lz_update_s(int64_t n, const double2* __restrict__ z,
                                                                const double2* __restrict__ wk,
                                                                const double2* __restrict__ wkm1,
                                                                double2* __restrict__ wn, const LzState* st, int k,
                                                                double2* __restrict__ partial) {
  __shared__ double2 sh[HP_RED_THREADS];
  double2 acc = make_double2(0.0, 0.0);
  if (!(st->broken && k >= st->m_eff)) {
    const double sk = st->scale[k];
    const double ca = st->alpha[k] * sk;
    const double cb = k > 0 ? st->beta[k - 1] * st->scale[k - 1] : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      double2 a = __ldg(z + i), b = __ldg(wk + i);
      double2 r = make_double2(fma(sk, a.x, -ca * b.x), fma(sk, a.y, -ca * b.y));
      if (k > 0) {
        double2 c = __ldg(wkm1 + i);
        r.x = fma(-cb, c.x, r.x);
        r.y = fma(-cb, c.y, r.y);
      }
      wn[i] = r;
      acc.x = fma(r.x, r.x, fma(r.y, r.y, acc.x));
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = HP_RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

// scaled reorthogonalisation: w' -= sum_{j<=k} reo[j] s_j w_j  (reo[j] = <v_j, w'>)
__global__ void k_lz_reorth_s(int64_t n, double2* __restrict__ w, const double2* __restrict__ w0,
                              const double2* __restrict__ V, const LzState* st, int k) {
  if (st->broken && k >= st->m_eff) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j <= k; ++j) {
      double2 c = st->reo[j];
      double sj = st->scale[j];
      double2 v = __ldg((j == 0 ? w0 : V + (int64_t)(j - 1) * n) + i);
      acc.x += sj * (c.x * v.x - c.y * v.y);
      acc.y += sj * (c.x * v.y + c.y * v.x);
    }
    w[i] = ssub(w[i], acc);
  }
}

// y = nrm0 * sum_{k < m_eff} col_k s_k w_k  (krylov_propagator.py:186); row 0 may alias y
__global__ void k_lz_combine_s(int64_t n, const double2* w0, const double2* __restrict__ V, const LzState* st,
                               double2* y) {
  const int m = st->m_eff;
  const double s = st->nrm0;
  double2 c[HP_MAXM];
  for (int k = 0; k < m; ++k) c[k] = make_double2(st->col[k].x * st->scale[k], st->col[k].y * st->scale[k]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < m; ++k) {
      double2 v = (k == 0 ? w0 : V + (int64_t)(k - 1) * n)[i];
      acc.x += v.x * c[k].x - v.y * c[k].y;
      acc.y += v.x * c[k].y + v.y * c[k].x;
    }
    y[i] = make_double2(s * acc.x, s * acc.y);
  }
}

// the same combine over separate basis vectors (the sharded path's per-rank own-plane views)
struct LzPtrs {
  const double2* v[HP_MAXM];
};
__global__ void k_lz_combine_ptrs(int64_t n, LzPtrs P, const LzState* st, double2* y) {
  const int m = st->m_eff;
  const double s = st->nrm0;
  double2 c[HP_MAXM];
  for (int k = 0; k < m; ++k) c[k] = make_double2(st->col[k].x * st->scale[k], st->col[k].y * st->scale[k]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < m; ++k) {
      double2 v = P.v[k][i];
      acc.x += v.x * c[k].x - v.y * c[k].y;
      acc.y += v.x * c[k].y + v.y * c[k].x;
    }
    y[i] = make_double2(s * acc.x, s * acc.y);
  }
}

// rows k >= 1 of an unnormalised basis -> v_k = s_k w_k (hp_lanczos output)
__global__ void k_lz_normalize_rows(int64_t n, double2* __restrict__ B, const LzState* st) {
  const int m = st->m_eff;
  for (int k = 0; k < m; ++k) {
    const double s = st->scale[k];
    double2* row = B + (int64_t)k * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      row[i] = make_double2(row[i].x * s, row[i].y * s);
  }
}

// ---------------------------------------------------------------- tridiagonal QL

// implicit-shift QL with eigenvectors (krylov_propagator.py:107-170);
// returns false on non-convergence.  d[m], e[m] (e[m-1] = 0), z[m*m] col-major z[i + j*m].
__device__ bool ql_eigh(int m, double* d, double* e, double* z) {
  for (int i = 0; i < m * m; ++i) z[i] = 0.0;
  for (int i = 0; i < m; ++i) z[i + i * m] = 1.0;
  if (m == 1) return true;
  for (int l = 0; l < m; ++l) {
    int it = 0;
    while (true) {
      int mm = l;
      while (mm < m - 1) {
        double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 1e-14 * dd) break;
        ++mm;
      }
      if (mm == l) break;
      if (it == 30) return false;
      ++it;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      double s = 1.0, c = 1.0, p = 0.0;
      bool early = false;
      for (int i = mm - 1; i >= l; --i) {
        double f = s * e[i];
        double b = c * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[mm] = 0.0;
          early = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        for (int row = 0; row < m; ++row) {
          double zi = z[row + i * m], zi1 = z[row + (i + 1) * m];
          z[row + (i + 1) * m] = s * zi + c * zi1;
          z[row + i * m] = c * zi - s * zi1;
        }
      }
      if (!early) {
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    }
  }
  return true;
}

// col = Z exp(-i tau Lambda) Z[0,:]  (krylov_propagator.py:173-177)
__device__ bool expm_col(int m, const double* alpha, const double* beta, double tau, double2* col) {
  double d[HP_MAXM], e[HP_MAXM], z[HP_MAXM * HP_MAXM];
  int order[HP_MAXM];
  for (int i = 0; i < m; ++i) {
    d[i] = alpha[i];
    e[i] = (i < m - 1) ? beta[i] : 0.0;
  }
  if (!ql_eigh(m, d, e, z)) return false;
  // stable ascending order (np.argsort kind="stable")
  for (int i = 0; i < m; ++i) order[i] = i;
  for (int i = 1; i < m; ++i) {
    int t = order[i], j = i - 1;
    while (j >= 0 && d[order[j]] > d[t]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = t;
  }
  double2 c[HP_MAXM];
  for (int jj = 0; jj < m; ++jj) {
    int j = order[jj];
    double x = tau * d[j];
    double sn, cs;
    sincos(x, &sn, &cs);
    double z0 = z[0 + j * m];
    c[jj] = make_double2(cs * z0, -sn * z0);
  }
  for (int i = 0; i < m; ++i) {
    double2 acc = make_double2(0.0, 0.0);
    for (int jj = 0; jj < m; ++jj) {
      double zij = z[i + order[jj] * m];
      acc.x += zij * c[jj].x;
      acc.y += zij * c[jj].y;
    }
    col[i] = acc;
  }
  return true;
}

// The same QL + exp as ql_eigh / expm_col, run by the 32 lanes of one warp: the scalar
// recurrence (d, e, rotation parameters) is evaluated redundantly and identically by every lane,
// and lane r applies each rotation to rows r and r + 32 of Z, kept in lane-private arrays (the
// single-thread version spends most of its time on the m x m local-memory eigenvector updates).
// Same operations in the same order per element: bitwise identical to expm_col.  Every lane
// returns the convergence flag; lane i writes col[i] (and col[i + 32]).
__device__ bool expm_col_warp(int m, const double* alpha, const double* beta, double tau, double2* col) {
  const int lane = threadIdx.x & 31;
  double d[HP_MAXM], e[HP_MAXM], z0r[HP_MAXM], z1r[HP_MAXM];  // rows lane, lane + 32 of Z
  for (int i = 0; i < m; ++i) {
    d[i] = alpha[i];
    e[i] = (i < m - 1) ? beta[i] : 0.0;
    z0r[i] = (i == lane) ? 1.0 : 0.0;
    z1r[i] = (i == lane + 32) ? 1.0 : 0.0;
  }
  const bool has0 = lane < m, has1 = lane + 32 < m;
  bool ok = true;
  if (m > 1) {
    for (int l = 0; l < m && ok; ++l) {
      int it = 0;
      while (true) {
        int mm = l;
        while (mm < m - 1) {
          double dd = fabs(d[mm]) + fabs(d[mm + 1]);
          if (fabs(e[mm]) <= 1e-14 * dd) break;
          ++mm;
        }
        if (mm == l) break;
        if (it == 30) {
          ok = false;
          break;
        }
        ++it;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
        double s = 1.0, c = 1.0, p = 0.0;
        bool early = false;
        for (int i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          if (has0) {
            double zi = z0r[i], zi1 = z0r[i + 1];
            z0r[i + 1] = s * zi + c * zi1;
            z0r[i] = c * zi - s * zi1;
          }
          if (has1) {
            double zi = z1r[i], zi1 = z1r[i + 1];
            z1r[i + 1] = s * zi + c * zi1;
            z1r[i] = c * zi - s * zi1;
          }
        }
        if (!early) {
          d[l] -= p;
          e[l] = g;
          e[mm] = 0.0;
        }
      }
    }
  }
  if (!ok) return false;
  int order[HP_MAXM];
  for (int i = 0; i < m; ++i) order[i] = i;
  for (int i = 1; i < m; ++i) {
    int t = order[i], j = i - 1;
    while (j >= 0 && d[order[j]] > d[t]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = t;
  }
  double2 c[HP_MAXM];
  for (int jj = 0; jj < m; ++jj) {
    int j = order[jj];
    double x = tau * d[j];
    double sn, cs;
    sincos(x, &sn, &cs);
    double zz0 = __shfl_sync(0xffffffffu, z0r[j], 0);  // Z[0, j] lives in lane 0
    c[jj] = make_double2(cs * zz0, -sn * zz0);
  }
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    if (i >= m) continue;
    const double* zr = h ? z1r : z0r;
    double2 acc = make_double2(0.0, 0.0);
    for (int jj = 0; jj < m; ++jj) {
      double zij = zr[order[jj]];
      acc.x += zij * c[jj].x;
      acc.y += zij * c[jj].y;
    }
    col[i] = acc;
  }
  return true;
}

}  // namespace hp
#include "hp_small.cuh"
namespace hp {

__global__ void k_lz_expm(LzState* st, double tau) {  // one warp
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const bool ok = expm_col_warp(st->m_eff, st->alpha, st->beta, tau, st->col);
  if (threadIdx.x == 0 && !ok) st->ql_fail = 1;
}

__global__ void k_expm_standalone(const double* alpha, const double* beta, int m, double tau, double2* col,
                                  int* status) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;  // one warp
  const bool ok = expm_col_warp(m, alpha, beta, tau, col);
  if (status && threadIdx.x == 0) *status = ok ? 0 : 1;
}

__global__ void k_tridiag_eigh(const double* alpha, const double* beta, int m, double* dout, double* zout,
                               int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double d[HP_MAXM], e[HP_MAXM], z[HP_MAXM * HP_MAXM];
  int order[HP_MAXM];
  for (int i = 0; i < m; ++i) {
    d[i] = alpha[i];
    e[i] = (i < m - 1) ? beta[i] : 0.0;
  }
  bool ok = ql_eigh(m, d, e, z);
  for (int i = 0; i < m; ++i) order[i] = i;
  for (int i = 1; i < m; ++i) {
    int t = order[i], j = i - 1;
    while (j >= 0 && d[order[j]] > d[t]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = t;
  }
  for (int j = 0; j < m; ++j) {
    dout[j] = d[order[j]];
    for (int i = 0; i < m; ++i) zout[i * m + j] = z[i + order[j] * m];
  }
  if (status) *status = ok ? 0 : 1;
}

__global__ void k_lz_init(LzState* st, int m) {
  if (threadIdx.x != 0) return;
  st->m_eff = m;
  st->broken = 0;
  st->breakdown_at = -1;
  st->ql_fail = 0;
  st->defect = 0.0;
  st->nrm0 = 0.0;
  st->scratch = 0.0;
}

__global__ void k_lz_diag(const LzState* st, double* diag, double* alpha, double* beta) {
  if (threadIdx.x != 0) return;
  if (diag) {
    diag[0] = st->m_eff;
    diag[1] = st->defect;
    diag[2] = st->breakdown_at;
    diag[3] = st->ql_fail ? 1.0 : 0.0;
  }
  if (alpha) for (int k = 0; k < st->m_eff; ++k) alpha[k] = st->alpha[k];
  if (beta) for (int k = 0; k + 1 < st->m_eff; ++k) beta[k] = st->beta[k];
}

// ---------------------------------------------------------------- operator

// A(t) v = (D + W_pol) v [+ q * square_sum v]  (error_lab.py:173-185)
struct Hamiltonian {
  const hp_set_s* s;
  Program prog;
  double halfwidth;
  double q;
  std::vector<Term> terms;
};

// the fused full-cube evaluator folds q * square_sum into its bands (*sq_done); the other
// evaluators leave it to apply_ham_full
static hp_status apply_ham(const Hamiltonian& H, const double2* v, double2* y, double2* ws, size_t ws_bytes,
                           cudaStream_t st, DotOut* dot, bool* sq_done) {
  bool done = false;
  *sq_done = false;
  hp_status rc = fullgrid_apply_split(H.s, H.terms, H.halfwidth, HP_C128, v, y, 1, HP_ADD_OSC, ws, ws_bytes, st, &done,
                                      dot, H.q);
  if (rc) return rc;
  if (done) {
    *sq_done = true;
    return HP_OK;
  }
  DotOut* d = H.q == 0.0 ? dot : nullptr;
  if (dot && !d) dot->n = 0;
  rc = level_apply(H.s, H.terms, H.halfwidth, HP_C128, v, y, 1, HP_ADD_OSC, ws, ws_bytes, st, &done, d);
  if (rc) return rc;
  if (!done) rc = run_program<double2>(H.s, H.prog, H.halfwidth, v, y, 1, ws, ws_bytes, st, d);
  return rc;
}

__global__ void k_axpy_c2(int64_t n, double c, const double2* __restrict__ x, double2* __restrict__ acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[i] = sadd(acc[i], smul(c, __ldg(x + i)));
}

// A(t) v; if `dot` is given and the evaluator could fuse it, dot->n partials of <v, A v>
static hp_status apply_ham_full(const Hamiltonian& H, const double2* v, double2* y, double2* tmp, double2* ws,
                                size_t ws_bytes, cudaStream_t st, DotOut* dot = nullptr) {
  bool sq_done = false;
  hp_status rc = apply_ham(H, v, y, ws, ws_bytes, st, dot, &sq_done);
  if (rc) return rc;
  if (H.q != 0.0 && !sq_done) {
    rc = launch_square<double2>(H.s, v, tmp, 1, st);
    if (rc) return rc;
    int64_t n = H.s->n;
    k_axpy_c2<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(n, H.q, tmp, y);
    HP_LAUNCH_CHECK("k_axpy_c2");
  }
  return HP_OK;
}

// ---------------------------------------------------------------- workspace layout

struct LzLayout {
  size_t off_state, off_partial, off_dot, off_V, off_w, off_tmp, off_g, off_prog, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// `rows`: basis rows kept in the workspace (row 0 is the caller's vector)
static LzLayout lz_layout(const hp_set_s* s, int rows, int scheme, size_t prog_bytes) {
  LzLayout L;
  size_t vec = (size_t)s->n * 16;
  size_t o = 0;
  L.off_state = o; o = align_up(o + sizeof(LzState));
  L.off_partial = o; o = align_up(o + HP_RED_BLOCKS * sizeof(double2));
  L.off_dot = o; o = align_up(o + HP_DOT_CAPACITY * sizeof(double2));
  L.off_V = o; o = align_up(o + (size_t)std::max(rows, 0) * vec);
  L.off_w = o; o = align_up(o + vec);
  L.off_tmp = o; o = align_up(o + vec);
  L.off_g = o; o = align_up(o + (scheme == 1 ? 4 * vec : 0));
  L.off_prog = o; o = align_up(o + prog_bytes);
  L.total = o;
  return L;
}

static size_t prog_bytes_for(const hp_set_s* s, const std::vector<Term>& terms) {
  Program p = build_program(s->dim, terms, HP_ADD_OSC, nullptr);
  size_t gen = (size_t)std::max(p.nslots, 1) * s->n * 16;
  size_t fg = fullgrid_workspace_bytes(s, terms, HP_C128, 1, HP_ADD_OSC);
  size_t lv = level_workspace_bytes(s, terms, HP_C128, 1);
  return std::max(std::max(gen, fg), lv);
}

// Scaled Lanczos recurrence (krylov_propagator.py:58-104) for `steps`
// iterations.  w0 = starting vector (row 0, read only); rows 1..steps-1 are
// written unnormalised into `rows`.  Per iteration: one matvec (with the
// <w_k, A w_k> partials fused into its last kernel when possible), one fused
// update + norm kernel and two tiny finalisers.  Fully asynchronous on `st`.
template <class MV>
static hp_status run_lanczos(const hp_set_s* s, MV&& matvec, const double2* w0, double2* rows, int steps,
                             bool reorth, LzState* state, double2* partial, double2* dotbuf, double2* z,
                             cudaStream_t st) {
  int64_t n = s->n;
  int g = grid_for(n, 256, 148 * 16);
  auto row = [&](int k) -> double2* { return k == 0 ? const_cast<double2*>(w0) : rows + (int64_t)(k - 1) * n; };
  k_lz_init<<<1, 32, 0, st>>>(state, steps);
  HP_LAUNCH_CHECK("k_lz_init");
  hp_status rc = reduce(1, n, w0, nullptr, partial, state, 0, 1, 0.0, nullptr, st);  // nrm0, scale_0
  if (rc) return rc;
  for (int k = 0; k < steps; ++k) {
    const double2* wk = row(k);
    DotOut dot;
    dot.partial = dotbuf;
    dot.capacity = HP_DOT_CAPACITY;
    rc = matvec(wk, z, &dot);
    if (rc) return rc;
    if (dot.n > 0) {
      k_red_final<<<1, HP_RED_THREADS, 0, st>>>(dotbuf, dot.n, state, k, 6, 0.0, nullptr);  // alpha_k
      HP_LAUNCH_CHECK("k_red_final");
    } else {
      rc = reduce(0, n, wk, z, partial, state, k, 6, 0.0, nullptr, st);
      if (rc) return rc;
    }
    if (k == steps - 1) break;
    double2* wn = row(k + 1);
    k_lz_update_s<<<HP_RED_BLOCKS, HP_RED_THREADS, 0, st>>>(n, z, wk, k > 0 ? row(k - 1) : wk, wn, state, k,
                                                           partial);
    HP_LAUNCH_CHECK("k_lz_update_s");
    if (!reorth) {
      k_red_final<<<1, HP_RED_THREADS, 0, st>>>(partial, HP_RED_BLOCKS, state, k, 7, 1e-14, nullptr);  // beta_k
      HP_LAUNCH_CHECK("k_red_final");
    } else {
      for (int j = 0; j <= k; ++j) {
        rc = reduce(0, n, row(j), wn, partial, state, j, 8, 0.0, nullptr, st);
        if (rc) return rc;
      }
      k_lz_reorth_s<<<g, 256, 0, st>>>(n, wn, w0, rows, state, k);
      HP_LAUNCH_CHECK("k_lz_reorth_s");
      rc = reduce(1, n, wn, nullptr, partial, state, k, 7, 1e-14, nullptr, st);
      if (rc) return rc;
    }
  }
  return HP_OK;
}

static hp_status check_m(int m) {
  if (m < 1) return fail(HP_ERR_VALUE, "steps must be at least 1");
  if (m > HP_MAXM) return fail(HP_ERR_VALUE, "krylov_steps exceeds the device limit of 48");
  return HP_OK;
}

}  // namespace hp

using namespace hp;

// ---------------------------------------------------------------- sharded Lanczos building blocks

// out = a x + b y + c z (z optional) with the per-block partial sums of ||out||^2: the update
// r = A v_k - alpha_k v_k - beta_{k-1} v_{k-1} (krylov_propagator.py:86-89) on one rank's owned
// planes, its norm reduced across ranks by the caller (sharding.sharded_propagate)
__global__ void __launch_bounds__(HP_RED_THREADS) k_lincomb3_part(int64_t n, double a, const double2* __restrict__ x,
                                                                  double b, const double2* __restrict__ y, double c,
                                                                  const double2* __restrict__ z,
                                                                  double2* __restrict__ out,
                                                                  double2* __restrict__ partial) {
  __shared__ double2 sh[HP_RED_THREADS];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 xv = __ldg(x + i), yv = __ldg(y + i);
    double2 r = make_double2(fma(b, yv.x, a * xv.x), fma(b, yv.y, a * xv.y));
    if (z) {
      const double2 zv = __ldg(z + i);
      r.x = fma(c, zv.x, r.x);
      r.y = fma(c, zv.y, r.y);
    }
    out[i] = r;
    acc.x = fma(r.x, r.x, fma(r.y, r.y, acc.x));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = HP_RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

constexpr int HP_LINCOMB_MAX = 32;
struct LinCombArgs {
  const double2* v[HP_LINCOMB_MAX];
  double2 c[HP_LINCOMB_MAX];
  int m;
};
// out = sum_k c_k V_k: the basis combine of lanczos_exp_apply (krylov_propagator.py:180-186)
__global__ void k_lincomb(int64_t n, LinCombArgs A, double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < A.m; ++k) {
      const double2 v = __ldg(A.v[k] + i), c = A.c[k];
      acc.x = fma(c.x, v.x, fma(-c.y, v.y, acc.x));
      acc.y = fma(c.x, v.y, fma(c.y, v.x, acc.y));
    }
    out[i] = acc;
  }
}

extern "C" {

size_t hp_reduce_workspace_bytes(int64_t n) {
  (void)n;
  return align_up(HP_RED_BLOCKS * sizeof(double2)) + align_up(sizeof(LzState));
}

hp_status hp_lincomb3_nrm2sq(int64_t n, double a, const void* x, double b, const void* y, double c, const void* z,
                             void* out, double* norm2_out, void* ws, void* stream) {
  if (n < 0 || !x || !y || !out || !norm2_out || !ws) return fail(HP_ERR_VALUE, "lincomb3: null buffer");
  cudaStream_t st = as_stream(stream);
  k_lincomb3_part<<<HP_RED_BLOCKS, HP_RED_THREADS, 0, st>>>(n, a, (const double2*)x, b, (const double2*)y, c,
                                                             (const double2*)z, (double2*)out, (double2*)ws);
  HP_LAUNCH_CHECK("k_lincomb3_part");
  k_red_final<<<1, HP_RED_THREADS, 0, st>>>((double2*)ws, HP_RED_BLOCKS, nullptr, 0, 4, 0.0, norm2_out);
  HP_LAUNCH_CHECK("k_red_final");
  return HP_OK;
}

hp_status hp_lincomb(int64_t n, int m, const void* const* vecs, const double* coef, void* out, void* stream) {
  if (n < 0 || m < 1 || m > HP_LINCOMB_MAX || !vecs || !coef || !out) return fail(HP_ERR_VALUE, "lincomb: bad arguments");
  LinCombArgs A;
  A.m = m;
  for (int k = 0; k < m; ++k) {
    A.v[k] = (const double2*)vecs[k];
    A.c[k] = make_double2(coef[2 * k], coef[2 * k + 1]);
  }
  k_lincomb<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, A, (double2*)out);
  HP_LAUNCH_CHECK("k_lincomb");
  return HP_OK;
}

hp_status hp_cdot(int64_t n, const void* a, const void* b, double* out, void* ws, void* stream) {
  cudaStream_t st = as_stream(stream);
  return reduce(0, n, (const double2*)a, (const double2*)b, (double2*)ws, nullptr, 0, 4, 0.0, out, st);
}

hp_status hp_cnrm2(int64_t n, const void* a, double* out, void* ws, void* stream) {
  cudaStream_t st = as_stream(stream);
  return reduce(1, n, (const double2*)a, nullptr, (double2*)ws, nullptr, 0, 5, 0.0, out, st);
}

// ---- device-resident Lanczos scalars for distributed callers (sharding.sharded_propagate)

size_t hp_lz_state_bytes(void) { return sizeof(LzState); }

hp_status hp_lz_init(void* state_dev, int m, void* stream) {
  hp_status rc = check_m(m);
  if (rc) return rc;
  k_lz_init<<<1, 32, 0, as_stream(stream)>>>((LzState*)state_dev, m);
  HP_LAUNCH_CHECK("k_lz_init");
  return HP_OK;
}

hp_status hp_lz_set(void* state_dev, int k, int what, const double* value_dev, double tol, void* stream) {
  if (!state_dev || !value_dev || k < 0 || k >= HP_MAXM) return fail(HP_ERR_VALUE, "lz_set: bad arguments");
  if (what != 1 && what != 6 && what != 7) return fail(HP_ERR_VALUE, "lz_set: what must be 1, 6 or 7");
  k_lz_set<<<1, 32, 0, as_stream(stream)>>>(value_dev, (LzState*)state_dev, k, what, tol);
  HP_LAUNCH_CHECK("k_lz_set");
  return HP_OK;
}

hp_status hp_lz_update(int64_t n, const void* z, const void* wk, const void* wkm1, void* wn, const void* state_dev,
                       int k, double* nrm2_out_dev, void* ws, void* stream) {
  if (n < 0 || !z || !wk || !wn || !state_dev || !nrm2_out_dev || !ws || (k > 0 && !wkm1))
    return fail(HP_ERR_VALUE, "lz_update: null buffer");
  cudaStream_t st = as_stream(stream);
  k_lz_update_s<<<HP_RED_BLOCKS, HP_RED_THREADS, 0, st>>>(n, (const double2*)z, (const double2*)wk,
                                                           (const double2*)wkm1, (double2*)wn,
                                                           (const LzState*)state_dev, k, (double2*)ws);
  HP_LAUNCH_CHECK("k_lz_update_s");
  k_red_final<<<1, HP_RED_THREADS, 0, st>>>((double2*)ws, HP_RED_BLOCKS, nullptr, 0, 4, 0.0, nrm2_out_dev);
  HP_LAUNCH_CHECK("k_red_final");
  return HP_OK;
}

hp_status hp_lz_expm(void* state_dev, double tau, void* stream) {
  k_lz_expm<<<1, 32, 0, as_stream(stream)>>>((LzState*)state_dev, tau);
  HP_LAUNCH_CHECK("k_lz_expm");
  return HP_OK;
}

hp_status hp_lz_combine(int64_t n, int m, const void* const* vecs_host, const void* state_dev, void* out,
                        void* stream) {
  hp_status rc = check_m(m);
  if (rc) return rc;
  if (!vecs_host || !state_dev || !out) return fail(HP_ERR_VALUE, "lz_combine: null buffer");
  LzPtrs P{};
  for (int k = 0; k < m; ++k) P.v[k] = (const double2*)vecs_host[k];
  k_lz_combine_ptrs<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, P, (const LzState*)state_dev,
                                                                     (double2*)out);
  HP_LAUNCH_CHECK("k_lz_combine_ptrs");
  return HP_OK;
}

hp_status hp_lz_diag(const void* state_dev, double* diag_dev, double* alpha_dev, double* beta_dev, void* stream) {
  k_lz_diag<<<1, 32, 0, as_stream(stream)>>>((const LzState*)state_dev, diag_dev, alpha_dev, beta_dev);
  HP_LAUNCH_CHECK("k_lz_diag");
  return HP_OK;
}

hp_status hp_expm_tridiag_column(const double* alpha, const double* beta, int m, double tau, void* col,
                                 int* status, void* stream) {
  hp_status rc = check_m(m);
  if (rc) return rc;
  k_expm_standalone<<<1, 32, 0, as_stream(stream)>>>(alpha, beta, m, tau, (double2*)col, status);
  HP_LAUNCH_CHECK("k_expm_standalone");
  return HP_OK;
}

hp_status hp_tridiag_eigh(const double* alpha, const double* beta, int m, double* d, double* z, int* status,
                          void* stream) {
  hp_status rc = check_m(m);
  if (rc) return rc;
  k_tridiag_eigh<<<1, 32, 0, as_stream(stream)>>>(alpha, beta, m, d, z, status);
  HP_LAUNCH_CHECK("k_tridiag_eigh");
  return HP_OK;
}

size_t hp_magnus_workspace_bytes(hp_set_t s, int scheme, const int32_t* d1, int n1, const int32_t* d2, int n2,
                                 int m) {
  if (!s) return 0;
  std::vector<double> ones(std::max(n1, n2) + 1, 1.0);
  size_t pb = prog_bytes_for(s, make_terms(s->dim, d1, ones.data(), n1));
  if (scheme == 1 && d2) pb = std::max(pb, prog_bytes_for(s, make_terms(s->dim, d2, ones.data(), n2)));
  return lz_layout(s, m - 1, scheme, pb).total;
}

hp_status hp_magnus_step(hp_set_t s, int scheme, const int32_t* d1, const double* c1, int n1, const int32_t* d2,
                         const double* c2, int n2, double halfwidth, double q, double h, int m, int reorth,
                         void* y, double* diag, void* ws, size_t ws_bytes, void* stream) {
  HP_NVTX("hp_magnus_step");
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  hp_status rc = check_m(m);
  if (rc) return rc;
  if (scheme != 0 && scheme != 1) return fail(HP_ERR_VALUE, "unknown scheme");
  if (!(halfwidth > 0)) return fail(HP_ERR_VALUE, "halfwidth must be positive");
  cudaStream_t st = as_stream(stream);
  int64_t n = s->n;
  Hamiltonian H1{s, {}, halfwidth, q, make_terms(s->dim, d1, c1, n1)};
  H1.prog = build_program(s->dim, H1.terms, HP_ADD_OSC, nullptr);
  Hamiltonian H2{s, {}, halfwidth, q, {}};
  size_t pb = prog_bytes_for(s, H1.terms);
  if (scheme == 1) {
    H2.terms = make_terms(s->dim, d2, c2, n2);
    H2.prog = build_program(s->dim, H2.terms, HP_ADD_OSC, nullptr);
    pb = std::max(pb, prog_bytes_for(s, H2.terms));
  }
  LzLayout L = lz_layout(s, m - 1, scheme, pb);
  if (ws_bytes < L.total) return fail(HP_ERR_NOMEM, "workspace too small for hp_magnus_step");
  char* base = (char*)ws;
  LzState* state = (LzState*)(base + L.off_state);
  double2* partial = (double2*)(base + L.off_partial);
  double2* dotbuf = (double2*)(base + L.off_dot);
  double2* V = (double2*)(base + L.off_V);
  double2* w = (double2*)(base + L.off_w);
  double2* tmp = (double2*)(base + L.off_tmp);
  double2* g = (double2*)(base + L.off_g);
  double2* pws = (double2*)(base + L.off_prog);
  size_t pws_bytes = L.total - L.off_prog;
  double2* yv = (double2*)y;
  double gamma = std::sqrt(3.0) / 12.0 * h;
  if (scheme == 0 && q == 0.0 && !reorth) {
    // small sets: the whole step in one launch (hp_small.cuh)
    bool done = false;
    rc = small_magnus_step(s, H1.prog, halfwidth, h, m, yv, diag, V, w, pws, pws_bytes, st, &done);
    if (rc || done) return rc;
  }
  auto mv = [&](const double2* v, double2* out, DotOut* dot) -> hp_status {
    if (scheme == 0) return apply_ham_full(H1, v, out, tmp, pws, pws_bytes, st, dot);
    double2 *y1 = g, *y2 = g + n, *z2 = g + 2 * n, *z1 = g + 3 * n;
    hp_status r;
    if ((r = apply_ham_full(H1, v, y1, tmp, pws, pws_bytes, st))) return r;
    if ((r = apply_ham_full(H2, v, y2, tmp, pws, pws_bytes, st))) return r;
    if ((r = apply_ham_full(H2, y1, z2, tmp, pws, pws_bytes, st))) return r;
    if ((r = apply_ham_full(H1, y2, z1, tmp, pws, pws_bytes, st))) return r;
    const int gg = grid_for(n, 256, 148 * 16);
    const bool fuse = dot && dot->partial && gg <= dot->capacity;
    k_gl2_combine<<<gg, 256, 0, st>>>(n, y1, y2, z2, z1, gamma, out, v, fuse ? dot->partial : nullptr);
    HP_LAUNCH_CHECK("k_gl2_combine");
    if (fuse) dot->n = gg;
    return HP_OK;
  };
  rc = run_lanczos(s, mv, yv, V, m, reorth != 0, state, partial, dotbuf, w, st);
  if (rc) return rc;
  k_lz_expm<<<1, 32, 0, st>>>(state, h);
  HP_LAUNCH_CHECK("k_lz_expm");
  k_lz_combine_s<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(n, yv, V, state, yv);
  HP_LAUNCH_CHECK("k_lz_combine_s");
  if (diag) {
    k_lz_diag<<<1, 32, 0, st>>>(state, diag, nullptr, nullptr);
    HP_LAUNCH_CHECK("k_lz_diag");
  }
  return HP_OK;
}

hp_status hp_lanczos(hp_set_t s, const int32_t* d, const double* c, int nterms, double halfwidth, double q,
                     const void* v0, int steps, int reorth, void* basis, double* alpha, double* beta, double* diag,
                     void* ws, size_t ws_bytes, void* stream) {
  HP_NVTX("hp_lanczos");
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  hp_status rc = check_m(steps);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  Hamiltonian H{s, {}, halfwidth, q, make_terms(s->dim, d, c, nterms)};
  H.prog = build_program(s->dim, H.terms, HP_ADD_OSC, nullptr);
  LzLayout L = lz_layout(s, 0, 0, prog_bytes_for(s, H.terms));
  if (ws_bytes < L.total) return fail(HP_ERR_NOMEM, "workspace too small for hp_lanczos");
  char* base = (char*)ws;
  LzState* state = (LzState*)(base + L.off_state);
  double2* partial = (double2*)(base + L.off_partial);
  double2* dotbuf = (double2*)(base + L.off_dot);
  double2* w = (double2*)(base + L.off_w);
  double2* tmp = (double2*)(base + L.off_tmp);
  double2* pws = (double2*)(base + L.off_prog);
  size_t pws_bytes = L.total - L.off_prog;
  auto mv = [&](const double2* v, double2* out, DotOut* dot) -> hp_status {
    return apply_ham_full(H, v, out, tmp, pws, pws_bytes, st, dot);
  };
  double2* B = (double2*)basis;
  int64_t n = s->n;
  HP_CUDA(cudaMemcpyAsync(B, v0, (size_t)n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  rc = run_lanczos(s, mv, B, B + n, steps, reorth != 0, state, partial, dotbuf, w, st);
  if (rc) return rc;
  k_lz_normalize_rows<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(n, B, state);
  HP_LAUNCH_CHECK("k_lz_normalize_rows");
  k_lz_diag<<<1, 32, 0, st>>>(state, diag, alpha, beta);
  HP_LAUNCH_CHECK("k_lz_diag");
  return HP_OK;
}

}  // extern "C"
