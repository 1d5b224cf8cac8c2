// Single-launch Magnus step for small sets (cfg1 class: n <= 16384).
//
// For small bases the exponential step is launch-bound: ~100 dependent
// kernels per step (7 polynomial matvecs of ~10 ops each plus the Lanczos
// scalars) cost ~0.5 ms while moving < 1 MB.  This kernel runs the whole
// step in ONE cooperative CTA of 1024 threads: the polynomial program
// (same Op list as hp_apply.cu's suffix-trie evaluator, passed by value as a
// kernel parameter) is interpreted op by op with __syncthreads between
// dependent ops; vectors live in global memory but the ~240 KB working set
// stays in L1/L2; the Lanczos reductions are block reductions; the
// tridiagonal QL and exp(-i h T) e_1 run in thread 0.  Same scaled-Lanczos
// algebra as hp_krylov.cu.
// Included by hp_krylov.cu (shares its tridiagonal QL / expm device code).
#pragma once
#include <algorithm>

#include "hp_common.cuh"
#include "hp_program.h"

namespace hp {

constexpr int SM_MAXOPS = 96;
constexpr int SM_MAXM = 48;
constexpr int SM_THREADS = 1024;

struct SmallOp {
  signed char kind, axis, a, b, dst, acc;  // buffer ids: -2 = v (w_k), -1 = y (z), >= 0 slot
  double hw;
};

struct SmallProg {
  int nops;
  int nslots_hint;  // program slots staged in shared memory (use_smem)
  SmallOp ops[SM_MAXOPS];
};

template <class AXS>
struct SmallArgs {
  AXS axs;
  int dim;
  int64_t n;
  int m;
  double inv_L, two_L, h;
  SmallProg prog;
};

__device__ __forceinline__ double2 blk_sum(double2 v) {
  v = block_sum2(v);
  __shared__ double2 bcast;
  if (threadIdx.x == 0) bcast = v;
  __syncthreads();
  double2 r = bcast;
  __syncthreads();
  return r;
}

template <class AXS>
__global__ void __launch_bounds__(SM_THREADS, 1) k_small_magnus(SmallArgs<AXS> A, double2* __restrict__ y,
                                                                 double2* __restrict__ V, double2* __restrict__ z,
                                                                 double2* __restrict__ slots, double* diag,
                                                                 int use_smem, int use_tab, int jmax) {
  __shared__ double alpha[SM_MAXM], beta[SM_MAXM], scale[SM_MAXM];
  __shared__ double2 col[SM_MAXM];
  __shared__ int m_eff_sh, brk_sh, fail_sh;
  __shared__ double defect_sh;
  extern __shared__ double2 dyn[];  // [z | w_k | program slots] when use_smem
  const int64_t n = A.n;
  const int t = threadIdx.x;
  double2* zb = use_smem ? dyn : z;
  double2* wkb = dyn + n;
  double2* sb = use_smem ? dyn + 2 * n : slots;
  auto row = [&](int k) -> double2* { return k == 0 ? y : V + (int64_t)(k - 1) * n; };
  // use_tab: per (axis, point) orders and neighbours, and sqrt(j / 2) for j <= jmax + 1, in
  // shared memory after the vectors -- each X application then costs three table reads instead
  // of the index arithmetic and two FP64 square roots per point
  const size_t vec_bytes = use_smem ? (size_t)(A.prog.nslots_hint + 2) * n * sizeof(double2) : 0;
  int* jt = (int*)((char*)dyn + vec_bytes);
  int* dnt = jt + A.dim * n;
  int* upt = dnt + A.dim * n;
  double* sqt = (double*)(jt + (((size_t)3 * A.dim * n + 1) & ~(size_t)1));  // 8-byte aligned: 3 dim n may be odd
  if (use_tab) {
    for (int64_t o = t; o < n; o += SM_THREADS)
      for (int a = 0; a < A.dim; ++a) {
        int j;
        int64_t dn, up;
        A.axs.at(a, o, j, dn, up);
        jt[a * n + o] = j;
        dnt[a * n + o] = (int)dn;
        upt[a * n + o] = (int)up;
      }
    for (int j = t; j <= jmax + 1; j += SM_THREADS) sqt[j] = sqrt((double)j * 0.5);
    __syncthreads();
  }
  // nrm0
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = t; i < n; i += SM_THREADS) {
    double2 x = y[i];
    acc.x = fma(x.x, x.x, fma(x.y, x.y, acc.x));
  }
  const double nrm0 = sqrt(blk_sum(acc).x);
  if (t == 0) {
    scale[0] = 1.0 / nrm0;
    m_eff_sh = A.m;
    brk_sh = -1;
    defect_sh = 0.0;
    fail_sh = 0;
  }
  __syncthreads();
  int m_eff = A.m;
  for (int k = 0; k < A.m; ++k) {
    const double2* wk = row(k);
    if (use_smem) {  // stage w_k in shared memory next to z and the program slots
      for (int64_t i = t; i < n; i += SM_THREADS) wkb[i] = wk[i];
      __syncthreads();
      wk = wkb;
    }
    auto buf = [&](int id) -> double2* {
      if (id == -2) return const_cast<double2*>(wk);
      if (id == -1) return zb;
      return sb + (int64_t)id * n;
    };
    // ---- z = A w_k: interpret the polynomial program
    for (int oi = 0; oi < A.prog.nops; ++oi) {
      const SmallOp op = A.prog.ops[oi];
      double2* dst = buf(op.dst);
      if (op.kind == OP_ZERO) {
        for (int64_t i = t; i < n; i += SM_THREADS) dst[i] = make_double2(0.0, 0.0);
      } else if (op.kind == OP_COPY) {
        const double2* src = buf(op.a);
        for (int64_t i = t; i < n; i += SM_THREADS) dst[i] = src[i];
      } else if (op.kind == OP_AXPY) {
        const double2* src = buf(op.a);
        for (int64_t i = t; i < n; i += SM_THREADS) {
          double2 x = src[i];
          dst[i] = make_double2(fma(op.hw, x.x, dst[i].x), fma(op.hw, x.y, dst[i].y));
        }
      } else if (op.kind == OP_FIRST || op.kind == OP_STEP) {
        const bool step = op.kind == OP_STEP;
        const double2* w = buf(step ? op.b : op.a);
        const double2* wm = step ? buf(op.a) : nullptr;
        double2* accb = op.acc != -100 ? buf(op.acc) : nullptr;
        const double sc = step ? A.two_L : A.inv_L;
        for (int64_t o = t; o < n; o += SM_THREADS) {
          int j;
          int64_t dn, up;
          double cd, cu;
          if (use_tab) {
            j = jt[op.axis * n + o];
            dn = dnt[op.axis * n + o];
            up = upt[op.axis * n + o];
            cd = sqt[j];
            cu = sqt[j + 1];
          } else {
            A.axs.at(op.axis, o, j, dn, up);
            cd = sqrt((double)j * 0.5), cu = sqrt(((double)j + 1.0) * 0.5);
          }
          double2 wd = dn >= 0 ? w[dn] : make_double2(0.0, 0.0);
          double2 wu = up >= 0 ? w[up] : make_double2(0.0, 0.0);
          double2 r = make_double2(sc * fma(cd, wd.x, cu * wu.x), sc * fma(cd, wd.y, cu * wu.y));
          if (step) {
            r.x -= wm[o].x;
            r.y -= wm[o].y;
          }
          dst[o] = r;
          if (accb) accb[o] = make_double2(fma(op.hw, r.x, accb[o].x), fma(op.hw, r.y, accb[o].y));
        }
      } else if (op.kind == OP_OSC) {
        const double2* src = buf(op.a);
        for (int64_t o = t; o < n; o += SM_THREADS) {
          double lev = 0.0;
          for (int a = 0; a < A.dim; ++a) lev += (double)(use_tab ? jt[a * n + o] : A.axs.j(a, o)) + 0.5;
          double2 x = src[o];
          dst[o] = make_double2(fma(lev, x.x, dst[o].x), fma(lev, x.y, dst[o].y));
        }
      }
      __syncthreads();
    }
    // ---- alpha_k = s_k^2 <w_k, z>
    acc = make_double2(0.0, 0.0);
    for (int64_t i = t; i < n; i += SM_THREADS) cdot_acc(wk[i], zb[i], acc);
    double2 d = blk_sum(acc);
    const double sk = scale[k];
    if (t == 0) {
      alpha[k] = sk * sk * d.x;
      defect_sh = fmax(defect_sh, fabs(sk * sk * d.y));
    }
    __syncthreads();
    if (k == A.m - 1) break;
    // ---- w_{k+1} = s_k z - alpha_k s_k w_k - beta_{k-1} s_{k-1} w_{k-1}, and its norm
    const double ca = alpha[k] * sk;
    const double cb = k > 0 ? beta[k - 1] * scale[k - 1] : 0.0;
    const double2* wkm1 = k > 0 ? row(k - 1) : wk;
    double2* wn = row(k + 1);
    acc = make_double2(0.0, 0.0);
    for (int64_t i = t; i < n; i += SM_THREADS) {
      double2 a = zb[i], b = wk[i], c = wkm1[i];
      double2 r = make_double2(fma(sk, a.x, -ca * b.x), fma(sk, a.y, -ca * b.y));
      r.x = fma(-cb, c.x, r.x);
      r.y = fma(-cb, c.y, r.y);
      wn[i] = r;
      acc.x = fma(r.x, r.x, fma(r.y, r.y, acc.x));
    }
    const double bk = sqrt(blk_sum(acc).x);
    if (bk <= 1e-14) {  // breakdown (krylov_propagator.py:90-93)
      m_eff = k + 1;
      if (t == 0) {
        m_eff_sh = k + 1;
        brk_sh = k + 1;
      }
      __syncthreads();
      break;
    }
    if (t == 0) {
      beta[k] = bk;
      scale[k + 1] = 1.0 / bk;
    }
    __syncthreads();
  }
  // ---- exp(-i h T) e_1 and the combine
  if (t < 32) {  // warp 0
    const bool ok = expm_col_warp(m_eff, alpha, beta, A.h, col);
    if (t == 0 && !ok) fail_sh = 1;
  }
  __syncthreads();
  for (int64_t i = t; i < n; i += SM_THREADS) {
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < m_eff; ++k) {
      double2 v = row(k)[i];
      double2 c = make_double2(col[k].x * scale[k], col[k].y * scale[k]);
      s.x += v.x * c.x - v.y * c.y;
      s.y += v.x * c.y + v.y * c.x;
    }
    y[i] = make_double2(nrm0 * s.x, nrm0 * s.y);
  }
  if (t == 0 && diag) {
    diag[0] = m_eff_sh;
    diag[1] = defect_sh;
    diag[2] = brk_sh;
    diag[3] = fail_sh;
  }
}

struct AllBoxS {
  AxBox ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return ax[a].jloc(o) + ax[a].joff; }
  __device__ __forceinline__ void at(int a, int64_t o, int& jj, int64_t& dn, int64_t& up) const {
    ax[a].at(o, jj, dn, up);
  }
};
struct AllTabS {
  AxTab ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return __ldg(ax[a].jv + o); }
  __device__ __forceinline__ void at(int a, int64_t o, int& jj, int64_t& dn, int64_t& up) const {
    ax[a].at(o, jj, dn, up);
  }
};

static bool to_small(const Program& p, SmallProg& sp) {
  if ((int)p.ops.size() > SM_MAXOPS || p.nslots > 120) return false;
  auto id = [](int b) -> int { return b == BUF_V ? -2 : (b == BUF_Y ? -1 : b - BUF_SLOT0); };
  sp.nops = (int)p.ops.size();
  sp.nslots_hint = std::max(p.nslots, 1);
  for (int i = 0; i < sp.nops; ++i) {
    const Op& o = p.ops[i];
    SmallOp& s = sp.ops[i];
    s.kind = (signed char)o.kind;
    s.axis = (signed char)o.axis;
    s.a = (signed char)(o.a == -100 ? -100 : id(o.a));
    s.b = (signed char)(o.b == -100 ? -100 : id(o.b));
    s.dst = (signed char)(o.dst == -100 ? -100 : id(o.dst));
    s.acc = (signed char)(o.acc == -100 ? -100 : id(o.acc));
    s.hw = o.hw;
  }
  return true;
}

// returns *done = false when the set / program does not qualify (caller runs
// the multi-kernel step).  V: m-1 rows, z: n, slots: program slots.
static hp_status small_magnus_step(const hp_set_s* s, const Program& p, double halfwidth, double h, int m,
                                   double2* y, double* diag, double2* V, double2* z, double2* slots,
                                   size_t slot_bytes, cudaStream_t st, bool* done) {
  *done = false;
  if (s->n > 16384 || m > SM_MAXM || s->n == 0) return HP_OK;
  if ((size_t)std::max(p.nslots, 1) * s->n * sizeof(double2) > slot_bytes) return HP_OK;
  SmallProg sp;
  if (!to_small(p, sp)) return HP_OK;
  // z, w_k and the program slots in shared memory when they fit (~0.2 us per op instead of ~2 us)
  size_t smem = (size_t)(std::max(p.nslots, 1) + 2) * s->n * sizeof(double2);
  if (smem > 200 * 1024) smem = 0;
  const int jmax = s->bound + 1;
  const size_t tab = (((size_t)s->dim * s->n * 3 + 1) & ~(size_t)1) * sizeof(int) + (size_t)(jmax + 2) * sizeof(double);
  const int use_tab = smem + tab <= 220 * 1024 ? 1 : 0;
  const size_t dyn = smem + (use_tab ? tab : 0);
  if (s->boxed) {
    SmallArgs<AllBoxS> A;
    for (int a = 0; a < s->dim; ++a) A.axs.ax[a] = s->box(a);
    A.dim = s->dim, A.n = s->n, A.m = m, A.inv_L = 1.0 / halfwidth, A.two_L = 2.0 / halfwidth, A.h = h, A.prog = sp;
    if (dyn) HP_CUDA(cudaFuncSetAttribute(k_small_magnus<AllBoxS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    k_small_magnus<AllBoxS><<<1, SM_THREADS, dyn, st>>>(A, y, V, z, slots, diag, smem ? 1 : 0, use_tab, jmax);
  } else {
    SmallArgs<AllTabS> A;
    for (int a = 0; a < s->dim; ++a) A.axs.ax[a] = s->tab(a);
    A.dim = s->dim, A.n = s->n, A.m = m, A.inv_L = 1.0 / halfwidth, A.two_L = 2.0 / halfwidth, A.h = h, A.prog = sp;
    if (dyn) HP_CUDA(cudaFuncSetAttribute(k_small_magnus<AllTabS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    k_small_magnus<AllTabS><<<1, SM_THREADS, dyn, st>>>(A, y, V, z, slots, diag, smem ? 1 : 0, use_tab, jmax);
  }
  HP_LAUNCH_CHECK("k_small_magnus");
  *done = true;
  return HP_OK;
}

}  // namespace hp
