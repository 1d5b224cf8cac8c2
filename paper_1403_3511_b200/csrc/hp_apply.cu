// Matrix-free Galerkin matvec on the device (reference: fast_apply.py).
//
// Element-parallel building blocks, each one sm_100a kernel:
//   coord   y = cdown*w[down] + cup*w[up]                 (fast_apply.py:59-65)
//   first   w+ = (1/L) X w                                (fast_apply.py:69-79)
//   step    s  = (2/L) X w+ - w-                          (fast_apply.py:81-92)
//   axpy    acc += c * x    (harvest / term accumulation, fast_apply.py:132-163, 191-192)
//   osc     acc += (sum_l j_l + 1/2) * v                  (fast_apply.py:195-198)
//   square  exact restricted sum_l x_l^2                  (fast_apply.py:202-245)
// first/step fuse an optional harvest (acc += c * result) so a shared
// single-axis sweep costs one pass per degree.
//
// Two evaluation programs are compiled on the host from the term list:
//   * REF_ORDER: the reference's own order of operations (constant term,
//     shared single-axis sweeps axis N..1, then per-term ordered products);
//     every rounding matches numpy, so the result is bit-identical to the
//     reference (tests pin this);
//   * default: a suffix trie over axes N..1.  Terms that share their
//     trailing degrees (r_{a+1..N}) share the vector T_{r_{a+1}}(X_{a+1})..
//     T_{r_N}(X_N) v, and each trie node runs ONE Chebyshev sweep up to the
//     largest degree its children need.  The product order inside every
//     term (axis N first) is unchanged, so on reduced sets the operator is
//     the reference's; only the summation order of the terms differs.
// Full cubes additionally dispatch to the fused line/slab kernels in
// hp_fullgrid.cu when the term structure allows it.
#include <algorithm>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "hp_common.cuh"
#include "hp_program.h"

namespace hp {

// ---------------------------------------------------------------- kernels

template <class T, class AX>
__global__ void k_coord(int64_t n, int64_t batch, AX ax, const T* __restrict__ in, T* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    int j;
    int64_t dn, up;
    ax.at(o, j, dn, up);
    double cd = __dsqrt_rn((double)j / 2.0);
    double cu = __dsqrt_rn(((double)j + 1.0) / 2.0);
    for (int64_t b = 0; b < batch; ++b) {
      const T* src = in + b * n;
      T wd = dn >= 0 ? ldg(src + dn) : zero_of(T());
      T wu = up >= 0 ? ldg(src + up) : zero_of(T());
      out[b * n + o] = sadd(smul(cd, wd), smul(cu, wu));
    }
  }
}

// MODE 0: out = scale * (X w)            (scale = 1/L)
// MODE 1: out = scale * (X w) - wm       (scale = 2/L)
// optional harvest: acc += hw * out
template <class T, class AX, int MODE>
__global__ void k_cheb(int64_t n, int64_t batch, AX ax, double scale, const T* __restrict__ w,
                       const T* __restrict__ wm, T* __restrict__ out, T* __restrict__ acc, double hw) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    int j;
    int64_t dn, up;
    ax.at(o, j, dn, up);
    double cd = __dsqrt_rn((double)j / 2.0);
    double cu = __dsqrt_rn(((double)j + 1.0) / 2.0);
    for (int64_t b = 0; b < batch; ++b) {
      const T* src = w + b * n;
      T wd = dn >= 0 ? ldg(src + dn) : zero_of(T());
      T wu = up >= 0 ? ldg(src + up) : zero_of(T());
      T r = sadd(smul(cd, wd), smul(cu, wu));
      r = smul(scale, r);
      if (MODE == 1) r = ssub(r, ldg(wm + b * n + o));
      out[b * n + o] = r;
      if (acc) acc[b * n + o] = sadd(acc[b * n + o], smul(hw, r));
    }
  }
}

template <class T>
__global__ void k_axpy(int64_t total, double c, const T* __restrict__ x, T* __restrict__ acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    acc[i] = sadd(acc[i], smul(c, ldg(x + i)));
}

template <class T, class AXS>
__global__ void k_osc(int64_t n, int64_t batch, int dim, AXS axs, const T* __restrict__ v, T* __restrict__ acc) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    double lev = 0.0;  // sum of half-integers: exact in any order
    for (int a = 0; a < dim; ++a) lev += (double)axs.j(a, o) + 0.5;
    for (int64_t b = 0; b < batch; ++b) acc[b * n + o] = sadd(acc[b * n + o], smul(lev, ldg(v + b * n + o)));
  }
}

// acc += levels * v, and one partial of <v, acc_new> per CTA (Lanczos alpha, fused)
template <class AXS>
__global__ void k_osc_dot(int64_t n, int dim, AXS axs, const double2* __restrict__ v, double2* __restrict__ acc,
                          double2* __restrict__ partial) {
  double2 d = make_double2(0.0, 0.0);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    double lev = 0.0;
    for (int a = 0; a < dim; ++a) lev += (double)axs.j(a, o) + 0.5;
    double2 x = ldg(v + o);
    double2 y = sadd(acc[o], smul(lev, x));
    acc[o] = y;
    cdot_acc(x, y, d);
  }
  d = block_sum2(d);
  if (threadIdx.x == 0) partial[blockIdx.x] = d;
}

template <class T>
__global__ void k_nonfinite(int64_t total, const T* __restrict__ x, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !sfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// exact restricted sum_l x_l^2 (fast_apply.py:229-245), reference order
template <class T, class AXS>
__global__ void k_square(int64_t n, int64_t batch, int dim, AXS axs, const T* __restrict__ v, T* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    double lev = 0.0;
    for (int a = 0; a < dim; ++a) lev += (double)axs.j(a, o) + 0.5;
    for (int64_t b = 0; b < batch; ++b) {
      const T* src = v + b * n;
      T acc = smul(lev, ldg(src + o));
      for (int a = 0; a < dim; ++a) {
        int j, j2;
        int64_t dn, up, dn2, up2, t;
        axs.at(a, o, j, dn, up);
        dn2 = -1;
        up2 = -1;
        if (dn >= 0) axs.at(a, dn, j2, dn2, t);
        if (up >= 0) axs.at(a, up, j2, t, up2);
        double jl = (double)j;
        double cd2 = __dsqrt_rn(__dmul_rn(jl, __dsub_rn(jl, 1.0))) / 2.0;
        double cu2 = __dsqrt_rn(__dmul_rn(__dadd_rn(jl, 1.0), __dadd_rn(jl, 2.0))) / 2.0;
        T wd = dn2 >= 0 ? ldg(src + dn2) : zero_of(T());
        T wu = up2 >= 0 ? ldg(src + up2) : zero_of(T());
        acc = sadd(acc, smul(cd2, wd));
        acc = sadd(acc, smul(cu2, wu));
      }
      out[b * n + o] = acc;
    }
  }
}

// all-axis views for the osc / square kernels
struct AllBox {
  AxBox ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return ax[a].jloc(o) + ax[a].joff; }
  __device__ __forceinline__ void at(int a, int64_t o, int& jj, int64_t& dn, int64_t& up) const {
    ax[a].at(o, jj, dn, up);
  }
};
struct AllTab {
  AxTab ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return __ldg(ax[a].jv + o); }
  __device__ __forceinline__ void at(int a, int64_t o, int& jj, int64_t& dn, int64_t& up) const {
    ax[a].at(o, jj, dn, up);
  }
};

// ---------------------------------------------------------------- launchers

static int g_blocks(int64_t n) { return grid_for(n, 256, 148 * 16); }

// workspace cap per call of the generic program; batches beyond it are chunked
// batched workspaces are capped (HP_CHUNK_GB overrides, GiB): larger chunks let the level
// kernels share each point's line walk across more vectors of the batch
static size_t chunk_cap() {
  static size_t v = [] {
    const char* e = getenv("HP_CHUNK_GB");
    // cfg5, round-1 plans: 24 GiB 830 ms, 48 GiB 795, 64 GiB 801; merged plans (24 slots): 32 GiB 729 ms,
    // 48 737, 64 744, 96 779 (profiles/r2/sweep_level.txt)
    return (size_t)(e ? std::max(1, atoi(e)) : 32) << 30;
  }();
  return v;
}
#define kChunkCap chunk_cap()

template <class T>
static hp_status launch_cheb(const hp_set_s* s, int a, int mode, double scale, const T* w, const T* wm,
                             T* out, T* acc, double hw, int64_t batch, cudaStream_t st) {
  int64_t n = s->n;
  if (n == 0) return HP_OK;
  if (s->boxed) {
    if (mode == 0) k_cheb<T, AxBox, 0><<<g_blocks(n), 256, 0, st>>>(n, batch, s->box(a), scale, w, wm, out, acc, hw);
    else k_cheb<T, AxBox, 1><<<g_blocks(n), 256, 0, st>>>(n, batch, s->box(a), scale, w, wm, out, acc, hw);
  } else {
    if (mode == 0) k_cheb<T, AxTab, 0><<<g_blocks(n), 256, 0, st>>>(n, batch, s->tab(a), scale, w, wm, out, acc, hw);
    else k_cheb<T, AxTab, 1><<<g_blocks(n), 256, 0, st>>>(n, batch, s->tab(a), scale, w, wm, out, acc, hw);
  }
  HP_LAUNCH_CHECK("k_cheb");
  return HP_OK;
}

template <class T>
static hp_status launch_osc(const hp_set_s* s, const T* v, T* acc, int64_t batch, cudaStream_t st) {
  int64_t n = s->n;
  if (n == 0) return HP_OK;
  if (s->boxed) {
    AllBox ab;
    for (int a = 0; a < s->dim; ++a) ab.ax[a] = s->box(a);
    k_osc<T, AllBox><<<g_blocks(n), 256, 0, st>>>(n, batch, s->dim, ab, v, acc);
  } else {
    AllTab at;
    for (int a = 0; a < s->dim; ++a) at.ax[a] = s->tab(a);
    k_osc<T, AllTab><<<g_blocks(n), 256, 0, st>>>(n, batch, s->dim, at, v, acc);
  }
  HP_LAUNCH_CHECK("k_osc");
  return HP_OK;
}

template <class T>
hp_status launch_square(const hp_set_s* s, const T* v, T* out, int64_t batch, cudaStream_t st) {
  int64_t n = s->n;
  if (n == 0) return HP_OK;
  if (s->boxed) {
    AllBox ab;
    for (int a = 0; a < s->dim; ++a) ab.ax[a] = s->box(a);
    k_square<T, AllBox><<<g_blocks(n), 256, 0, st>>>(n, batch, s->dim, ab, v, out);
  } else {
    AllTab at;
    for (int a = 0; a < s->dim; ++a) at.ax[a] = s->tab(a);
    k_square<T, AllTab><<<g_blocks(n), 256, 0, st>>>(n, batch, s->dim, at, v, out);
  }
  HP_LAUNCH_CHECK("k_square");
  return HP_OK;
}
template hp_status launch_square<double>(const hp_set_s*, const double*, double*, int64_t, cudaStream_t);
template hp_status launch_square<double2>(const hp_set_s*, const double2*, double2*, int64_t, cudaStream_t);

// ---------------------------------------------------------------- programs

std::vector<Term> make_terms(int dim, const int32_t* degrees, const double* coeffs, int nterms) {
  std::vector<Term> t(nterms);
  for (int i = 0; i < nterms; ++i) {
    for (int a = 0; a < dim; ++a) t[i].r[a] = degrees[(int64_t)i * dim + a];
    t[i].alpha = coeffs[i];
  }
  return t;
}

// Reference order (fast_apply.py:110-193), buffer names emulated exactly.
static void build_ref_program(int dim, const std::vector<Term>& terms, const int32_t* axis_order,
                              Program& p) {
  // slots 0..2: wm wp sp; slot 3: mixed accumulator
  p.nslots = 4;
  p.ops.push_back(Op::zero(BUF_Y));
  auto ordered = [&](const std::vector<int>& rows, const std::vector<int>& order, int accbuf) {
    for (int it : rows) {
      int wm = 0, wp = 1, sp = 2;
      p.ops.push_back(Op::copy(slot(wm), BUF_V));
      for (int axis : order) {
        int deg = terms[it].r[axis - 1];
        if (deg == 0) continue;
        // _chebyshev_axis: first into wp, then deg-1 steps rotating
        p.ops.push_back(Op::first(axis - 1, slot(wm), slot(wp)));
        for (int s = 0; s < deg - 1; ++s) {
          p.ops.push_back(Op::step(axis - 1, slot(wm), slot(wp), slot(sp)));
          int t0 = wm; wm = wp; wp = sp; sp = t0;
        }
        std::swap(wm, wp);  // result becomes the next input
      }
      p.ops.push_back(Op::axpy(accbuf, slot(wm), terms[it].alpha));
    }
  };
  if (axis_order) {
    std::vector<int> rows(terms.size()), order(axis_order, axis_order + dim);
    for (size_t i = 0; i < terms.size(); ++i) rows[i] = (int)i;
    ordered(rows, order, BUF_Y);
    return;
  }
  std::vector<int> nact(terms.size(), 0);
  for (size_t i = 0; i < terms.size(); ++i)
    for (int a = 0; a < dim; ++a) nact[i] += terms[i].r[a] > 0;
  double c0 = 0.0;
  for (size_t i = 0; i < terms.size(); ++i) if (nact[i] == 0) c0 += terms[i].alpha;
  if (c0 != 0.0) p.ops.push_back(Op::axpy(BUF_Y, BUF_V, c0));
  int wm = 0, wp = 1, sp = 2;
  for (int axis = dim; axis >= 1; --axis) {
    std::map<int, double> wsum;
    bool any = false;
    for (size_t i = 0; i < terms.size(); ++i)
      if (nact[i] == 1 && terms[i].r[axis - 1] > 0) {
        any = true;
        int d = terms[i].r[axis - 1];
        wsum[d] = (wsum.count(d) ? wsum[d] : 0.0) + terms[i].alpha;
      }
    if (!any) continue;
    p.ops.push_back(Op::copy(slot(wm), BUF_V));
    Op f = Op::first(axis - 1, slot(wm), slot(wp));
    if (wsum.count(1)) f.acc = BUF_Y, f.hw = wsum[1];
    p.ops.push_back(f);
    int dmax = wsum.rbegin()->first;
    for (int d = 2; d <= dmax; ++d) {
      Op s = Op::step(axis - 1, slot(wm), slot(wp), slot(sp));
      if (wsum.count(d)) s.acc = BUF_Y, s.hw = wsum[d];
      p.ops.push_back(s);
      int t0 = wm; wm = wp; wp = sp; sp = t0;
    }
  }
  std::vector<int> mixed;
  for (size_t i = 0; i < terms.size(); ++i) if (nact[i] >= 2) mixed.push_back((int)i);
  if (!mixed.empty()) {
    std::vector<int> order;
    for (int a = dim; a >= 1; --a) order.push_back(a);
    p.ops.push_back(Op::zero(slot(3)));
    ordered(mixed, order, slot(3));
    p.ops.push_back(Op::axpy(BUF_Y, slot(3), 1.0));
  }
}

// Suffix-trie program: node vectors are never copied; every trie level owns
// a rotating triple of slots.
struct TrieBuilder {
  int dim;
  const std::vector<Term>& terms;
  Program& p;
  int xapps = 0;
  void node(int ubuf, int a, const std::vector<int>& rows) {
    // leaves: all remaining degrees (axes 0..a) zero
    std::vector<int> rest;
    for (int it : rows) {
      bool leaf = true;
      for (int l = 0; l <= a; ++l) leaf &= terms[it].r[l] == 0;
      if (leaf) p.ops.push_back(Op::axpy(BUF_Y, ubuf, terms[it].alpha));
      else rest.push_back(it);
    }
    if (rest.empty()) return;
    std::map<int, std::vector<int>> groups;
    for (int it : rest) groups[terms[it].r[a]].push_back(it);
    if (groups.count(0)) node(ubuf, a - 1, groups[0]);
    int kmax = groups.rbegin()->first;
    if (kmax == 0) return;
    int depth = dim - 1 - a;
    int A = slot(3 * depth), B = slot(3 * depth + 1), C = slot(3 * depth + 2);
    p.nslots = std::max(p.nslots, 3 * depth + 3);
    int prev = ubuf, cur = A;
    for (int k = 1; k <= kmax; ++k) {
      int dst;
      if (k == 1) dst = A;
      else {
        int bufs[3] = {A, B, C};
        dst = -1;
        for (int b : bufs) if (b != prev && b != cur) { dst = b; break; }
      }
      Op op = (k == 1) ? Op::first(a, ubuf, dst) : Op::step(a, prev, cur, dst);
      ++xapps;
      std::vector<int> nonleaf;
      auto g = groups.find(k);
      if (g != groups.end()) {
        double hw = 0.0;
        bool has = false;
        for (int it : g->second) {
          bool leaf = true;
          for (int l = 0; l < a; ++l) leaf &= terms[it].r[l] == 0;
          if (leaf) { hw += terms[it].alpha; has = true; }
          else nonleaf.push_back(it);
        }
        if (has) op.acc = BUF_Y, op.hw = hw;
      }
      p.ops.push_back(op);
      if (k > 1) prev = cur;
      cur = dst;
      if (!nonleaf.empty()) node(cur, a - 1, nonleaf);
    }
  }
};

Program build_program(int dim, const std::vector<Term>& terms, int flags, const int32_t* axis_order) {
  Program p;
  if ((flags & HP_REF_ORDER) || axis_order) {
    build_ref_program(dim, terms, axis_order, p);
  } else {
    p.ops.push_back(Op::zero(BUF_Y));
    std::vector<int> rows(terms.size());
    for (size_t i = 0; i < terms.size(); ++i) rows[i] = (int)i;
    TrieBuilder tb{dim, terms, p};
    if (!rows.empty()) tb.node(BUF_V, dim - 1, rows);
    p.xapps = tb.xapps;
  }
  if (flags & HP_ADD_OSC) p.ops.push_back(Op::osc(BUF_Y, BUF_V));
  return p;
}

template <class T>
static hp_status launch_osc_dot(const hp_set_s* s, const T* v, T* acc, DotOut* dot, cudaStream_t st) {
  if constexpr (std::is_same<T, double2>::value) {
    int64_t n = s->n;
    int g = std::min(g_blocks(n), dot->capacity);
    if (s->boxed) {
      AllBox ab;
      for (int a = 0; a < s->dim; ++a) ab.ax[a] = s->box(a);
      k_osc_dot<AllBox><<<g, 256, 0, st>>>(n, s->dim, ab, v, acc, dot->partial);
    } else {
      AllTab at;
      for (int a = 0; a < s->dim; ++a) at.ax[a] = s->tab(a);
      k_osc_dot<AllTab><<<g, 256, 0, st>>>(n, s->dim, at, v, acc, dot->partial);
    }
    HP_LAUNCH_CHECK("k_osc_dot");
    dot->n = g;
  }
  return HP_OK;
}

template <class T>
hp_status run_program(const hp_set_s* s, const Program& p, double halfwidth, const T* v, T* y,
                      int64_t batch, T* ws, size_t ws_bytes, cudaStream_t st, DotOut* dot) {
  if (dot) dot->n = 0;
  int64_t n = s->n;
  int64_t vec = n * batch;
  if ((size_t)p.nslots * vec * sizeof(T) > ws_bytes)
    return fail(HP_ERR_NOMEM, "workspace too small for the polynomial program");
  auto buf = [&](int id) -> T* {
    if (id == BUF_V) return const_cast<T*>(v);
    if (id == BUF_Y) return y;
    return ws + (int64_t)(id - BUF_SLOT0) * vec;
  };
  const double inv = 1.0 / halfwidth, two = 2.0 / halfwidth;
  for (const Op& op : p.ops) {
    hp_status rc = HP_OK;
    switch (op.kind) {
      case OP_ZERO:
        HP_CUDA(cudaMemsetAsync(buf(op.dst), 0, vec * sizeof(T), st));
        break;
      case OP_COPY:
        HP_CUDA(cudaMemcpyAsync(buf(op.dst), buf(op.a), vec * sizeof(T), cudaMemcpyDeviceToDevice, st));
        break;
      case OP_AXPY:
        if (vec) {
          k_axpy<T><<<g_blocks(vec), 256, 0, st>>>(vec, op.hw, buf(op.a), buf(op.dst));
          HP_LAUNCH_CHECK("k_axpy");
        }
        break;
      case OP_FIRST:
        rc = launch_cheb<T>(s, op.axis, 0, inv, buf(op.a), nullptr, buf(op.dst),
                            op.acc != -100 ? buf(op.acc) : nullptr, op.hw, batch, st);
        break;
      case OP_STEP:
        rc = launch_cheb<T>(s, op.axis, 1, two, buf(op.b), buf(op.a), buf(op.dst),
                            op.acc != -100 ? buf(op.acc) : nullptr, op.hw, batch, st);
        break;
      case OP_OSC:
        if (dot && dot->partial && batch == 1 && op.dst == BUF_Y && op.a == BUF_V && &op == &p.ops.back() &&
            std::is_same<T, double2>::value)
          rc = launch_osc_dot<T>(s, buf(op.a), buf(op.dst), dot, st);
        else
          rc = launch_osc<T>(s, buf(op.a), buf(op.dst), batch, st);
        break;
    }
    if (rc != HP_OK) return rc;
  }
  return HP_OK;
}
template hp_status run_program<double>(const hp_set_s*, const Program&, double, const double*, double*,
                                       int64_t, double*, size_t, cudaStream_t, DotOut*);
template hp_status run_program<double2>(const hp_set_s*, const Program&, double, const double2*, double2*,
                                        int64_t, double2*, size_t, cudaStream_t, DotOut*);

template <class T>
hp_status check_finite(const T* y, int64_t total, cudaStream_t st, bool* ok) {
  int* flag = nullptr;
  HP_CUDA(cudaMallocAsync(&flag, sizeof(int), st));
  HP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  if (total) {
    k_nonfinite<T><<<g_blocks(total), 256, 0, st>>>(total, y, flag);
    HP_LAUNCH_CHECK("k_nonfinite");
  }
  int h = 0;
  HP_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  HP_CUDA(cudaFreeAsync(flag, st));
  *ok = (h == 0);
  return HP_OK;
}

static hp_status check_set(hp_set_t s) {
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  return HP_OK;
}

static hp_status check_terms(hp_set_t s, const int32_t* degrees, int nterms, double halfwidth) {
  if (nterms < 0) return fail(HP_ERR_VALUE, "nterms must be nonnegative");
  if (!(halfwidth > 0.0)) return fail(HP_ERR_VALUE, "halfwidth must be positive");
  for (int64_t i = 0; i < (int64_t)nterms * s->dim; ++i)
    if (degrees[i] < 0) return fail(HP_ERR_VALUE, "negative Chebyshev degree in term list");
  return HP_OK;
}

}  // namespace hp

using namespace hp;

extern "C" {

hp_status hp_apply_coordinate(hp_set_t s, int axis, int dtype, const void* in, void* out, int64_t batch,
                              void* stream) {
  HP_NVTX("hp_apply_coordinate");
  hp_status rc = check_set(s);
  if (rc) return rc;
  if (axis < 1 || axis > s->dim)
    return fail(HP_ERR_VALUE, "axis must satisfy 1 <= axis <= " + std::to_string(s->dim) + ", got " +
                                  std::to_string(axis));
  cudaStream_t st = as_stream(stream);
  int64_t n = s->n;
  if (n == 0 || batch == 0) return HP_OK;
  int a = axis - 1;
  if (dtype == HP_C128) {
    if (s->boxed) k_coord<double2, AxBox><<<g_blocks(n), 256, 0, st>>>(n, batch, s->box(a), (const double2*)in, (double2*)out);
    else k_coord<double2, AxTab><<<g_blocks(n), 256, 0, st>>>(n, batch, s->tab(a), (const double2*)in, (double2*)out);
  } else {
    if (s->boxed) k_coord<double, AxBox><<<g_blocks(n), 256, 0, st>>>(n, batch, s->box(a), (const double*)in, (double*)out);
    else k_coord<double, AxTab><<<g_blocks(n), 256, 0, st>>>(n, batch, s->tab(a), (const double*)in, (double*)out);
  }
  HP_LAUNCH_CHECK("k_coord");
  return HP_OK;
}

size_t hp_cheb_workspace_bytes(hp_set_t s, int dtype, int64_t batch) {
  if (!s) return 0;
  return (size_t)3 * s->n * batch * (dtype == HP_C128 ? 16 : 8);
}

hp_status hp_cheb_apply(hp_set_t s, int axis, int degree, double halfwidth, int dtype, const void* in,
                        void* out, int64_t batch, void* ws, size_t ws_bytes, void* stream) {
  HP_NVTX("hp_cheb_apply");
  hp_status rc = check_set(s);
  if (rc) return rc;
  if (axis < 1 || axis > s->dim)
    return fail(HP_ERR_VALUE, "axis must satisfy 1 <= axis <= " + std::to_string(s->dim) + ", got " +
                                  std::to_string(axis));
  if (degree < 0) return fail(HP_ERR_VALUE, "degree must be nonnegative, got " + std::to_string(degree));
  if (!(halfwidth > 0)) return fail(HP_ERR_VALUE, "halfwidth must be positive");
  cudaStream_t st = as_stream(stream);
  size_t es = dtype == HP_C128 ? 16 : 8;
  int64_t vec = s->n * batch;
  if (degree == 0) {
    HP_CUDA(cudaMemcpyAsync(out, in, vec * es, cudaMemcpyDeviceToDevice, st));
    return HP_OK;
  }
  Term t;
  for (int a = 0; a < s->dim; ++a) t.r[a] = 0;
  t.r[axis - 1] = degree;
  t.alpha = 1.0;
  Program p;
  // cheb_of_coordinate_apply: one sweep, result = T_deg X v (no scaling)
  int wm = 0, wp = 1, sp = 2;
  p.nslots = 3;
  p.ops.push_back(Op::first(axis - 1, BUF_V, slot(wp)));
  wm = -1;  // wm is the input itself for the first advance
  int prev = BUF_V, cur = slot(wp);
  int bufs[3] = {slot(0), slot(1), slot(2)};
  for (int k = 2; k <= degree; ++k) {
    int dst = -1;
    for (int b : bufs) if (b != prev && b != cur) { dst = b; break; }
    p.ops.push_back(Op::step(axis - 1, prev, cur, dst));
    prev = cur;
    cur = dst;
  }
  (void)wm; (void)sp;
  if (ws_bytes < 3 * vec * es) return fail(HP_ERR_NOMEM, "workspace too small");
  if (dtype == HP_C128) rc = run_program<double2>(s, p, halfwidth, (const double2*)in, (double2*)out, batch, (double2*)ws, ws_bytes, st);
  else rc = run_program<double>(s, p, halfwidth, (const double*)in, (double*)out, batch, (double*)ws, ws_bytes, st);
  if (rc) return rc;
  // copy the result slot to out
  int64_t off = (int64_t)(cur - BUF_SLOT0) * vec;
  HP_CUDA(cudaMemcpyAsync(out, (char*)ws + off * es, vec * es, cudaMemcpyDeviceToDevice, st));
  return HP_OK;
}

size_t hp_poly_workspace_bytes(hp_set_t s, const int32_t* degrees, int nterms, int dtype, int64_t batch,
                               int flags) {
  if (!s || nterms < 0) return 0;
  std::vector<double> ones(nterms, 1.0);
  auto terms = make_terms(s->dim, degrees, ones.data(), nterms);
  Program p = build_program(s->dim, terms, flags, nullptr);
  int ns = std::max(p.nslots, 4);
  size_t fg = fullgrid_workspace_bytes(s, terms, dtype, batch, flags);
  size_t per_vec = (size_t)ns * s->n * (dtype == HP_C128 ? 16 : 8);
  // large batches run in chunks whose trie workspace stays below kChunkCap
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)(kChunkCap / std::max<size_t>(per_vec, 1))));
  size_t gen = per_vec * chunk;
  size_t lv = 0;
  if (!(flags & HP_REF_ORDER)) {
    // level-fused evaluator: its child vectors for one (chunk of the) batch
    size_t lv1 = level_workspace_bytes(s, terms, dtype, 1);
    if (lv1) lv = lv1 * std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)(kChunkCap / lv1)));
  }
  return std::max(std::max(gen, fg), lv);
}

hp_status hp_apply_polynomial(hp_set_t s, const int32_t* degrees, const double* coeffs, int nterms,
                              double halfwidth, int dtype, const void* in, void* out, int64_t batch,
                              int flags, const int32_t* axis_order, void* ws, size_t ws_bytes,
                              void* stream) {
  HP_NVTX("hp_apply_polynomial");
  hp_status rc = check_set(s);
  if (rc) return rc;
  if ((rc = check_terms(s, degrees, nterms, halfwidth))) return rc;
  if (axis_order) {
    std::vector<int> o(axis_order, axis_order + s->dim);
    std::sort(o.begin(), o.end());
    for (int a = 0; a < s->dim; ++a)
      if (o[a] != a + 1) return fail(HP_ERR_VALUE, "axis_order must permute 1.." + std::to_string(s->dim));
  }
  cudaStream_t st = as_stream(stream);
  if (s->n == 0 || batch == 0) return HP_OK;
  auto terms = make_terms(s->dim, degrees, coeffs, nterms);
  bool done = false;
  if (!(flags & HP_REF_ORDER) && !axis_order) {
    rc = fullgrid_apply_split(s, terms, halfwidth, dtype, in, out, batch, flags, ws, ws_bytes, st, &done);
    if (rc) return rc;
    if (!done) {
      rc = level_apply(s, terms, halfwidth, dtype, in, out, batch, flags, ws, ws_bytes, st, &done);
      if (rc) return rc;
    }
  }
  if (!done) {
    Program p = build_program(s->dim, terms, flags, axis_order);
    size_t es = dtype == HP_C128 ? 16 : 8;
    size_t per_vec = (size_t)std::max(p.nslots, 1) * s->n * es;
    int64_t chunk = std::min<int64_t>(batch, (int64_t)(ws_bytes / per_vec));
    if (chunk < 1) return fail(HP_ERR_NOMEM, "workspace too small for the polynomial program");
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
      int64_t nb = std::min(chunk, batch - b0);
      size_t off = (size_t)b0 * s->n * es;
      if (dtype == HP_C128)
        rc = run_program<double2>(s, p, halfwidth, (const double2*)((const char*)in + off),
                                  (double2*)((char*)out + off), nb, (double2*)ws, ws_bytes, st);
      else
        rc = run_program<double>(s, p, halfwidth, (const double*)((const char*)in + off), (double*)((char*)out + off),
                                 nb, (double*)ws, ws_bytes, st);
      if (rc) return rc;
    }
  }
  if (flags & HP_CHECK_FINITE) {
    bool ok = true;
    int64_t total = s->n * batch;
    if (dtype == HP_C128) rc = check_finite<double2>((const double2*)out, total, st, &ok);
    else rc = check_finite<double>((const double*)out, total, st, &ok);
    if (rc) return rc;
    if (!ok)
      return fail(HP_ERR_RUNTIME, (flags & HP_ADD_OSC)
                                      ? "Hamiltonian application produced non-finite values"
                                      : "fast application produced non-finite values; check surrogate "
                                        "coefficients and halfwidth");
  }
  return HP_OK;
}

hp_status hp_apply_polynomial_streamed(hp_set_t s, const int32_t* degrees, const double* coeffs, int nterms,
                                       double halfwidth, int dtype, const void* in_host, void* out_host,
                                       void* in_dev, void* out_dev, int64_t batch, int flags, void* ws,
                                       size_t ws_bytes, void* stream) {
  HP_NVTX("hp_apply_polynomial_streamed");
  hp_status rc = check_set(s);
  if (rc) return rc;
  if ((rc = check_terms(s, degrees, nterms, halfwidth))) return rc;
  if (!in_host || !out_host || !in_dev || !out_dev) return fail(HP_ERR_VALUE, "null buffer");
  cudaStream_t st = as_stream(stream);
  if (s->n == 0 || batch == 0) return HP_OK;
  const size_t bytes = (size_t)s->n * batch * (dtype == HP_C128 ? 16 : 8);
  if (batch == 1 && !(flags & (HP_REF_ORDER | HP_CHECK_FINITE))) {
    auto terms = make_terms(s->dim, degrees, coeffs, nterms);
    bool done = false;
    rc = fullgrid_apply_streamed(s, terms, halfwidth, dtype, in_host, out_host, in_dev, out_dev, flags, ws,
                                 ws_bytes, st, &done);
    if (rc || done) return rc;
  }
  // other sets / term structures: the batch streams through in groups of vectors (>= 32 MB
  // each): group k+1 is copied in and group k-1 out while group k is computed
  const size_t vbytes = bytes / batch;
  const int64_t g = std::min<int64_t>(batch, std::max<int64_t>(1, (int64_t)(((size_t)32 << 20) / vbytes)));
  const int64_t ng = (batch + g - 1) / g;
  if (ng == 1) {
    HP_CUDA(cudaMemcpyAsync(in_dev, in_host, bytes, cudaMemcpyHostToDevice, st));
    rc = hp_apply_polynomial(s, degrees, coeffs, nterms, halfwidth, dtype, in_dev, out_dev, batch, flags, nullptr,
                             ws, ws_bytes, stream);
    if (rc) return rc;
    HP_CUDA(cudaMemcpyAsync(out_host, out_dev, bytes, cudaMemcpyDeviceToHost, st));
    return HP_OK;
  }
  cudaStream_t sin, sout;
  if ((rc = copy_streams(&sin, &sout))) return rc;
  StreamedEvents ev;
  if ((rc = ev.create(2 * ng + 2))) return rc;
  ev.drain[0] = sin;
  ev.drain[1] = sout;
  HP_CUDA(cudaEventRecord(ev[2 * ng], st));  // after the caller's prior work
  HP_CUDA(cudaStreamWaitEvent(sin, ev[2 * ng], 0));
  HP_CUDA(cudaStreamWaitEvent(sout, ev[2 * ng], 0));
  for (int64_t k = 0; k < ng; ++k) {
    const int64_t b0 = k * g, nb = std::min(g, batch - b0);
    HP_CUDA(cudaMemcpyAsync((char*)in_dev + b0 * vbytes, (const char*)in_host + b0 * vbytes, nb * vbytes,
                            cudaMemcpyHostToDevice, sin));
    HP_CUDA(cudaEventRecord(ev[k], sin));
  }
  for (int64_t k = 0; k < ng; ++k) {
    const int64_t b0 = k * g, nb = std::min(g, batch - b0);
    HP_CUDA(cudaStreamWaitEvent(st, ev[k], 0));
    rc = hp_apply_polynomial(s, degrees, coeffs, nterms, halfwidth, dtype, (const char*)in_dev + b0 * vbytes,
                             (char*)out_dev + b0 * vbytes, nb, flags, nullptr, ws, ws_bytes, stream);
    if (rc) return rc;
    HP_CUDA(cudaEventRecord(ev[ng + k], st));
    HP_CUDA(cudaStreamWaitEvent(sout, ev[ng + k], 0));
    HP_CUDA(cudaMemcpyAsync((char*)out_host + b0 * vbytes, (const char*)out_dev + b0 * vbytes, nb * vbytes,
                            cudaMemcpyDeviceToHost, sout));
  }
  HP_CUDA(cudaEventRecord(ev[2 * ng + 1], sout));
  HP_CUDA(cudaStreamWaitEvent(st, ev[2 * ng + 1], 0));
  ev.committed = true;
  return HP_OK;
}

hp_status hp_apply_polynomial_planes_dot(hp_set_t s, const int32_t* degrees, const double* coeffs, int nterms,
                                         double halfwidth, int dtype, const void* in, void* out, int plane_lo,
                                         int plane_hi, int flags, double* dot_dev, void* ws, size_t ws_bytes,
                                         void* stream) {
  return hp_apply_hamiltonian_planes_dot(s, degrees, coeffs, nterms, halfwidth, 0.0, dtype, in, out, plane_lo,
                                         plane_hi, flags, dot_dev, ws, ws_bytes, stream);
}

hp_status hp_apply_hamiltonian_planes_dot(hp_set_t s, const int32_t* degrees, const double* coeffs, int nterms,
                                          double halfwidth, double q, int dtype, const void* in, void* out,
                                          int plane_lo, int plane_hi, int flags, double* dot_dev, void* ws,
                                          size_t ws_bytes, void* stream) {
  HP_NVTX("hp_apply_hamiltonian_planes_dot");
  hp_status rc = check_set(s);
  if (rc) return rc;
  if ((rc = check_terms(s, degrees, nterms, halfwidth))) return rc;
  if (!s->boxed || plane_lo < 0 || plane_hi > s->side[0] || plane_lo > plane_hi)
    return fail(HP_ERR_VALUE, "plane range must lie inside a full cube or slab");
  if (s->n == 0) return HP_OK;
  if (flags & (HP_REF_ORDER | HP_CHECK_FINITE))
    return fail(HP_ERR_VALUE, "plane-range matvec: the fused full-cube evaluator only");
  if (dot_dev && dtype != HP_C128) return fail(HP_ERR_VALUE, "plane-range dot: complex128 only");
  auto terms = make_terms(s->dim, degrees, coeffs, nterms);
  bool done = false;
  rc = fullgrid_apply_planes(s, terms, halfwidth, dtype, in, out, plane_lo, plane_hi, flags, ws, ws_bytes,
                             as_stream(stream), &done, dot_dev, q);
  if (rc) return rc;
  if (!done) return fail(HP_ERR_VALUE, "plane-range matvec: the fused full-cube evaluator only");
  return HP_OK;
}

hp_status hp_apply_polynomial_planes(hp_set_t s, const int32_t* degrees, const double* coeffs, int nterms,
                                     double halfwidth, int dtype, const void* in, void* out, int plane_lo,
                                     int plane_hi, int flags, void* ws, size_t ws_bytes, void* stream) {
  return hp_apply_polynomial_planes_dot(s, degrees, coeffs, nterms, halfwidth, dtype, in, out, plane_lo, plane_hi,
                                        flags, nullptr, ws, ws_bytes, stream);
}

hp_status hp_square_sum(hp_set_t s, int dtype, const void* in, void* out, int64_t batch, void* stream) {
  HP_NVTX("hp_square_sum");
  hp_status rc = check_set(s);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (s->n == 0 || batch == 0) return HP_OK;
  if (dtype == HP_C128) return launch_square<double2>(s, (const double2*)in, (double2*)out, batch, st);
  return launch_square<double>(s, (const double*)in, (double*)out, batch, st);
}

}  // extern "C"
