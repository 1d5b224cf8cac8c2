// Level-fused evaluator: one kernel per axis level of the suffix trie.
//
// The suffix trie (hp_apply.cu) runs one kernel per Chebyshev *step*; every
// step re-reads its input through the neighbour tables, writes a vector and
// read-modify-writes y for each harvested term (~90 B per coefficient per
// step, 32 steps for cfg3).  Here every trie level -- all nodes that apply
// axis a, all their degrees, all their harvests -- is ONE kernel:
//
//   for each ordinal o: walk the axis-a line through o to +-K (K = largest
//   degree at this level) via the neighbour tables (down-chains never break
//   in a downward-closed set; up-chains stop at the first pruned index),
//   load each input node vector on that segment, run the three-term
//   recurrence T_k = (2/L) X T_{k-1} - T_{k-2} on the shrinking window
//   (K^2 tiny evaluations in registers, absent positions forced to zero, so
//   T_k(o) is exactly the restricted operator of fast_apply.py:69-92), then
//   write the child vectors the next level needs and accumulate every
//   harvested term into y with a single read-modify-write per level.
//
// Product order inside each term (axis N first) is unchanged, so on pruned
// sets the operator is the reference's; only summation order differs.
#include <algorithm>
#include <map>
#include <vector>

#include "hp_common.cuh"
#include "hp_program.h"

namespace hp {

constexpr int LV_MAXIN = 48;
constexpr int LV_MAXACT = 10;
constexpr int LV_MAXK = 4;

struct LvAct {
  signed char k;      // degree
  signed char child;  // >= 0: write T_k into slot `child`; -1: acc += w * T_k
  double w;
};

struct LvLevel {
  int axis;
  int K;
  int nin;
  short in_buf[LV_MAXIN];  // -2 = v, >= 0 slot
  unsigned char nact[LV_MAXIN];
  LvAct act[LV_MAXIN][LV_MAXACT];
};

struct LvProgram {
  std::vector<LvLevel> levels;
  int nslots = 0;
  bool ok = false;
};

// ---------------------------------------------------------------- planner

static LvProgram plan_levels(int dim, const std::vector<Term>& terms) {
  LvProgram P;
  struct Node {
    int buf;
    std::vector<int> rows;
  };
  std::vector<Node> nodes{{-2, {}}};
  for (size_t i = 0; i < terms.size(); ++i) nodes[0].rows.push_back((int)i);
  std::vector<int> free_slots;
  int next_slot = 0;
  auto all_zero = [&](int it, int upto) {  // r[0..upto] all zero (upto < 0: true)
    for (int l = 0; l <= upto; ++l)
      if (terms[it].r[l] != 0) return false;
    return true;
  };
  for (int a = dim - 1; a >= 0; --a) {
    LvLevel L{};
    L.axis = a;
    L.K = 0;
    L.nin = 0;
    std::vector<Node> next;
    std::vector<int> in_use;  // slots read at this level (children must not alias them)
    for (auto& nd : nodes) if (nd.buf >= 0) in_use.push_back(nd.buf);
    std::vector<int> released;
    for (auto& nd : nodes) {
      if ((int)L.nin >= LV_MAXIN) return P;
      int ii = L.nin++;
      L.in_buf[ii] = (short)nd.buf;
      L.nact[ii] = 0;
      std::map<int, std::vector<int>> groups;
      std::vector<int> pass;
      for (int it : nd.rows) {
        int k = terms[it].r[a];
        if (k > LV_MAXK) return P;
        if (k == 0 && !all_zero(it, a - 1)) pass.push_back(it);
        else groups[k].push_back(it);
      }
      for (auto& g : groups) {
        int k = g.first;
        double w = 0.0;
        bool has_leaf = false;
        std::vector<int> nonleaf;
        for (int it : g.second) {
          if (all_zero(it, a - 1)) {
            w += terms[it].alpha;
            has_leaf = true;
          } else {
            nonleaf.push_back(it);
          }
        }
        if (has_leaf) {
          if (L.nact[ii] >= LV_MAXACT) return P;
          L.act[ii][L.nact[ii]++] = LvAct{(signed char)k, -1, w};
          L.K = std::max(L.K, k);
        }
        if (!nonleaf.empty()) {
          if (k == 0) return P;  // cannot happen (k == 0 non-leaves pass through)
          int slot;
          // a fresh slot, never one this level reads
          auto it = std::find_if(free_slots.begin(), free_slots.end(),
                                 [&](int s) { return std::find(in_use.begin(), in_use.end(), s) == in_use.end(); });
          if (it != free_slots.end()) {
            slot = *it;
            free_slots.erase(it);
          } else {
            slot = next_slot++;
          }
          if (L.nact[ii] >= LV_MAXACT || slot > 120) return P;
          L.act[ii][L.nact[ii]++] = LvAct{(signed char)k, (signed char)slot, 0.0};
          L.K = std::max(L.K, k);
          next.push_back({slot, nonleaf});
        }
      }
      if (L.nact[ii] == 0) --L.nin;  // pass-through only: nothing to read at this level
      if (!pass.empty()) next.push_back({nd.buf, pass});
      else if (nd.buf >= 0) released.push_back(nd.buf);
    }
    if (L.nin > 0) P.levels.push_back(L);
    for (int s : released) free_slots.push_back(s);
    nodes = next;
    if (nodes.empty()) break;
  }
  if (!nodes.empty()) return P;  // unreachable: axis 0 harvests everything
  if (P.levels.empty()) {        // no terms: one empty level still writes y (= levels * v)
    LvLevel L{};
    L.axis = 0;
    P.levels.push_back(L);
  }
  P.nslots = next_slot;
  P.ok = true;
  return P;
}

// ---------------------------------------------------------------- kernel

template <int K, class AX, class AXS>
__global__ void __launch_bounds__(256) k_level(int64_t n, int64_t batch, AX ax, AXS axs, int dim, LvLevel lv,
                                               double inv_L, double two_L, const double2* __restrict__ v,
                                               double2* __restrict__ slots, double2* __restrict__ y, int first,
                                               int osc, double2* __restrict__ dotp) {
  constexpr int S = 2 * K + 1;
  double2 dacc = make_double2(0.0, 0.0);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    // the axis line through o: seg[K + d] = ordinal of j + d e_a, or -1
    int64_t seg[S];
    int jo;
    {
      int64_t dn, up;
      ax.at(o, jo, dn, up);
      seg[K] = o;
      if (K > 0) {
        seg[K - 1] = dn;
        seg[K + 1] = up;
      }
#pragma unroll
      for (int d = 2; d <= K; ++d) {
        int jj;
        int64_t a0, b0, a1, b1;
        if (seg[K - d + 1] >= 0) ax.at(seg[K - d + 1], jj, a0, b0); else a0 = -1;
        if (seg[K + d - 1] >= 0) ax.at(seg[K + d - 1], jj, a1, b1); else b1 = -1;
        seg[K - d] = a0;
        seg[K + d] = b1;
      }
    }
    double cd[S], cu[S];
#pragma unroll
    for (int p = 0; p < S; ++p) {
      double j = (double)(jo + p - K);
      cd[p] = j > 0.0 ? sqrt(j * 0.5) : 0.0;
      cu[p] = sqrt((j + 1.0) * 0.5);
    }
    double lev = 0.0;
    if (osc)
      for (int a = 0; a < dim; ++a) lev += (double)axs.j(a, o) + 0.5;
    for (int64_t b = 0; b < batch; ++b) {
      const int64_t bo = b * n;
      double2 acc = make_double2(0.0, 0.0);
      for (int ii = 0; ii < lv.nin; ++ii) {
        const double2* x = lv.in_buf[ii] == -2 ? v + bo : slots + (int64_t)lv.in_buf[ii] * n * batch + bo;
        double2 Tm[S], Tc[S], Tn[S];
#pragma unroll
        for (int p = 0; p < S; ++p) Tm[p] = seg[p] >= 0 ? __ldg(x + seg[p]) : make_double2(0.0, 0.0);
        const int na = lv.nact[ii];
        // k = 0 actions
        for (int q = 0; q < na; ++q) {
          LvAct A = lv.act[ii][q];
          if (A.k == 0) {
            acc.x = fma(A.w, Tm[K].x, acc.x);
            acc.y = fma(A.w, Tm[K].y, acc.y);
          }
        }
#pragma unroll
        for (int k = 1; k <= K; ++k) {
          const double sc = k == 1 ? inv_L : two_L;
#pragma unroll
          for (int p = k; p < S - k; ++p) {
            const double2 lo = k == 1 ? Tm[p - 1] : Tc[p - 1];
            const double2 hi = k == 1 ? Tm[p + 1] : Tc[p + 1];
            double2 r = make_double2(sc * fma(cd[p], lo.x, cu[p] * hi.x), sc * fma(cd[p], lo.y, cu[p] * hi.y));
            if (k > 1) {
              r.x -= Tm[p].x;
              r.y -= Tm[p].y;
            }
            if (seg[p] < 0) r = make_double2(0.0, 0.0);
            Tn[p] = r;
          }
          // rotate: (T_{k-2}, T_{k-1}) <- (T_{k-1}, T_k)
          if (k > 1) {
#pragma unroll
            for (int p = 0; p < S; ++p) Tm[p] = Tc[p];
          }
#pragma unroll
          for (int p = 0; p < S; ++p) Tc[p] = Tn[p];
          const double2 val = Tc[K];
          for (int q = 0; q < na; ++q) {
            LvAct A = lv.act[ii][q];
            if (A.k != k) continue;
            if (A.child >= 0) {
              slots[(int64_t)A.child * n * batch + bo + o] = val;
            } else {
              acc.x = fma(A.w, val.x, acc.x);
              acc.y = fma(A.w, val.y, acc.y);
            }
          }
        }
      }
      if (osc) {
        double2 x = __ldg(v + bo + o);
        acc.x = fma(lev, x.x, acc.x);
        acc.y = fma(lev, x.y, acc.y);
      }
      double2 out = acc;
      if (!first) {
        double2 old = y[bo + o];
        out.x += old.x;
        out.y += old.y;
      }
      y[bo + o] = out;
      if (dotp) cdot_acc(__ldg(v + bo + o), out, dacc);
    }
  }
  if (dotp) {
    dacc = block_sum2(dacc);
    if (threadIdx.x == 0) dotp[blockIdx.x] = dacc;
  }
}

struct LvAllBox {
  AxBox ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return ax[a].jloc(o) + ax[a].joff; }
};
struct LvAllTab {
  AxTab ax[HP_MAXDIM];
  __device__ __forceinline__ int j(int a, int64_t o) const { return __ldg(ax[a].jv + o); }
};

template <int K>
static hp_status launch_level(const hp_set_s* s, const LvLevel& lv, double L, const double2* v, double2* slots,
                              double2* y, int64_t batch, int first, int osc, double2* dotp, int grid,
                              cudaStream_t st) {
  const int64_t n = s->n;
  if (s->boxed) {
    LvAllBox axs;
    for (int a = 0; a < s->dim; ++a) axs.ax[a] = s->box(a);
    k_level<K, AxBox, LvAllBox><<<grid, 256, 0, st>>>(n, batch, s->box(lv.axis), axs, s->dim, lv, 1.0 / L, 2.0 / L,
                                                     v, slots, y, first, osc, dotp);
  } else {
    LvAllTab axs;
    for (int a = 0; a < s->dim; ++a) axs.ax[a] = s->tab(a);
    k_level<K, AxTab, LvAllTab><<<grid, 256, 0, st>>>(n, batch, s->tab(lv.axis), axs, s->dim, lv, 1.0 / L, 2.0 / L,
                                                     v, slots, y, first, osc, dotp);
  }
  HP_LAUNCH_CHECK("k_level");
  return HP_OK;
}

// ---------------------------------------------------------------- entry points

size_t level_workspace_bytes(const hp_set_s* s, const std::vector<Term>& terms, int dtype, int64_t batch) {
  if (dtype != HP_C128) return 0;
  LvProgram P = plan_levels(s->dim, terms);
  if (!P.ok) return 0;
  return (size_t)std::max(P.nslots, 1) * s->n * batch * sizeof(double2);
}

hp_status level_apply(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                      const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                      cudaStream_t st, bool* done, DotOut* dot) {
  *done = false;
  if (dot) dot->n = 0;
  if (dtype != HP_C128 || (flags & HP_REF_ORDER) || s->n == 0) return HP_OK;
  LvProgram P = plan_levels(s->dim, terms);
  if (!P.ok) return HP_OK;
  // batches are chunked so that the child vectors fit the workspace
  size_t per_vec = (size_t)std::max(P.nslots, 1) * s->n * sizeof(double2);
  int64_t chunk = std::min<int64_t>(batch, (int64_t)(ws_bytes / per_vec));
  if (chunk < 1) return HP_OK;
  const int64_t n = s->n;
  const int grid = grid_for(n, 256, 148 * 8);
  const bool osc = flags & HP_ADD_OSC;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t nb = std::min(chunk, batch - b0);
    const double2* v = (const double2*)in + b0 * n;
    double2* y = (double2*)out + b0 * n;
    double2* slots = (double2*)ws;
    const int nl = (int)P.levels.size();
    for (int li = 0; li < nl; ++li) {
      const LvLevel& lv = P.levels[li];
      const bool last = li == nl - 1;
      const int first = li == 0 ? 1 : 0;
      double2* dotp = (last && dot && dot->partial && batch == 1 && grid <= dot->capacity) ? dot->partial : nullptr;
      hp_status rc;
      switch (lv.K) {
        case 0: rc = launch_level<0>(s, lv, halfwidth, v, slots, y, nb, first, last && osc, dotp, grid, st); break;
        case 1: rc = launch_level<1>(s, lv, halfwidth, v, slots, y, nb, first, last && osc, dotp, grid, st); break;
        case 2: rc = launch_level<2>(s, lv, halfwidth, v, slots, y, nb, first, last && osc, dotp, grid, st); break;
        case 3: rc = launch_level<3>(s, lv, halfwidth, v, slots, y, nb, first, last && osc, dotp, grid, st); break;
        default: rc = launch_level<4>(s, lv, halfwidth, v, slots, y, nb, first, last && osc, dotp, grid, st); break;
      }
      if (rc) return rc;
      if (dotp) dot->n = grid;
    }
  }
  *done = true;
  return HP_OK;
}

}  // namespace hp
