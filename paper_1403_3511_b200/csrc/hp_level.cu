// Level-fused evaluator: one kernel per axis level, suffix trie + prefix Clenshaw.
//
// The surrogate y = sum_r alpha_r T_{r_1}(X_1) ... T_{r_N}(X_N) v is
// evaluated axis by axis, innermost axis first (the reference's product
// order, fast_apply.py:166-193).  Each level a is ONE kernel: for every
// ordinal o it walks the axis-a line through o to +-K (K = largest degree
// at this level) via the neighbour tables (down-chains never break in a
// downward-closed set; up-chains stop at the first pruned index), and runs
// the three-term recurrence T_k = (2/L) X T_{k-1} - T_{k-2} on the shrinking
// window in registers with absent positions forced to zero -- so T_k(X_a) x
// at o is exactly the restricted operator of fast_apply.py:69-92 -- and
// accumulates "targets": each target is a linear combination
// sum_e w_e T_{k_e}(X_a) x_{i_e}, written once per level.
//
// Levels N-1 .. c+1 run in suffix mode (targets = child vectors
// T_k(X_a) u_sigma that share trailing degrees, plus y for finished terms);
// level c forms prefix vectors z_pi = sum alpha T_{r_c}(X_c) u_sigma grouped by
// the degrees still to apply on axes 0..c-1; levels c-1 .. 0 run in prefix
// (Clenshaw) mode, z'_pi' = sum_k T_k(X_a) z_(pi',k).  The planner picks the
// cut c that minimises the vectors read and written.  Product order inside
// every term is unchanged, so on pruned sets the operator is the
// reference's; only the summation order of the terms differs.
#include <algorithm>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <mutex>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "hp_common.cuh"
#include "hp_program.h"

namespace hp {

struct LvProgram {
  std::vector<LvLevel> levels;
  int nslots = 0;
  bool ok = false;
  double cost = 0.0;
};

// ---------------------------------------------------------------- planner

namespace {

struct Builder {
  LvLevel L{};
  std::map<int, int> in_index;                        // buffer -> input index
  std::map<int, std::vector<std::pair<int, LvEnt>>> tg;  // target buffer -> (order, entry)
  bool ok = true;
  int nent = 0;
  int input(int buf) {
    auto it = in_index.find(buf);
    if (it != in_index.end()) return it->second;
    if (L.nin >= LV_MAXIN) { ok = false; return 0; }
    in_index[buf] = L.nin;
    L.in_buf[L.nin] = (short)buf;
    return L.nin++;
  }
  void add(int target_buf, int in_buf, int k, double w) {
    LvEnt e;
    e.input = (unsigned char)input(in_buf);
    e.k = (signed char)k;
    e.w = w;
    L.K = std::max(L.K, k);
    tg[target_buf].push_back({(int)tg[target_buf].size(), e});
  }
  bool finish() {
    if (!ok) return false;
    std::vector<LvEnt> all;
    L.ntg = 0;
    for (auto& t : tg) {
      if (t.second.size() == 1 && t.first >= 0) {  // single-term child vector: written directly
        LvEnt x = t.second[0].second;
        x.tg = 0xFF;
        x.slot = (short)t.first;
        all.push_back(x);
        continue;
      }
      if (L.ntg >= LV_MAXTG) return false;
      L.tg_buf[L.ntg] = (short)t.first;
      for (auto& e : t.second) {
        LvEnt x = e.second;
        x.tg = (unsigned char)L.ntg;
        x.slot = -1;
        all.push_back(x);
      }
      ++L.ntg;
    }
    if ((int)all.size() > LV_MAXENT) return false;
    L.tgn = L.ntg <= 1 ? 1 : L.ntg <= 2 ? 2 : L.ntg <= 4 ? 4 : L.ntg <= 8 ? 8 : LV_MAXTG;
    if (L.nin * (L.K + 1) * L.tgn > LV_WT) return false;
    for (int i = 0; i < L.nin * (L.K + 1) * L.tgn; ++i) L.wt[i] = 0.0;
    for (int i = 0; i < L.nin; ++i) L.in_pmask[i] = 0, L.in_kmask[i] = 0, L.in_dmask[i] = 0;
    std::stable_sort(all.begin(), all.end(), [](const LvEnt& a, const LvEnt& b) { return a.input < b.input; });
    int nd = 0, cur = 0;
    for (const LvEnt& e : all) {
      while (cur <= e.input) L.d_start[cur++] = (short)nd;
      // T_k reads the offsets d = -k, -k + 2, .., k of the level's window
      for (int d = -e.k; d <= e.k; d += 2) L.in_pmask[e.input] |= (unsigned short)(1u << (L.K + d));
      if (e.tg == 0xFF) {
        if (nd >= LV_MAXDIRECT) return false;
        L.direct[nd++] = {e.slot, e.k, e.w};
        L.in_dmask[e.input] |= (unsigned char)(1u << e.k);
      } else {
        L.wt[(e.input * (L.K + 1) + e.k) * L.tgn + e.tg] += e.w;
        L.in_kmask[e.input] |= (unsigned char)(1u << e.k);
      }
    }
    while (cur <= L.nin) L.d_start[cur++] = (short)nd;
    nent = (int)all.size();
    return true;
  }
};

}  // namespace

static LvProgram plan_with_cut(int dim, const std::vector<Term>& terms, int cut, bool merge_enabled) {
  LvProgram P;
  const int BUF_V_ = -2, BUF_Y_ = -1;
  int next_slot = 0;
  std::vector<int> free_slots;
  auto alloc = [&](const std::vector<int>& avoid) {
    for (size_t i = 0; i < free_slots.size(); ++i)
      if (std::find(avoid.begin(), avoid.end(), free_slots[i]) == avoid.end()) {
        int s = free_slots[i];
        free_slots.erase(free_slots.begin() + i);
        return s;
      }
    return next_slot++;
  };
  auto zero_upto = [&](const Term& t, int upto) {
    for (int l = 0; l <= upto; ++l)
      if (t.r[l] != 0) return false;
    return true;
  };
  // suffix nodes: (buffer, terms that still need axes <= a)
  struct Node {
    int buf;
    std::vector<int> rows;
  };
  std::vector<Node> nodes{{BUF_V_, {}}};
  bool y_written = false;
  double cost = 0.0;
  // y entries moved from the first y level to the level after it (see below): (buffer, weight) of T_0 entries
  std::vector<std::pair<int, double>> deferred;
  static const bool defer_enabled = [] {
    const char* e = getenv("HP_LEVEL_DEFER");
    return !e || atoi(e) != 0;
  }();
  auto flush_deferred = [&](Builder& B) {
    for (auto& d : deferred) B.add(BUF_Y_, d.first, 0, d.second);
    deferred.clear();
  };
  // terms with all degrees zero: harvested at the first level
  std::vector<int> consts;
  for (size_t i = 0; i < terms.size(); ++i) {
    if (zero_upto(terms[i], dim - 1)) consts.push_back((int)i);
    else nodes[0].rows.push_back((int)i);
  }
  for (int a = dim - 1; a > cut; --a) {  // ---- suffix levels
    Builder B;
    B.L.axis = a;
    std::vector<int> inputs;
    for (auto& nd : nodes) if (nd.buf >= 0) inputs.push_back(nd.buf);
    if (!y_written) for (int it : consts) B.add(BUF_Y_, BUF_V_, 0, terms[it].alpha);
    flush_deferred(B);
    // candidate next nodes: T_k(X_a) u_parent (k > 0: a new vector) or u_parent itself (k = 0)
    struct Cand {
      int parent, k;
      std::vector<int> rows;
    };
    std::vector<Cand> cands;
    for (auto& nd : nodes) {
      std::map<int, std::vector<int>> groups;
      for (int it : nd.rows) {
        int k = terms[it].r[a];
        if (k > LV_MAXK) return P;
        groups[k].push_back(it);
      }
      for (auto& g : groups) {
        const int k = g.first;
        std::vector<int> nonleaf;
        for (int it : g.second) {
          if (k > 0 && zero_upto(terms[it], a - 1)) B.add(BUF_Y_, nd.buf, k, terms[it].alpha);
          else nonleaf.push_back(it);  // k == 0 rows cannot be leaves: some r[0..a-1] != 0
        }
        if (!nonleaf.empty()) cands.push_back({nd.buf, k, nonleaf});
      }
    }
    // Merge candidates whose remaining term patterns (r_0 .. r_{a-1}) carry proportional
    // coefficients: every later level would apply them identically, so one accumulated vector
    // m = u_1 + lambda u_2 + ... replaces them (the representative's terms stand for all).  For
    // cfg3's equal pair coefficients this turns the per-axis suffix vectors into one running sum;
    // single-term suffixes with the same remaining pattern merge on any set.
    auto signature = [&](const std::vector<int>& rows) {
      std::map<std::vector<int>, double> sig;
      for (int it : rows) sig[std::vector<int>(terms[it].r, terms[it].r + a)] = terms[it].alpha;
      return sig;
    };
    struct Group {
      std::map<std::vector<int>, double> sig;
      std::vector<std::pair<int, double>> members;  // (candidate, lambda)
    };
    std::vector<Group> groups;
    for (int ci = 0; ci < (int)cands.size(); ++ci) {
      auto sig = signature(cands[ci].rows);
      bool placed = !merge_enabled;
      for (auto& gr : groups) {
        if (placed) break;
        if (gr.sig.size() != sig.size()) continue;
        const double lam = sig.begin()->second / gr.sig.begin()->second;
        bool prop = true;
        for (auto ia = gr.sig.begin(), ib = sig.begin(); prop && ia != gr.sig.end(); ++ia, ++ib)
          prop = ia->first == ib->first && std::fabs(ib->second - lam * ia->second) <= 1e-15 * std::fabs(ib->second);
        if (prop) {
          gr.members.push_back({ci, lam});
          placed = true;
        }
      }
      if (!placed || !merge_enabled) groups.push_back({sig, {{ci, 1.0}}});
    }
    std::vector<Node> next;
    for (auto& gr : groups) {
      const Cand& rep = cands[gr.members[0].first];
      if (gr.members.size() == 1) {
        if (rep.k == 0) {
          next.push_back({rep.parent, rep.rows});  // passes through: no new vector
        } else {
          int sl = alloc(inputs);
          B.add(sl, rep.parent, rep.k, 1.0);
          next.push_back({sl, rep.rows});
        }
        continue;
      }
      int sl = alloc(inputs);
      for (auto& mem : gr.members) B.add(sl, cands[mem.first].parent, cands[mem.first].k, mem.second);
      next.push_back({sl, rep.rows});
    }
    // The first level that writes y does not have to: a T_0 entry on v, and an entry that equals a
    // single-term child vector of this level up to a factor, are the same numbers at the next
    // level, which reads v and that child anyway -- y is then first written there, and this level
    // neither writes nor the next one re-reads it (cfg3: 32 of 500 B per coefficient).
    if (defer_enabled && !y_written && B.tg.count(BUF_Y_)) {
      std::vector<std::pair<int, double>> moved;
      bool all = true;
      for (auto& oe : B.tg[BUF_Y_]) {
        const LvEnt& e = oe.second;
        if (e.k == 0) {
          if (B.L.in_buf[e.input] != BUF_V_) { all = false; break; }
          moved.push_back({BUF_V_, e.w});
          continue;
        }
        bool found = false;
        for (auto& t : B.tg) {
          if (t.first < 0 || t.second.size() != 1) continue;
          const LvEnt& c = t.second[0].second;
          bool is_node = false;
          for (auto& nd : next) is_node |= nd.buf == t.first;
          if (is_node && c.input == e.input && c.k == e.k && c.w != 0.0) {
            moved.push_back({t.first, e.w / c.w});
            found = true;
            break;
          }
        }
        if (!found) { all = false; break; }
      }
      if (all) {
        B.tg.erase(BUF_Y_);
        deferred = moved;
        y_written = true;  // the constants travel with the deferred entries
      }
    }
    std::vector<int> released;
    for (int buf : inputs) {
      bool live = false;
      for (auto& nd : next) live |= nd.buf == buf;
      if (!live) released.push_back(buf);
    }
    if (!B.finish()) return P;
    // a level whose targets are all directly written child vectors has ntg == 0 but still runs
    if (!B.tg.empty()) {
      if (B.tg.count(BUF_Y_)) y_written = true;
      cost += B.L.nin + B.L.ntg + (B.tg.count(BUF_Y_) && P.levels.size() ? 1 : 0);
      P.levels.push_back(B.L);
    }
    for (int sl : released) free_slots.push_back(sl);
    nodes = next;
  }
  // ---- cut level: z_pi = sum alpha T_{r_cut}(X_cut) u_sigma, pi = (r_0..r_{cut-1})
  std::map<std::vector<int>, int> zbuf;  // prefix -> slot (empty prefix -> y)
  {
    Builder B;
    B.L.axis = cut;
    std::vector<int> inputs;
    for (auto& nd : nodes) if (nd.buf >= 0) inputs.push_back(nd.buf);
    if (!y_written) for (int it : consts) B.add(BUF_Y_, BUF_V_, 0, terms[it].alpha);
    flush_deferred(B);
    for (auto& nd : nodes) {
      for (int it : nd.rows) {
        const Term& t = terms[it];
        if (t.r[cut] > LV_MAXK) return P;
        std::vector<int> pre(t.r, t.r + cut);
        bool zero = std::all_of(pre.begin(), pre.end(), [](int x) { return x == 0; });
        int target;
        if (zero) target = BUF_Y_;
        else {
          auto f = zbuf.find(pre);
          if (f == zbuf.end()) {
            target = alloc(inputs);
            zbuf[pre] = target;
          } else {
            target = f->second;
          }
        }
        B.add(target, nd.buf, t.r[cut], t.alpha);
      }
    }
    if (!B.finish()) return P;
    cost += B.L.nin + B.L.ntg;
    P.levels.push_back(B.L);
    for (int s : inputs) free_slots.push_back(s);
  }
  // ---- prefix levels: z'_pi' = sum_k T_k(X_a) z_(pi',k)
  for (int a = cut - 1; a >= 0; --a) {
    Builder B;
    B.L.axis = a;
    std::vector<int> inputs;
    for (auto& z : zbuf) inputs.push_back(z.second);
    std::map<std::vector<int>, int> nz;
    for (auto& z : zbuf) {
      std::vector<int> pre(z.first.begin(), z.first.begin() + a);
      int k = z.first[a];
      if (k > LV_MAXK) return P;
      bool zero = std::all_of(pre.begin(), pre.end(), [](int x) { return x == 0; });
      int target;
      if (zero) target = BUF_Y_;
      else {
        auto f = nz.find(pre);
        if (f == nz.end()) {
          target = alloc(inputs);
          nz[pre] = target;
        } else {
          target = f->second;
        }
      }
      B.add(target, z.second, k, 1.0);
    }
    if (!B.finish()) return P;
    cost += B.L.nin + B.L.ntg + 1;
    P.levels.push_back(B.L);
    for (int s : inputs) free_slots.push_back(s);
    zbuf = nz;
  }
  if (!zbuf.empty() || P.levels.empty()) return P;
  P.nslots = next_slot;
  P.cost = cost + 0.25 * next_slot;
  P.ok = true;
  return P;
}

static void dump_plan(const LvProgram& P) {  // HP_LEVEL_DEBUG=1: planner output on stderr (2: every input)
  const char* e = getenv("HP_LEVEL_DEBUG");
  const bool detail = e && atoi(e) >= 2;
  fprintf(stderr, "[hp_level] %zu levels, %d slots, cost %.2f\n", P.levels.size(), P.nslots, P.cost);
  for (const LvLevel& L : P.levels) {
    fprintf(stderr, "  axis %d K %d inputs %d targets %d (accumulators %d) direct children %d\n", L.axis, L.K, L.nin,
            L.ntg, L.tgn, (int)L.d_start[L.nin]);
    if (!detail) continue;
    for (int q = 0; q < L.ntg; ++q) fprintf(stderr, "    target %d -> buffer %d\n", q, L.tg_buf[q]);
    for (int i = 0; i < L.nin; ++i) {
      fprintf(stderr, "    input buffer %d window %#x:", L.in_buf[i], L.in_pmask[i]);
      for (int k = 0; k <= L.K; ++k) {
        for (int q = 0; q < L.tgn; ++q)
          if (((L.in_kmask[i] >> k) & 1) && L.wt[(i * (L.K + 1) + k) * L.tgn + q] != 0.0)
            fprintf(stderr, " T%d->t%d", k, q);
        for (int d = L.d_start[i]; d < L.d_start[i + 1]; ++d)
          if (L.direct[d].k == k) fprintf(stderr, " T%d=>s%d", k, L.direct[d].slot);
      }
      fprintf(stderr, "\n");
    }
  }
}

static int merge_mode() {  // HP_LEVEL_MERGE=0 disables merging of proportional suffix nodes
  static int v = [] {
    const char* e = getenv("HP_LEVEL_MERGE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

static LvProgram plan_levels(int dim, const std::vector<Term>& terms) {
  LvProgram best;
  if (const char* e = getenv("HP_LEVEL_CUT")) {  // experiments: force the suffix/prefix cut
    int c = atoi(e);
    if (c >= 0 && c < dim) return plan_with_cut(dim, terms, c, merge_mode() != 0);
  }
  // every cut, with and without merging proportional suffix nodes (merged plans can exceed the
  // per-level target limit); the cheapest plan wins
  for (int cut = 0; cut < dim; ++cut)
    for (int mg = 0; mg < 2; ++mg) {
      if (mg == 1 && merge_mode() == 0) continue;
      LvProgram P = plan_with_cut(dim, terms, cut, mg == 1);
      if (P.ok && (!best.ok || P.cost < best.cost)) best = std::move(P);
    }
  return best;
}

// plans are cached per (dim, term list): the planner tries every cut with map-heavy builders,
// which is tens of microseconds of host time per call -- the whole budget of a small matvec
static std::shared_ptr<const LvProgram> cached_plan(int dim, const std::vector<Term>& terms) {
  static std::mutex mtx;
  static std::map<std::string, std::shared_ptr<const LvProgram>> cache;
  std::string key((const char*)&dim, sizeof(int));
  for (const Term& t : terms) {
    key.append((const char*)t.r, sizeof(int) * dim);
    key.append((const char*)&t.alpha, sizeof(double));
  }
  std::lock_guard<std::mutex> g(mtx);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 256) cache.clear();  // time-dependent surrogates: bounded
  auto P = std::make_shared<const LvProgram>(plan_levels(dim, terms));
  cache.emplace(key, P);
  return P;
}

// ---------------------------------------------------------------- precomputed windows

template <int K>
__global__ void k_build_win(int64_t n, AxTab ax, int32_t* __restrict__ win) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t seg[2 * K + 1];
    int j;
    ax.template segment<K>(o, j, seg);
#pragma unroll
    for (int d = 1; d <= K; ++d) {
      win[(int64_t)(K - d) * n + o] = (int32_t)seg[K - d];
      win[(int64_t)(K + d - 1) * n + o] = (int32_t)seg[K + d];
    }
  }
}

static int win_mode() {  // HP_LEVEL_WIN=0: walk the tables in every level (no precomputed windows)
  static int v = [] {
    const char* e = getenv("HP_LEVEL_WIN");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// the +-K windows of axis a, built once per set (and rebuilt for a larger K): 2K int32 per point
static hp_status window_table(const hp_set_s* s, int a, int K, cudaStream_t st, const int32_t** out, int* kout) {
  *out = nullptr;
  if (s->boxed || !win_mode() || K < 1 || s->n < 1 || s->n > INT32_MAX) return HP_OK;
  std::lock_guard<std::mutex> g(s->perm_mtx);
  if (!s->d_win[a] || s->d_win_k[a] < K) {
    if (s->d_win[a]) {
      HP_CUDA(cudaStreamSynchronize(st));
      HP_CUDA(cudaFree(s->d_win[a]));
      s->d_win[a] = nullptr;
    }
    int32_t* w = nullptr;
    HP_CUDA(cudaMalloc(&w, (size_t)2 * K * s->n * sizeof(int32_t)));
    const int grid = grid_for(s->n, 256);
    switch (K) {
      case 1: k_build_win<1><<<grid, 256, 0, st>>>(s->n, s->tab(a), w); break;
      case 2: k_build_win<2><<<grid, 256, 0, st>>>(s->n, s->tab(a), w); break;
      case 3: k_build_win<3><<<grid, 256, 0, st>>>(s->n, s->tab(a), w); break;
      default: k_build_win<4><<<grid, 256, 0, st>>>(s->n, s->tab(a), w); break;
    }
    HP_LAUNCH_CHECK("k_build_win");
    s->d_win[a] = w;
    s->d_win_k[a] = K;
  }
  *out = s->d_win[a];
  *kout = s->d_win_k[a];
  return HP_OK;
}

static hp_status level_sums(const hp_set_s* s, cudaStream_t st, const int32_t** out);

// hp_level_jit.cu
bool level_jit_enabled(int64_t work);
bool level_jit_launch(int device, const char* ax_name, const void* ax, const char* axs_name, const void* axs,
                      const LvLevel& lv, int grid, cudaStream_t st, int64_t n, int64_t batch, int dim, double inv_L,
                      double two_L, const double2* v, double2* slots, double2* y, int first, int osc, double2* dotp,
                      const int32_t* perm, const double* sqtab);

bool level_jit_compile_only(const LvLevel& lv, const char* ax_name, const char* axs_name);
int level_jit_compiled();

// the specialised kernel of a large level if there is one, else the instantiation whose accumulator
// count matches the level's dense weight table
template <int K, class AX, class AXS>
static void launch_tgn(int device, int grid, cudaStream_t st, int64_t n, int64_t batch, const AX& ax, const AXS& axs, int dim,
                       const LvLevel& lv, double L, const double2* v, double2* slots, double2* y, int first,
                       int osc, double2* dotp, const int32_t* perm, const double* sqtab) {
  if (level_jit_enabled(n * batch) &&
      level_jit_launch(device, AX::name(), &ax, AXS::name(), &axs, lv, grid, st, n, batch, dim, 1.0 / L, 2.0 / L, v, slots,
                       y, first, osc, dotp, perm, sqtab))
    return;
#define HP_LV_GO(T)                                                                                          \
  k_level<K, T, AX, AXS, LvLevel><<<grid, 256, 0, st>>>(n, batch, ax, axs, dim, lv, 1.0 / L, 2.0 / L, v, slots, y, \
                                                 first, osc, dotp, perm, sqtab)
  switch (lv.tgn) {
    case 1: HP_LV_GO(1); break;
    case 2: HP_LV_GO(2); break;
    case 4: HP_LV_GO(4); break;
    case 8: HP_LV_GO(8); break;
    default: HP_LV_GO(LV_MAXTG); break;
  }
#undef HP_LV_GO
}

template <int K>
static hp_status launch_level(const hp_set_s* s, const LvLevel& lv, double L, const double2* v, double2* slots,
                              double2* y, int64_t batch, int first, int osc, double2* dotp, int grid,
                              cudaStream_t st, const int32_t* perm, const double* sqtab) {
  const int64_t n = s->n;
  if (s->boxed) {
    LvAllBox axs;
    for (int a = 0; a < s->dim; ++a) axs.ax[a] = s->box(a);
    launch_tgn<K>(s->device, grid, st, n, batch, s->box(lv.axis), axs, s->dim, lv, L, v, slots, y, first, osc, dotp, perm, sqtab);
  } else {
    LvAllTab axs;
    for (int a = 0; a < s->dim; ++a) axs.ax[a] = s->tab(a);
    axs.jsum = nullptr;
    if (osc)
      if (hp_status rc = level_sums(s, st, &axs.jsum)) return rc;
    int kwin = 0;
    const int32_t* win = nullptr;
    if (lv.axis == s->dim - 1 && !perm && s->kind == HP_KIND_HYPERBOLIC) {
      // innermost axis of a hyperbolic cross (downward closed, lexicographic): windows from the j table
      launch_tgn<K>(s->device, grid, st, n, batch, AxInner(s->tab(lv.axis), n), axs, s->dim, lv, L, v, slots, y, first, osc,
                    dotp, perm, sqtab);
    } else if (batch > 1 && window_table(s, lv.axis, K, st, &win, &kwin) == HP_OK && win) {
      // batched levels read precomputed windows (cfg5 713 -> 696 ms); single vectors walk the tables
      // with the first hop prefetched (cfg3: 5.86 ms vs 6.03 with windows; profiles/r2/sweep_level.txt)
      launch_tgn<K>(s->device, grid, st, n, batch, AxWin(s->tab(lv.axis), win, n, kwin), axs, s->dim, lv, L, v, slots, y,
                    first, osc, dotp, perm, sqtab);
    } else if (batch == 1) {
      launch_tgn<K>(s->device, grid, st, n, batch, AxTabPf(s->tab(lv.axis)), axs, s->dim, lv, L, v, slots, y, first, osc,
                    dotp, perm, sqtab);
    } else {
      launch_tgn<K>(s->device, grid, st, n, batch, s->tab(lv.axis), axs, s->dim, lv, L, v, slots, y, first, osc, dotp, perm,
                    sqtab);
    }
  }
  HP_LAUNCH_CHECK("k_level");
  return HP_OK;
}

// ---------------------------------------------------------------- ladder coefficients

__global__ void k_ladder_table(int m, double* __restrict__ t) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    t[i] = i > 8 ? sqrt((i - 8) * 0.5) : 0.0;
}

// sqrt(j / 2) tabulated once per set (pointer to the entry of j = 0), so the level kernels load
// their 2K window links instead of evaluating 2K double-precision square roots per ordinal.
// Sets whose indices may exceed `bound` (explicit lists) get no table (the kernels call sqrt).
static hp_status ladder_table(const hp_set_s* s, cudaStream_t st, const double** out) {
  *out = nullptr;
  static const int on = [] {
    const char* e = getenv("HP_LEVEL_SQTAB");
    return e ? atoi(e) : 1;
  }();
  if (!on || s->kind == HP_KIND_CUSTOM) return HP_OK;
  std::lock_guard<std::mutex> g(s->perm_mtx);
  if (!s->d_sqtab) {
    const int m = s->bound + 17;
    double* t = nullptr;
    HP_CUDA(cudaMalloc(&t, (size_t)m * sizeof(double)));
    k_ladder_table<<<grid_for(m, 256), 256, 0, st>>>(m, t);
    HP_LAUNCH_CHECK("k_ladder_table");
    s->d_sqtab = t;
  }
  *out = s->d_sqtab + 8;
  return HP_OK;
}

// ---------------------------------------------------------------- oscillator levels

__global__ void k_level_sums(int64_t n, int dim, LvAllTab axs, int32_t* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    int sum = 0;
    for (int a = 0; a < dim; ++a) sum += axs.j(a, o);
    out[o] = sum;
  }
}

// sum_l j_l per ordinal of a tabled set, built once: the level that adds the oscillator diagonal
// (apply_hamiltonian, fast_apply.py:195-198) then loads 4 bytes per ordinal instead of one j per axis
static hp_status level_sums(const hp_set_s* s, cudaStream_t st, const int32_t** out) {
  *out = nullptr;
  if (s->boxed || s->n < 1) return HP_OK;
  std::lock_guard<std::mutex> g(s->perm_mtx);
  if (!s->d_jsum) {
    int32_t* t = nullptr;
    HP_CUDA(cudaMalloc(&t, (size_t)s->n * sizeof(int32_t)));
    LvAllTab axs;
    for (int a = 0; a < s->dim; ++a) axs.ax[a] = s->tab(a);
    axs.jsum = nullptr;
    k_level_sums<<<grid_for(s->n, 256), 256, 0, st>>>(s->n, s->dim, axs, t);
    HP_LAUNCH_CHECK("k_level_sums");
    s->d_jsum = t;
  }
  *out = s->d_jsum;
  return HP_OK;
}

// ---------------------------------------------------------------- line order of an axis

// Line-blocked order: the heads (points without a -e_a neighbour) are taken in blocks of 32
// consecutive heads; a block emits row k = the k-th points of its lines for k = 0, 1, ...  A row
// is (nearly) contiguous in storage, so a warp's loads stay coalesced, and the rows k +- d that
// the +-K windows read are processed by the neighbouring warps: each input element is fetched
// from HBM about once instead of once per window position.
// Pass 1: per block of 32 heads, the number of points of its lines (one warp per block).
__global__ void k_line_count(int64_t nheads, const int32_t* __restrict__ heads, const int32_t* __restrict__ up,
                             int32_t* __restrict__ bcount) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t w = w0; w * 32 < nheads; w += nw) {
    const int64_t i = w * 32 + lane;
    int L = 0;
    if (i < nheads)
      for (int64_t q = __ldg(heads + i); q >= 0; q = __ldg(up + q)) ++L;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_down_sync(0xffffffffu, L, o);
    if (lane == 0) bcount[w] = L;
  }
}
// Pass 2: each warp writes its block's rows at the block offset
__global__ void k_line_fill(int64_t nheads, const int32_t* __restrict__ heads, const int32_t* __restrict__ up,
                            const int32_t* __restrict__ boff, int32_t* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t w = w0; w * 32 < nheads; w += nw) {
    const int64_t i = w * 32 + lane;
    int64_t q = i < nheads ? (int64_t)__ldg(heads + i) : -1;
    int32_t pos = __ldg(boff + w);
    for (;;) {
      const unsigned live = __ballot_sync(0xffffffffu, q >= 0);
      if (!live) break;
      if (q >= 0) {
        perm[pos + __popc(live & ((1u << lane) - 1))] = (int32_t)q;
        q = __ldg(up + q);
      }
      pos += __popc(live);
    }
  }
}
__global__ void k_line_heads_flag(int64_t n, const int32_t* __restrict__ down, int32_t* __restrict__ flag) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
    flag[o] = __ldg(down + o) < 0 ? 1 : 0;
}
__global__ void k_line_heads_list(int64_t n, const int32_t* __restrict__ down, const int32_t* __restrict__ pos,
                                  int32_t* __restrict__ heads) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
    if (__ldg(down + o) < 0) heads[__ldg(pos + o)] = (int32_t)o;
}

// axes whose level kernels run in line order (HP_LEVEL_PERM: bit a = axis a).  Measured with the
// merged plans of round 2 (ms per matvec; profiles/r2/sweep_level.txt): cfg3 (N = 6) no axis 6.23,
// {1} 6.42, {0,1} 6.53, {1,2} 6.65; cfg5 (N = 8, 32 vectors) {0,1,2} 708, {1,2} 715, {0,1} 731,
// {1} 737.  Round 1 (unmerged plans) preferred {1} on both: the line order pays where a level
// reads many outer-axis windows, which merging made rarer on N = 6.
static unsigned perm_axes(int dim) {
  static int env = [] {
    const char* e = getenv("HP_LEVEL_PERM");
    return e ? atoi(e) : -1;
  }();
  if (env >= 0) return (unsigned)env;
  return dim >= 7 ? 7u : 0u;
}

// perm: the line-blocked order of the ordinals (a permutation of 0..n-1: every ordinal lies on
// exactly one axis line, which has exactly one head)
static hp_status line_order(const hp_set_s* s, int a, cudaStream_t st, const int32_t** out) {
  *out = nullptr;
  if (s->boxed || !(perm_axes(s->dim) >> a & 1) || s->n < 2 || s->n > INT32_MAX) return HP_OK;
  std::lock_guard<std::mutex> g(s->perm_mtx);
  if (!s->d_perm[a]) {
    const int64_t n = s->n;
    // heads in ordinal order: flag, exclusive scan, compact
    int32_t *flag = nullptr, *pos = nullptr, *heads = nullptr, *perm = nullptr;
    HP_CUDA(cudaMallocAsync(&flag, (n + 1) * sizeof(int32_t), st));
    HP_CUDA(cudaMallocAsync(&pos, (n + 1) * sizeof(int32_t), st));
    void* tmp = nullptr;
    size_t tb = 0;
    HP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n + 1, st));
    HP_CUDA(cudaMallocAsync(&tmp, tb, st));
    const int grid = grid_for(n, 256);
    HP_CUDA(cudaMemsetAsync(flag + n, 0, sizeof(int32_t), st));
    k_line_heads_flag<<<grid, 256, 0, st>>>(n, s->d_down[a], flag);
    HP_LAUNCH_CHECK("k_line_heads_flag");
    HP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)n + 1, st));
    int32_t nheads = 0;
    HP_CUDA(cudaMemcpyAsync(&nheads, pos + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HP_CUDA(cudaStreamSynchronize(st));
    HP_CUDA(cudaMallocAsync(&heads, std::max<int64_t>(nheads, 1) * sizeof(int32_t), st));
    k_line_heads_list<<<grid, 256, 0, st>>>(n, s->d_down[a], pos, heads);
    HP_LAUNCH_CHECK("k_line_heads_list");
    // per-block counts -> offsets (reusing flag / pos)
    const int64_t nb = (nheads + 31) / 32;
    const int wgrid = grid_for(nb * 32, 256);
    HP_CUDA(cudaMemsetAsync(flag + nb, 0, sizeof(int32_t), st));
    k_line_count<<<wgrid, 256, 0, st>>>(nheads, heads, s->d_up[a], flag);
    HP_LAUNCH_CHECK("k_line_count");
    HP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)nb + 1, st));
    HP_CUDA(cudaMalloc(&perm, n * sizeof(int32_t)));
    k_line_fill<<<wgrid, 256, 0, st>>>(nheads, heads, s->d_up[a], pos, perm);
    HP_LAUNCH_CHECK("k_line_fill");
    HP_CUDA(cudaFreeAsync(flag, st));
    HP_CUDA(cudaFreeAsync(pos, st));
    HP_CUDA(cudaFreeAsync(heads, st));
    HP_CUDA(cudaFreeAsync(tmp, st));
    s->d_perm[a] = perm;
  }
  *out = s->d_perm[a];
  return HP_OK;
}

// ---------------------------------------------------------------- entry points

double level_plan_cost(int dim, const std::vector<Term>& terms) {
  const auto P = cached_plan(dim, terms);
  return P->ok ? P->cost : -1.0;
}

size_t level_workspace_bytes(const hp_set_s* s, const std::vector<Term>& terms, int dtype, int64_t batch) {
  if (dtype != HP_C128) return 0;
  const auto Pp = cached_plan(s->dim, terms);
  const LvProgram& P = *Pp;
  if (!P.ok) return 0;
  return (size_t)std::max(P.nslots, 1) * s->n * batch * sizeof(double2);
}

hp_status level_apply(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                      const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                      cudaStream_t st, bool* done, DotOut* dot) {
  *done = false;
  if (dot) dot->n = 0;
  if (dtype != HP_C128 || (flags & HP_REF_ORDER) || s->n == 0) return HP_OK;
  const auto Pp = cached_plan(s->dim, terms);
  const LvProgram& P = *Pp;
  if (!P.ok) return HP_OK;
  if (const char* e = getenv("HP_LEVEL_DEBUG"))
    if (atoi(e)) dump_plan(P);
  // batches are chunked so that the intermediate vectors fit the workspace
  size_t per_vec = (size_t)std::max(P.nslots, 1) * s->n * sizeof(double2);
  int64_t chunk = std::min<int64_t>(batch, (int64_t)(ws_bytes / per_vec));
  if (chunk < 1) return HP_OK;
  const int64_t n = s->n;
  // blocks per SM of the grid-stride level kernels (HP_LEVEL_GRID overrides): batched levels 16,
  // single vectors 4 = one resident wave (specialised kernels, profiles/r2/sweep_level.txt: cfg3
  // 3.53 ms at 4, 3.68 at 8, 3.73 at 16; cfg5 418 / 412 / 406 / 398 ms at 4 / 8 / 16 / 32)
  static const int bps_env = [] {
    const char* e = getenv("HP_LEVEL_GRID");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const int bps = bps_env ? bps_env : (batch > 1 ? 16 : 4);
  const int grid = grid_for(n, 256, 148 * bps);
  const bool osc = flags & HP_ADD_OSC;
  // y must be written by the first level that targets it and osc/dot applied at the last
  int first_y = -1, last_y = -1;
  for (int li = 0; li < (int)P.levels.size(); ++li)
    for (int t = 0; t < P.levels[li].ntg; ++t)
      if (P.levels[li].tg_buf[t] == -1) {
        if (first_y < 0) first_y = li;
        last_y = li;
      }
  if (first_y < 0) return HP_OK;
  const double* sqtab = nullptr;
  if (hp_status rc = ladder_table(s, st, &sqtab)) return rc;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t nb = std::min(chunk, batch - b0);
    const double2* v = (const double2*)in + b0 * n;
    double2* y = (double2*)out + b0 * n;
    double2* slots = (double2*)ws;
    for (int li = 0; li < (int)P.levels.size(); ++li) {
      const LvLevel& lv = P.levels[li];
      const bool last = li == last_y;
      const int first = (li == first_y && !(flags & HP_LV_ACCUMULATE)) ? 1 : 0;
      double2* dotp = (last && dot && dot->partial && batch == 1 && grid <= dot->capacity) ? dot->partial : nullptr;
      const int32_t* perm = nullptr;
      hp_status rc = line_order(s, lv.axis, st, &perm);
      if (rc) return rc;
      const int oscf = last && osc ? 1 : 0;
      switch (lv.K) {
        case 0: rc = launch_level<0>(s, lv, halfwidth, v, slots, y, nb, first, oscf, dotp, grid, st, perm, sqtab); break;
        case 1: rc = launch_level<1>(s, lv, halfwidth, v, slots, y, nb, first, oscf, dotp, grid, st, perm, sqtab); break;
        case 2: rc = launch_level<2>(s, lv, halfwidth, v, slots, y, nb, first, oscf, dotp, grid, st, perm, sqtab); break;
        case 3: rc = launch_level<3>(s, lv, halfwidth, v, slots, y, nb, first, oscf, dotp, grid, st, perm, sqtab); break;
        default: rc = launch_level<4>(s, lv, halfwidth, v, slots, y, nb, first, oscf, dotp, grid, st, perm, sqtab); break;
      }
      if (rc) return rc;
      if (dotp) dot->n = grid;
    }
  }
  *done = true;
  return HP_OK;
}

}  // namespace hp

extern "C" int hp_level_jit_kernels(void) { return hp::level_jit_compiled(); }

extern "C" hp_status hp_level_jit_selftest(int dim, const int32_t* degrees, const double* coeffs, int nterms,
                                           int* nkernels_out) {
  using namespace hp;
  if (nkernels_out) *nkernels_out = 0;
  if (dim < 1 || dim > HP_MAXDIM || nterms < 1 || !degrees || !coeffs)
    return fail(HP_ERR_VALUE, "hp_level_jit_selftest: bad arguments");
  const auto terms = make_terms(dim, degrees, coeffs, nterms);
  const LvProgram P = plan_levels(dim, terms);
  if (!P.ok) return fail(HP_ERR_VALUE, "hp_level_jit_selftest: the level planner does not cover this polynomial");
  int n = 0;
  for (const LvLevel& lv : P.levels) {
    if (!level_jit_compile_only(lv, AxTab::name(), LvAllTab::name()) ||
        !level_jit_compile_only(lv, AxBox::name(), LvAllBox::name()))
      return fail(HP_ERR_RUNTIME, "hp_level_jit_selftest: NVRTC unavailable or compilation failed (axis " +
                                      std::to_string(lv.axis) + ")");
    n += 2;
  }
  if (nkernels_out) *nkernels_out = n;
  return HP_OK;
}

