// Index sets on the device: full cubes, j1-slabs, hyperbolic crosses and
// custom downward-closed sets (reference: pkg/src/hprop/index_set.py).
//
// Hyperbolic crosses {j : prod_l (1 + j_l) <= B}, B = bound + 1, are
// enumerated by *unranking*: with cnt(d, r) = #{d-tuples, prod(1+k) <= r}
// and pre(d, r, k) = sum_{k' < k} cnt(d, floor(r / (k'+1))), the ordinal o
// is decoded level by level (binary search for k, o -= pre, r //= k+1).
// This is exactly the depth-first emission order of the reference recursion
// (index_set.py:163-180), whose child budget is remaining // (k+1) and whose
// last level emits k < remaining.  Ranking j +- e_l with the same tables
// gives the neighbour ordinals of index_set.py:104-130 without any hash map.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hp_common.cuh"

namespace hp {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
hp_status fail(hp_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
hp_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return HP_ERR_CUDA;
}

// ---------------------------------------------------------------- kernels

__global__ void k_full_indices(int64_t n, int dim, const int64_t* __restrict__ stride,
                               const int* __restrict__ side, int joff0, int64_t* out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < dim; ++a) {
      int64_t j = (o / stride[a]) % side[a];
      out[o * dim + a] = j + (a == 0 ? joff0 : 0);
    }
  }
}

// unrank ordinals of a hyperbolic cross into per-axis j arrays
__global__ void k_hyp_unrank(int64_t n, int dim, int64_t budget, const int64_t* __restrict__ pref,
                             const int64_t* __restrict__ off, int32_t* const* jout) {
  for (int64_t o0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o0 < n;
       o0 += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = o0, r = budget;
    for (int l = 0; l < dim - 1; ++l) {
      int d = dim - 1 - l;
      const int64_t* p = pref + off[(int64_t)d * (budget + 1) + r];
      // largest k in [0, r-1] with p[k] <= o  (p[0] = 0, strictly increasing)
      int64_t lo = 0, hi = r - 1;
      while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(p + mid) <= o) lo = mid; else hi = mid - 1;
      }
      o -= __ldg(p + lo);
      jout[l][o0] = (int32_t)lo;
      r = r / (lo + 1);
    }
    jout[dim - 1][o0] = (int32_t)o;
  }
}

// rank of (j_0..j_{a-1} fixed, suffix from level a); returns -1 if absent
__device__ __forceinline__ int64_t hyp_rank_from(int dim, int64_t budget, const int64_t* pref,
                                                 const int64_t* off, int a, int64_t r,
                                                 int64_t base, const int* j) {
  int64_t ord = base;
  for (int l = a; l < dim; ++l) {
    int64_t k = j[l];
    if (k < 0 || k + 1 > r) return -1;
    if (l == dim - 1) return ord + k;
    int d = dim - 1 - l;
    ord += __ldg(pref + off[(int64_t)d * (budget + 1) + r] + k);
    r = r / (k + 1);
  }
  return ord;
}

__global__ void k_hyp_neighbors(int64_t n, int dim, int64_t budget, const int64_t* __restrict__ pref,
                                const int64_t* __restrict__ off, int32_t* const* jin,
                                int32_t* const* down, int32_t* const* up) {
  int j[HP_MAXDIM];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    for (int l = 0; l < dim; ++l) j[l] = jin[l][o];
    int64_t base = 0, r = budget;
    for (int a = 0; a < dim; ++a) {
      // base/r describe the fixed prefix j_0..j_{a-1}
      j[a] -= 1;
      int64_t dn = (j[a] >= 0) ? hyp_rank_from(dim, budget, pref, off, a, r, base, j) : -1;
      j[a] += 2;
      int64_t upo = hyp_rank_from(dim, budget, pref, off, a, r, base, j);
      j[a] -= 1;
      down[a][o] = (int32_t)dn;
      up[a][o] = (int32_t)upo;
      if (a < dim - 1) {
        int d = dim - 1 - a;
        base += __ldg(pref + off[(int64_t)d * (budget + 1) + r] + j[a]);
        r = r / (j[a] + 1);
      }
    }
  }
}

// custom sets: neighbours by lexicographic binary search over the rows
__global__ void k_custom_neighbors(int64_t n, int dim, const int64_t* __restrict__ rows,
                                   int32_t* const* down, int32_t* const* up) {
  int64_t q[HP_MAXDIM];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < dim; ++a) {
      for (int delta = -1; delta <= 1; delta += 2) {
        for (int l = 0; l < dim; ++l) q[l] = rows[o * dim + l];
        q[a] += delta;
        int64_t res = -1;
        if (q[a] >= 0) {
          int64_t lo = 0, hi = n - 1;
          while (lo <= hi) {
            int64_t mid = (lo + hi) >> 1;
            int c = 0;
            for (int l = 0; l < dim && c == 0; ++l) {
              int64_t x = rows[mid * dim + l];
              c = (x < q[l]) ? -1 : (x > q[l] ? 1 : 0);
            }
            if (c == 0) { res = mid; break; }
            if (c < 0) lo = mid + 1; else hi = mid - 1;
          }
        }
        (delta < 0 ? down : up)[a][o] = (int32_t)res;
      }
    }
  }
}

__global__ void k_custom_j(int64_t n, int dim, const int64_t* __restrict__ rows, int32_t* const* jout) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x)
    for (int a = 0; a < dim; ++a) jout[a][o] = (int32_t)rows[o * dim + a];
}

__global__ void k_tab_indices(int64_t n, int dim, int32_t* const* jin, int64_t* out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x)
    for (int a = 0; a < dim; ++a) out[o * dim + a] = jin[a][o];
}

__global__ void k_box_neighbors(int64_t n, AxBox ax, int64_t* down, int64_t* up) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    int j;
    int64_t dn, u;
    ax.at(o, j, dn, u);
    down[o] = dn;
    up[o] = u;
  }
}

__global__ void k_widen(int64_t n, const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                        int64_t* oa, int64_t* ob) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    oa[o] = a[o];
    ob[o] = b[o];
  }
}

// ---------------------------------------------------------------- host helpers

// Count tables for the hyperbolic cross.  Reachable budgets are floor(B/m).
static hp_status build_hyp_tables(int dim, int64_t B, std::vector<int64_t>& pref,
                                  std::vector<int64_t>& off, int64_t& total) {
  std::vector<char> reach(B + 1, 0);
  for (int64_t m = 1; m <= B; ) {
    int64_t v = B / m;
    reach[v] = 1;
    m = B / v + 1;
  }
  std::vector<int64_t> budgets;
  for (int64_t r = 1; r <= B; ++r) if (reach[r]) budgets.push_back(r);
  int64_t entries = 0;
  for (int d = 1; d < dim; ++d)
    for (int64_t r : budgets) entries += r + 1;
  if (entries > ((int64_t)1 << 27) || (int64_t)dim * (B + 1) > ((int64_t)1 << 28))
    return fail(HP_ERR_VALUE, "hyperbolic bound too large for the device rank tables");
  // cnt[d][r] for reachable r (indexed by r directly)
  const int64_t LIM = (int64_t)1 << 40;
  std::vector<std::vector<int64_t>> cnt(dim, std::vector<int64_t>(B + 1, 0));
  for (int64_t r : budgets) cnt[0][r] = 1;
  for (int d = 1; d < dim; ++d) {
    for (int64_t r : budgets) {
      int64_t s = 0;
      for (int64_t k = 0; k < r; ++k) {
        s += cnt[d - 1][r / (k + 1)];
        if (s > LIM) s = LIM;
      }
      cnt[d][r] = s;
    }
  }
  // total size = cnt(dim, B) = sum_k cnt(dim-1, B/(k+1))
  int64_t n = 0;
  if (dim == 1) n = B;
  else {
    for (int64_t k = 0; k < B; ++k) {
      n += cnt[dim - 1][B / (k + 1)];
      if (n > LIM) n = LIM;
    }
  }
  total = n;
  off.assign((size_t)dim * (B + 1), -1);
  pref.clear();
  pref.reserve(entries);
  for (int d = 1; d < dim; ++d) {
    for (int64_t r : budgets) {
      off[(size_t)d * (B + 1) + r] = (int64_t)pref.size();
      int64_t s = 0;
      for (int64_t k = 0; k <= r; ++k) {
        pref.push_back(s);
        if (k < r) s += cnt[d][r / (k + 1)];
      }
    }
  }
  if (pref.empty()) pref.push_back(0);
  return HP_OK;
}

static hp_status alloc_tables(hp_set_s* s, cudaStream_t st) {
  for (int a = 0; a < s->dim; ++a) {
    HP_CUDA(cudaMallocAsync(&s->d_j[a], std::max<int64_t>(s->n, 1) * sizeof(int32_t), st));
    HP_CUDA(cudaMallocAsync(&s->d_down[a], std::max<int64_t>(s->n, 1) * sizeof(int32_t), st));
    HP_CUDA(cudaMallocAsync(&s->d_up[a], std::max<int64_t>(s->n, 1) * sizeof(int32_t), st));
  }
  return HP_OK;
}

template <class T>
static hp_status upload_ptr_array(T* const* ptrs, int count, T*** dev, cudaStream_t st) {
  HP_CUDA(cudaMallocAsync((void**)dev, sizeof(T*) * count, st));
  HP_CUDA(cudaMemcpyAsync(*dev, ptrs, sizeof(T*) * count, cudaMemcpyHostToDevice, st));
  return HP_OK;
}

static void init_box(hp_set_s* s, int dim, int bound, int lo, int hi) {
  s->dim = dim;
  s->bound = bound;
  s->kind = HP_KIND_FULL;
  s->boxed = true;
  s->lo = lo;
  s->hi = hi;
  int64_t st = 1;
  for (int a = dim - 1; a >= 0; --a) {
    s->side[a] = (a == 0) ? (hi - lo) : (bound + 1);
    s->stride[a] = st;
    st *= s->side[a];
  }
  s->n = st;
}

}  // namespace hp

using namespace hp;

extern "C" {

int hp_abi_version(void) { return HP_ABI; }
int64_t hp_launch_count(void) { return hp::g_launches.load(); }
const char* hp_last_error(void) { return hp::g_last_error.c_str(); }
int hp_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

hp_status hp_set_create_full(int dim, int bound, void* stream, hp_set_t* out, int64_t* n_out) {
  return hp_set_create_slab(dim, bound, 0, bound + 1, stream, out, n_out);
}

hp_status hp_set_create_slab(int dim, int bound, int lo, int hi, void* stream, hp_set_t* out,
                             int64_t* n_out) {
  if (dim <= 0) return fail(HP_ERR_VALUE, "dimension must be positive, got " + std::to_string(dim));
  if (bound < 0) return fail(HP_ERR_VALUE, "bound must be nonnegative, got " + std::to_string(bound));
  if (dim > HP_MAXDIM) return fail(HP_ERR_VALUE, "dimension exceeds HP_MAXDIM");
  if (lo < 0 || hi > bound + 1 || lo >= hi) return fail(HP_ERR_VALUE, "bad slab range");
  double total = (double)(hi - lo);
  for (int a = 1; a < dim; ++a) total *= (double)(bound + 1);
  if (total > 9.0e18)
    return fail(HP_ERR_VALUE, "index set with " + std::to_string(total) +
                                  " elements exceeds the addressable range of this platform");
  auto* s = new hp_set_s();
  cudaGetDevice(&s->device);
  init_box(s, dim, bound, lo, hi);
  *out = s;
  if (n_out) *n_out = s->n;
  (void)stream;
  return HP_OK;
}

hp_status hp_set_create_hyperbolic(int dim, int bound, void* stream, hp_set_t* out, int64_t* n_out) {
  HP_NVTX("hp_set_create_hyperbolic");
  if (dim <= 0) return fail(HP_ERR_VALUE, "dimension must be positive, got " + std::to_string(dim));
  if (bound < 0) return fail(HP_ERR_VALUE, "bound must be nonnegative, got " + std::to_string(bound));
  if (dim > HP_MAXDIM) return fail(HP_ERR_VALUE, "dimension exceeds HP_MAXDIM");
  cudaStream_t st = as_stream(stream);
  auto* s = new hp_set_s();
  cudaGetDevice(&s->device);
  s->dim = dim;
  s->bound = bound;
  s->kind = HP_KIND_HYPERBOLIC;
  int64_t B = (int64_t)bound + 1;
  int64_t total = 0;
  hp_status rc = build_hyp_tables(dim, B, s->h_pref, s->h_off, total);
  if (rc != HP_OK) { delete s; return rc; }
  if (total >= ((int64_t)1 << 31) - 1) {
    delete s;
    return fail(HP_ERR_VALUE, "hyperbolic set too large for 32-bit device ordinals");
  }
  s->n = total;
  rc = alloc_tables(s, st);
  if (rc != HP_OK) { delete s; return rc; }
  HP_CUDA(cudaMallocAsync(&s->d_pref, s->h_pref.size() * sizeof(int64_t), st));
  HP_CUDA(cudaMallocAsync(&s->d_off, s->h_off.size() * sizeof(int64_t), st));
  HP_CUDA(cudaMemcpyAsync(s->d_pref, s->h_pref.data(), s->h_pref.size() * sizeof(int64_t),
                          cudaMemcpyHostToDevice, st));
  HP_CUDA(cudaMemcpyAsync(s->d_off, s->h_off.data(), s->h_off.size() * sizeof(int64_t),
                          cudaMemcpyHostToDevice, st));
  int32_t **dj = nullptr, **dd = nullptr, **du = nullptr;
  if ((rc = upload_ptr_array(s->d_j, dim, &dj, st)) != HP_OK) return rc;
  if ((rc = upload_ptr_array(s->d_down, dim, &dd, st)) != HP_OK) return rc;
  if ((rc = upload_ptr_array(s->d_up, dim, &du, st)) != HP_OK) return rc;
  if (s->n > 0) {
    k_hyp_unrank<<<grid_for(s->n, 256, 148 * 64), 256, 0, st>>>(s->n, dim, B, s->d_pref, s->d_off, dj);
    HP_LAUNCH_CHECK("k_hyp_unrank");
    k_hyp_neighbors<<<grid_for(s->n, 128, 148 * 64), 128, 0, st>>>(s->n, dim, B, s->d_pref, s->d_off,
                                                                    dj, dd, du);
    HP_LAUNCH_CHECK("k_hyp_neighbors");
  }
  HP_CUDA(cudaFreeAsync(dj, st));
  HP_CUDA(cudaFreeAsync(dd, st));
  HP_CUDA(cudaFreeAsync(du, st));
  *out = s;
  if (n_out) *n_out = s->n;
  return HP_OK;
}

hp_status hp_set_create_custom(int dim, int bound, const int64_t* indices_host, int64_t n,
                               void* stream, hp_set_t* out) {
  HP_NVTX("hp_set_create_custom");
  if (dim <= 0) return fail(HP_ERR_VALUE, "dimension must be positive, got " + std::to_string(dim));
  if (bound < 0) return fail(HP_ERR_VALUE, "bound must be nonnegative, got " + std::to_string(bound));
  if (dim > HP_MAXDIM) return fail(HP_ERR_VALUE, "dimension exceeds HP_MAXDIM");
  if (n < 0 || n >= ((int64_t)1 << 31) - 1) return fail(HP_ERR_VALUE, "bad custom set size");
  cudaStream_t st = as_stream(stream);
  auto* s = new hp_set_s();
  cudaGetDevice(&s->device);
  s->dim = dim;
  s->bound = bound;
  s->kind = HP_KIND_CUSTOM;
  s->n = n;
  s->h_indices.assign(indices_host, indices_host + n * dim);
  hp_status rc = alloc_tables(s, st);
  if (rc != HP_OK) { delete s; return rc; }
  int64_t* rows = nullptr;
  HP_CUDA(cudaMallocAsync(&rows, std::max<int64_t>(n * dim, 1) * sizeof(int64_t), st));
  if (n > 0)
    HP_CUDA(cudaMemcpyAsync(rows, s->h_indices.data(), n * dim * sizeof(int64_t),
                            cudaMemcpyHostToDevice, st));
  int32_t **dj = nullptr, **dd = nullptr, **du = nullptr;
  if ((rc = upload_ptr_array(s->d_j, dim, &dj, st)) != HP_OK) return rc;
  if ((rc = upload_ptr_array(s->d_down, dim, &dd, st)) != HP_OK) return rc;
  if ((rc = upload_ptr_array(s->d_up, dim, &du, st)) != HP_OK) return rc;
  if (n > 0) {
    k_custom_j<<<grid_for(n, 256), 256, 0, st>>>(n, dim, rows, dj);
    HP_LAUNCH_CHECK("k_custom_j");
    k_custom_neighbors<<<grid_for(n, 128), 128, 0, st>>>(n, dim, rows, dd, du);
    HP_LAUNCH_CHECK("k_custom_neighbors");
  }
  HP_CUDA(cudaFreeAsync(rows, st));
  HP_CUDA(cudaFreeAsync(dj, st));
  HP_CUDA(cudaFreeAsync(dd, st));
  HP_CUDA(cudaFreeAsync(du, st));
  // the host copy of the rows is needed by hp_set_position; it must outlive
  // the async upload, which it does (owned by the handle)
  HP_CUDA(cudaStreamSynchronize(st));
  *out = s;
  return HP_OK;
}

hp_status hp_set_info(hp_set_t s, int* dim, int* bound, int* kind, int64_t* n) {
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  if (dim) *dim = s->dim;
  if (bound) *bound = s->bound;
  if (kind) *kind = s->kind;
  if (n) *n = s->n;
  return HP_OK;
}

hp_status hp_set_indices(hp_set_t s, int64_t* out_dev, void* stream) {
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  cudaStream_t st = as_stream(stream);
  if (s->n == 0) return HP_OK;
  if (s->boxed) {
    int64_t* dstride = nullptr;
    int* dside = nullptr;
    HP_CUDA(cudaMallocAsync(&dstride, sizeof(int64_t) * s->dim, st));
    HP_CUDA(cudaMallocAsync(&dside, sizeof(int) * s->dim, st));
    HP_CUDA(cudaMemcpyAsync(dstride, s->stride, sizeof(int64_t) * s->dim, cudaMemcpyHostToDevice, st));
    HP_CUDA(cudaMemcpyAsync(dside, s->side, sizeof(int) * s->dim, cudaMemcpyHostToDevice, st));
    k_full_indices<<<grid_for(s->n, 256), 256, 0, st>>>(s->n, s->dim, dstride, dside, s->lo, out_dev);
    HP_LAUNCH_CHECK("k_full_indices");
    HP_CUDA(cudaFreeAsync(dstride, st));
    HP_CUDA(cudaFreeAsync(dside, st));
    // the host arrays are members of the handle, safe for the async copy
    return HP_OK;
  }
  int32_t** dj = nullptr;
  hp_status rc = upload_ptr_array(s->d_j, s->dim, &dj, st);
  if (rc != HP_OK) return rc;
  k_tab_indices<<<grid_for(s->n, 256), 256, 0, st>>>(s->n, s->dim, dj, out_dev);
  HP_LAUNCH_CHECK("k_tab_indices");
  HP_CUDA(cudaFreeAsync(dj, st));
  return HP_OK;
}

hp_status hp_neighbor_tables(hp_set_t s, int axis, int64_t* down_dev, int64_t* up_dev, void* stream) {
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  if (axis < 1 || axis > s->dim)
    return fail(HP_ERR_VALUE, "axis must satisfy 1 <= axis <= " + std::to_string(s->dim) +
                                  ", got " + std::to_string(axis));
  cudaStream_t st = as_stream(stream);
  if (s->n == 0) return HP_OK;
  int a = axis - 1;
  if (s->boxed) {
    k_box_neighbors<<<grid_for(s->n, 256), 256, 0, st>>>(s->n, s->box(a), down_dev, up_dev);
    HP_LAUNCH_CHECK("k_box_neighbors");
  } else {
    k_widen<<<grid_for(s->n, 256), 256, 0, st>>>(s->n, s->d_down[a], s->d_up[a], down_dev, up_dev);
    HP_LAUNCH_CHECK("k_widen");
  }
  return HP_OK;
}

hp_status hp_set_position(hp_set_t s, const int64_t* j, int64_t* ord_out) {
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  *ord_out = -1;
  int dim = s->dim;
  for (int a = 0; a < dim; ++a) if (j[a] < 0) return HP_OK;
  if (s->boxed) {
    int64_t o = 0;
    for (int a = 0; a < dim; ++a) {
      int64_t jl = j[a] - (a == 0 ? s->lo : 0);
      if (jl < 0 || jl >= s->side[a]) return HP_OK;
      o += jl * s->stride[a];
    }
    *ord_out = o;
    return HP_OK;
  }
  if (s->kind == HP_KIND_HYPERBOLIC) {
    int64_t B = (int64_t)s->bound + 1, r = B, ord = 0;
    for (int l = 0; l < dim; ++l) {
      int64_t k = j[l];
      if (k + 1 > r) return HP_OK;
      if (l == dim - 1) { *ord_out = ord + k; return HP_OK; }
      int d = dim - 1 - l;
      ord += s->h_pref[s->h_off[(size_t)d * (B + 1) + r] + k];
      r /= (k + 1);
    }
    return HP_OK;
  }
  // custom: binary search on the host copy
  int64_t lo = 0, hi = s->n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) >> 1;
    int c = 0;
    for (int l = 0; l < dim && c == 0; ++l) {
      int64_t x = s->h_indices[mid * dim + l];
      c = (x < j[l]) ? -1 : (x > j[l] ? 1 : 0);
    }
    if (c == 0) { *ord_out = mid; return HP_OK; }
    if (c < 0) lo = mid + 1; else hi = mid - 1;
  }
  return HP_OK;
}

hp_status hp_set_destroy(hp_set_t s) {
  if (!s) return HP_OK;
  cudaDeviceSynchronize();
  for (int a = 0; a < HP_MAXDIM; ++a) {
    if (s->d_j[a]) cudaFree(s->d_j[a]);
    if (s->d_down[a]) cudaFree(s->d_down[a]);
    if (s->d_up[a]) cudaFree(s->d_up[a]);
    if (s->d_perm[a]) cudaFree(s->d_perm[a]);
    if (s->d_win[a]) cudaFree(s->d_win[a]);
  }
  if (s->d_sqtab) cudaFree(s->d_sqtab);
  if (s->d_jsum) cudaFree(s->d_jsum);
  if (s->d_pref) cudaFree(s->d_pref);
  if (s->d_off) cudaFree(s->d_off);
  if (s->fg_basis) cudaFree(s->fg_basis);
  if (s->fg_tiles) cudaFree(s->fg_tiles);
  if (s->fg_tiles4) cudaFree(s->fg_tiles4);
  delete s;
  return HP_OK;
}

}  // extern "C"
