// Full-cube <-> subset maps on the device: restrict / extend (index_set.py:296-319), the fused
// reduction-error components |W_set v - R W_full E v| (error_lab.py:114-130) and the
// reduction-local mask (error_lab.py:133-148).
//
// A member j of a subset sits at ordinal  pos(j) = sum_l j_l (bound+1)^(N-l)  of the full cube
// of the same (dim, bound) (index_set.py:296-305).  The reference materialises the subset's
// indices on the host and forms pos by a matrix product; here pos is computed per element from
// the set's device j-tables (tabled sets) or stride arithmetic (boxes), so restrict is one
// gather pass and extend one zero-fill plus one scatter pass, both HBM-bound.
#include <algorithm>

#include "hp_common.cuh"

namespace hp {

struct PosMap {
  int dim;
  int boxed;
  int64_t cube_stride[HP_MAXDIM];  // full-cube strides (bound+1)^(N-1-l)
  // boxes (full / slab subsets): local strides and sides, axis-0 offset
  int64_t stride[HP_MAXDIM];
  int side[HP_MAXDIM];
  int lo;
  const int32_t* jv[HP_MAXDIM];  // tabled sets
  __device__ __forceinline__ int j(int a, int64_t o) const {
    if (boxed) return (int)((o / stride[a]) % side[a]) + (a == 0 ? lo : 0);
    return __ldg(jv[a] + o);
  }
  __device__ __forceinline__ int64_t pos(int64_t o) const {
    int64_t p = 0;
#pragma unroll 4
    for (int a = 0; a < dim; ++a) p += (int64_t)j(a, o) * cube_stride[a];
    return p;
  }
};

static PosMap pos_map(const hp_set_s* s) {
  PosMap m{};
  m.dim = s->dim;
  m.boxed = s->boxed ? 1 : 0;
  m.lo = s->lo;
  int64_t st = 1;
  for (int a = s->dim - 1; a >= 0; --a) {
    m.cube_stride[a] = st;
    st *= (int64_t)s->bound + 1;
    m.stride[a] = s->stride[a];
    m.side[a] = s->side[a];
    m.jv[a] = s->d_j[a];
  }
  return m;
}

template <class T>
__global__ void k_restrict(int64_t n, int64_t nfull, int64_t batch, PosMap m, const T* __restrict__ full,
                           T* __restrict__ sub) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = m.pos(o);
    HP_DCHECK(p >= 0 && p < nfull);
    for (int64_t b = 0; b < batch; ++b) sub[b * n + o] = __ldg(full + b * nfull + p);
  }
}

template <class T>
__global__ void k_extend(int64_t n, int64_t nfull, int64_t batch, PosMap m, const T* __restrict__ sub,
                         T* __restrict__ full) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = m.pos(o);
    HP_DCHECK(p >= 0 && p < nfull);
    for (int64_t b = 0; b < batch; ++b) full[b * nfull + p] = __ldg(sub + b * n + o);
  }
}

__device__ __forceinline__ double absdiff(double a, double b) { return fabs(a - b); }
__device__ __forceinline__ double absdiff(double2 a, double2 b) {
  // numpy's abs of a complex difference: hypot of the parts
  return hypot(a.x - b.x, a.y - b.y);
}

template <class T>
__global__ void k_reduction_components(int64_t n, PosMap m, const T* __restrict__ on_set,
                                       const T* __restrict__ on_full, double* __restrict__ comp) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
    comp[o] = absdiff(__ldg(on_set + o), __ldg(on_full + m.pos(o)));
}

// mask[o] = 1 iff j(o) + r lies in the set for every degree tuple r of the term list.  Sets are
// downward closed, so j + r is a member iff the up-walk r_1 e_1, then r_2 e_2, ... from j stays
// in the set (every point of the walk is <= j + r componentwise); boxes test the bound directly.
struct MaskTerms {
  int nterms;
  const int32_t* deg;  // device (nterms x dim)
};
__global__ void k_local_mask(int64_t n, int dim, int boxed, PosMap m, int bound, AxTab* __restrict__ tabs,
                             MaskTerms t, uint8_t* __restrict__ mask) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int i = 0; ok && i < t.nterms; ++i) {
      const int32_t* r = t.deg + (int64_t)i * dim;
      if (boxed) {
        for (int a = 0; a < dim && ok; ++a) ok = m.j(a, o) + __ldg(r + a) <= bound;
        continue;
      }
      int64_t q = o;
      for (int a = 0; a < dim && ok; ++a) {
        const int ra = __ldg(r + a);
        for (int k = 0; k < ra && ok; ++k) {
          q = __ldg(tabs[a].up + q);
          ok = q >= 0;
        }
      }
    }
    mask[o] = ok ? 1 : 0;
  }
}

// make_decay_vector's entries (error_lab.py:43-56): prod_l max(j_l, 1)^(-beta), normalised by the
// caller's device norm pass
__global__ void k_decay(int64_t n, int dim, PosMap m, double mbeta, double* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    double p = 1.0;
    for (int a = 0; a < dim; ++a) p *= pow((double)max(m.j(a, o), 1), mbeta);
    out[o] = p;
  }
}

static hp_status check_pair(const hp_set_s* sub, const hp_set_s* full) {
  if (!sub || !full) return fail(HP_ERR_VALUE, "null set handle");
  if (full->kind != HP_KIND_FULL || !full->boxed || full->lo != 0 || full->hi != full->bound + 1)
    return fail(HP_ERR_VALUE, "target of restrict/extend must be a full cube");
  if (sub->dim != full->dim || sub->bound != full->bound)
    return fail(HP_ERR_VALUE, "set mismatch: subset has (dim, bound) = (" + std::to_string(sub->dim) + ", " +
                                  std::to_string(sub->bound) + "), full cube has (" + std::to_string(full->dim) +
                                  ", " + std::to_string(full->bound) + ")");
  return HP_OK;
}

}  // namespace hp

using namespace hp;

extern "C" {

hp_status hp_restrict(hp_set_t sub, hp_set_t full, int dtype, const void* full_dev, void* sub_dev, int64_t batch,
                      void* stream) {
  HP_NVTX("hp_restrict");
  hp_status rc = check_pair(sub, full);
  if (rc) return rc;
  if (sub->n == 0 || batch <= 0) return HP_OK;
  cudaStream_t st = as_stream(stream);
  const PosMap m = pos_map(sub);
  const int grid = grid_for(sub->n, 256);
  if (dtype == HP_C128)
    k_restrict<double2><<<grid, 256, 0, st>>>(sub->n, full->n, batch, m, (const double2*)full_dev, (double2*)sub_dev);
  else
    k_restrict<double><<<grid, 256, 0, st>>>(sub->n, full->n, batch, m, (const double*)full_dev, (double*)sub_dev);
  HP_LAUNCH_CHECK("k_restrict");
  return HP_OK;
}

hp_status hp_extend(hp_set_t sub, hp_set_t full, int dtype, const void* sub_dev, void* full_dev, int64_t batch,
                    void* stream) {
  HP_NVTX("hp_extend");
  hp_status rc = check_pair(sub, full);
  if (rc) return rc;
  if (batch <= 0) return HP_OK;
  cudaStream_t st = as_stream(stream);
  const size_t es = dtype == HP_C128 ? 16 : 8;
  HP_CUDA(cudaMemsetAsync(full_dev, 0, (size_t)full->n * batch * es, st));
  if (sub->n == 0) return HP_OK;
  const PosMap m = pos_map(sub);
  const int grid = grid_for(sub->n, 256);
  if (dtype == HP_C128)
    k_extend<double2><<<grid, 256, 0, st>>>(sub->n, full->n, batch, m, (const double2*)sub_dev, (double2*)full_dev);
  else
    k_extend<double><<<grid, 256, 0, st>>>(sub->n, full->n, batch, m, (const double*)sub_dev, (double*)full_dev);
  HP_LAUNCH_CHECK("k_extend");
  return HP_OK;
}

hp_status hp_reduction_components(hp_set_t sub, hp_set_t full, int dtype, const void* on_set_dev,
                                  const void* on_full_dev, double* comp_dev, void* stream) {
  HP_NVTX("hp_reduction_components");
  hp_status rc = check_pair(sub, full);
  if (rc) return rc;
  if (sub->n == 0) return HP_OK;
  cudaStream_t st = as_stream(stream);
  const PosMap m = pos_map(sub);
  const int grid = grid_for(sub->n, 256);
  if (dtype == HP_C128)
    k_reduction_components<double2><<<grid, 256, 0, st>>>(sub->n, m, (const double2*)on_set_dev,
                                                           (const double2*)on_full_dev, comp_dev);
  else
    k_reduction_components<double><<<grid, 256, 0, st>>>(sub->n, m, (const double*)on_set_dev,
                                                          (const double*)on_full_dev, comp_dev);
  HP_LAUNCH_CHECK("k_reduction_components");
  return HP_OK;
}

hp_status hp_decay_vector(hp_set_t s, int beta, double* out_dev, void* stream) {
  HP_NVTX("hp_decay_vector");
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  if (beta < 1) return fail(HP_ERR_VALUE, "beta must be a positive integer, got " + std::to_string(beta));
  if (s->n == 0) return HP_OK;
  k_decay<<<grid_for(s->n, 256), 256, 0, as_stream(stream)>>>(s->n, s->dim, pos_map(s), -(double)beta, out_dev);
  HP_LAUNCH_CHECK("k_decay");
  return HP_OK;
}

hp_status hp_reduction_local_mask(hp_set_t s, const int32_t* degrees_host, int nterms, uint8_t* mask_dev,
                                  void* stream) {
  HP_NVTX("hp_reduction_local_mask");
  if (!s) return fail(HP_ERR_VALUE, "null set handle");
  if (nterms < 0) return fail(HP_ERR_VALUE, "nterms must be nonnegative");
  for (int64_t i = 0; i < (int64_t)nterms * s->dim; ++i)
    if (degrees_host[i] < 0) return fail(HP_ERR_VALUE, "negative Chebyshev degree in term list");
  if (s->n == 0) return HP_OK;
  cudaStream_t st = as_stream(stream);
  int32_t* deg = nullptr;
  AxTab* tabs = nullptr;
  const size_t db = std::max<size_t>((size_t)nterms * s->dim, 1) * sizeof(int32_t);
  HP_CUDA(cudaMallocAsync(&deg, db, st));
  HP_CUDA(cudaMallocAsync(&tabs, HP_MAXDIM * sizeof(AxTab), st));
  AxTab ht[HP_MAXDIM] = {};
  if (!s->boxed)
    for (int a = 0; a < s->dim; ++a) ht[a] = s->tab(a);
  if (nterms) HP_CUDA(cudaMemcpyAsync(deg, degrees_host, (size_t)nterms * s->dim * sizeof(int32_t),
                                      cudaMemcpyHostToDevice, st));
  HP_CUDA(cudaMemcpyAsync(tabs, ht, sizeof(ht), cudaMemcpyHostToDevice, st));
  k_local_mask<<<grid_for(s->n, 256), 256, 0, st>>>(s->n, s->dim, s->boxed ? 1 : 0, pos_map(s), s->bound, tabs,
                                                    MaskTerms{nterms, deg}, mask_dev);
  HP_LAUNCH_CHECK("k_local_mask");
  // the host arrays are staged by stream-ordered copies; free after the kernel on the same stream
  HP_CUDA(cudaFreeAsync(deg, st));
  HP_CUDA(cudaFreeAsync(tabs, st));
  HP_CUDA(cudaStreamSynchronize(st));  // pageable host sources: keep them alive until copied
  return HP_OK;
}

}  // extern "C"
