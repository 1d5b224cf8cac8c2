// Host-side representation of a polynomial-evaluation program: a linear
// list of kernel launches over named vector buffers (the input v, the output
// y and workspace slots).  Built once per call from the term list; executing
// it issues only stream-ordered launches, so it can be graph-captured.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "hp_common.cuh"

namespace hp {

enum { BUF_V = -10, BUF_Y = -9, BUF_SLOT0 = 0 };
inline int slot(int i) { return BUF_SLOT0 + i; }

enum OpKind { OP_ZERO, OP_COPY, OP_AXPY, OP_FIRST, OP_STEP, OP_OSC };

struct Op {
  OpKind kind;
  int axis = 0;   // 0-based axis
  int a = -100;   // src / wm
  int b = -100;   // wp (step)
  int dst = -100;
  int acc = -100; // harvest target or -100
  double hw = 0.0;
  static Op zero(int dst) { Op o; o.kind = OP_ZERO; o.dst = dst; return o; }
  static Op copy(int dst, int src) { Op o; o.kind = OP_COPY; o.dst = dst; o.a = src; return o; }
  static Op axpy(int dst, int src, double c) { Op o; o.kind = OP_AXPY; o.dst = dst; o.a = src; o.hw = c; return o; }
  static Op first(int axis, int src, int dst) { Op o; o.kind = OP_FIRST; o.axis = axis; o.a = src; o.dst = dst; return o; }
  static Op step(int axis, int wm, int wp, int dst) {
    Op o; o.kind = OP_STEP; o.axis = axis; o.a = wm; o.b = wp; o.dst = dst; return o;
  }
  static Op osc(int dst, int v) { Op o; o.kind = OP_OSC; o.dst = dst; o.a = v; return o; }
};

struct Program {
  std::vector<Op> ops;
  int nslots = 0;
  int xapps = 0;
};

struct Term {
  int r[HP_MAXDIM];
  double alpha;
};

std::vector<Term> make_terms(int dim, const int32_t* degrees, const double* coeffs, int nterms);
Program build_program(int dim, const std::vector<Term>& terms, int flags, const int32_t* axis_order);

// Optional fused inner product <v, y> of the matvec input and output
// (complex, batch 1): the kernel that writes the final y also writes one
// partial sum per CTA into `partial`; `n` is set to the number written.
// Used by the Lanczos recurrence to avoid a separate pass over v and y.
struct DotOut {
  double2* partial = nullptr;
  int capacity = 0;
  int n = 0;
};
constexpr int HP_DOT_CAPACITY = 1 << 15;

template <class T>
hp_status run_program(const hp_set_s* s, const Program& p, double halfwidth, const T* v, T* y,
                      int64_t batch, T* ws, size_t ws_bytes, cudaStream_t st, DotOut* dot = nullptr);
template <class T>
hp_status launch_square(const hp_set_s* s, const T* v, T* out, int64_t batch, cudaStream_t st);
template <class T>
hp_status check_finite(const T* y, int64_t total, cudaStream_t st, bool* ok);

// fused full-cube evaluator (hp_fullgrid.cu); *done = false when the
// set / term structure is not covered and the generic program must run
size_t fullgrid_workspace_bytes(const hp_set_s* s, const std::vector<Term>& terms, int dtype,
                                int64_t batch, int flags);
hp_status fullgrid_apply(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                         const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                         cudaStream_t st, bool* done, DotOut* dot = nullptr, double sq = 0.0);

hp_status fullgrid_apply_planes(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                                const void* in, void* out, int plo, int phi, int flags, void* ws, size_t ws_bytes,
                                cudaStream_t st, bool* done, double* dot_accum = nullptr, double sq = 0.0);
// per-device host<->device copy streams of the streamed entry points (hp_fullgrid.cu)
hp_status copy_streams(cudaStream_t* in, cudaStream_t* out);
hp_status fullgrid_apply_streamed(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                                  const void* in_host, void* out_host, void* in_dev, void* out_dev, int flags,
                                  void* ws, size_t ws_bytes, cudaStream_t st, bool* done);

// fullgrid_apply, and where the whole polynomial is outside the fused class of an N = 4 box: its
// fused part (constants, even single-axis terms, T_1 x T_1 pairs) through the fused evaluator and
// only the remaining terms through level passes accumulated onto y -- when the level planner
// prices that below the whole polynomial
hp_status fullgrid_apply_split(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                               const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                               cudaStream_t st, bool* done, DotOut* dot = nullptr, double sq = 0.0);

// level-fused evaluator (hp_level.cu): complex vectors, degrees <= 4
constexpr int HP_LV_ACCUMULATE = 1 << 16;  // internal flag of level_apply: y += W v instead of y = W v
// vector passes the level planner charges for the polynomial (< 0: not covered)
double level_plan_cost(int dim, const std::vector<Term>& terms);
size_t level_workspace_bytes(const hp_set_s* s, const std::vector<Term>& terms, int dtype, int64_t batch);
hp_status level_apply(const hp_set_s* s, const std::vector<Term>& terms, double halfwidth, int dtype,
                      const void* in, void* out, int64_t batch, int flags, void* ws, size_t ws_bytes,
                      cudaStream_t st, bool* done, DotOut* dot = nullptr);

}  // namespace hp
