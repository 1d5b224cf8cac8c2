/*
 * hprop_b200 -- C ABI of the B200-native matrix-free Galerkin matvec.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `hprop` 0.1.0 (/root/reference/pkg/src/hprop).  The reference is pure
 * Python/numpy and has no FFI; its seams are the duck-typed objects listed
 * below.  Every entry point here replaces one reference routine (cited as
 * <module>.py:<lines>) and is bound from Python through ctypes by
 * paper_1403_3511_b200/_native.py (see INTEGRATION.md for the binding a
 * maintainer adds to hprop itself).
 *
 * Conventions
 *  - every function returns an hp_status (0 = HP_OK); hp_last_error() gives
 *    the message of the last failure on the calling thread;
 *  - pointers named *_dev are device pointers owned by the caller (PyTorch
 *    tensors on the Python side); the library only borrows them for the
 *    duration of the call; pointers named *_host are host memory;
 *  - `stream` is a cudaStream_t passed as void*; all device work is
 *    stream-ordered and asynchronous unless stated otherwise;
 *  - coefficient vectors are `batch` consecutive vectors of n scalars in the
 *    set's canonical (lexicographic) order; dtype HP_F64 (double) or
 *    HP_C128 (interleaved re/im doubles, i.e. numpy complex128);
 *  - axes are 1-based as in the reference API;
 *  - set handles are immutable after creation and may be shared by
 *    concurrent callers that use distinct streams, outputs and workspaces
 *    (fast_apply.py:36-37).
 */
#ifndef HPROP_B200_H
#define HPROP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int hp_status;
enum {
  HP_OK = 0,
  HP_ERR_VALUE = 1,     /* maps to Python ValueError   */
  HP_ERR_RUNTIME = 2,   /* maps to Python RuntimeError */
  HP_ERR_CUDA = 3,      /* CUDA failure                */
  HP_ERR_NOMEM = 4,     /* workspace too small / OOM   */
  HP_ERR_KEY = 5        /* maps to Python KeyError     */
};

enum { HP_F64 = 0, HP_C128 = 1 };
enum { HP_KIND_FULL = 0, HP_KIND_HYPERBOLIC = 1, HP_KIND_CUSTOM = 2 };

/* flags for hp_apply_polynomial */
enum {
  HP_ADD_OSC = 1,       /* add sum_l (j_l + 1/2) v: apply_hamiltonian (fast_apply.py:195-198) */
  HP_REF_ORDER = 2,     /* reproduce the reference evaluation order bit for bit (fast_apply.py:110-193) */
  HP_CHECK_FINITE = 4   /* raise HP_ERR_RUNTIME on non-finite output (fast_apply.py:316-318); synchronises */
};

typedef struct hp_set_s* hp_set_t;

int hp_abi_version(void);
const char* hp_last_error(void);
int hp_device_count(void);
/* number of kernels this library has launched in the process so far */
int64_t hp_launch_count(void);
/* Compiles (NVRTC, no device needed, nothing launched) the run-time specialised level kernels
 * of the polynomial `degrees`/`coeffs` (as in hp_apply_polynomial) for both set kinds (tabled,
 * boxed); *nkernels_out = kernels compiled.  HP_ERR_RUNTIME if NVRTC is unavailable or a
 * compilation fails.  The build check of the path hp_apply_polynomial takes on large sets
 * (fast_apply.py:110-164; csrc/hp_level_jit.cu). */
/* level kernels this process has compiled at run time so far (0: every level ran the library's
 * interpreted kernel) */
int hp_level_jit_kernels(void);
hp_status hp_level_jit_selftest(int dim, const int32_t* degrees, const double* coeffs, int nterms,
                                int* nkernels_out);

/* ---- index sets (index_set.py) ------------------------------------------ */

/* build_full(dim, bound) -- index_set.py:144-154.  Ordinal of j is
 * sum_l j_l (bound+1)^(dim-l); nothing is materialised. */
hp_status hp_set_create_full(int dim, int bound, void* stream, hp_set_t* out, int64_t* n_out);

/* Slab of a full cube: planes j1 in [lo, hi) (multi-GPU shards, §8(e)).
 * Neighbours across the slab faces are absent; j1 keeps its global value. */
hp_status hp_set_create_slab(int dim, int bound, int lo, int hi, void* stream,
                             hp_set_t* out, int64_t* n_out);

/* build_hyperbolic(dim, bound) -- index_set.py:157-181.  Enumerated on the
 * device by budget-count unranking, bit-exact with the reference order;
 * neighbour tables are built by ranking j +- e_l. */
hp_status hp_set_create_hyperbolic(int dim, int bound, void* stream, hp_set_t* out,
                                   int64_t* n_out);

/* from_indices / IndexSet(dim, bound, kind, indices) -- index_set.py:46-65,
 * 184-214.  indices_host: n x dim, strictly lexicographically sorted,
 * downward closed (validated by the caller, as the reference does). */
hp_status hp_set_create_custom(int dim, int bound, const int64_t* indices_host, int64_t n,
                               void* stream, hp_set_t* out);

hp_status hp_set_info(hp_set_t s, int* dim, int* bound, int* kind, int64_t* n);

/* IndexSet.indices (index_set.py:60): n x dim int64, written to device memory. */
hp_status hp_set_indices(hp_set_t s, int64_t* out_dev, void* stream);

/* IndexSet.neighbor_ordinals(axis) -- index_set.py:104-130: int64 ordinals,
 * -1 where absent. */
hp_status hp_neighbor_tables(hp_set_t s, int axis, int64_t* down_dev, int64_t* up_dev,
                             void* stream);

/* Ordinal of one multi-index (IndexSet.position, index_set.py:86-88);
 * *ord_out = -1 if absent.  Host-side, no device work. */
hp_status hp_set_position(hp_set_t s, const int64_t* index_host, int64_t* ord_out);

hp_status hp_set_destroy(hp_set_t s);

/* ---- matvec (fast_apply.py) --------------------------------------------- */

/* PolynomialApplier.apply_coordinate / direct_op -- fast_apply.py:59-65, 273-278 */
hp_status hp_apply_coordinate(hp_set_t s, int axis, int dtype, const void* in_dev,
                              void* out_dev, int64_t batch, void* stream);

/* cheb_of_coordinate_apply -- fast_apply.py:281-302: T_degree(X_axis/L) v */
size_t hp_cheb_workspace_bytes(hp_set_t s, int dtype, int64_t batch);
hp_status hp_cheb_apply(hp_set_t s, int axis, int degree, double halfwidth, int dtype,
                        const void* in_dev, void* out_dev, int64_t batch, void* workspace_dev,
                        size_t workspace_bytes, void* stream);

/* apply_polynomial / apply_hamiltonian -- fast_apply.py:110-198.
 * degrees_host: nterms x dim (any integer degrees >= 0), coeffs_host: nterms.
 * axis_order_host: NULL for the defined order, else a permutation of 1..dim
 * (first entry applied first; disables grouping, fast_apply.py:121-125). */
size_t hp_poly_workspace_bytes(hp_set_t s, const int32_t* degrees_host, int nterms, int dtype,
                               int64_t batch, int flags);
hp_status hp_apply_polynomial(hp_set_t s, const int32_t* degrees_host, const double* coeffs_host,
                              int nterms, double halfwidth, int dtype, const void* in_dev,
                              void* out_dev, int64_t batch, int flags,
                              const int32_t* axis_order_host, void* workspace_dev,
                              size_t workspace_bytes, void* stream);

/* apply_polynomial on HOST-resident vectors (the reference's numpy arrays live in host memory:
 * fast_apply.py:110-164 takes and returns ndarrays).  in_host/out_host: n*batch elements, pinned
 * for overlap; in_dev/out_dev: device buffers of the same size.  On full cubes of the fused
 * class the copies run in j1-plane chunks on internal streams, overlapped with the kernels
 * (input chunk k+1 in flight while chunk k is computed and chunk k-1 copied out); otherwise
 * whole-vector copies around hp_apply_polynomial.  Ordered on `stream`; returns once queued. */
hp_status hp_apply_polynomial_streamed(hp_set_t s, const int32_t* degrees_host, const double* coeffs_host,
                                       int nterms, double halfwidth, int dtype, const void* in_host,
                                       void* out_host, void* in_dev, void* out_dev, int64_t batch,
                                       int flags, void* workspace_dev, size_t workspace_bytes,
                                       void* stream);

/* apply_polynomial restricted to the output j1-planes [plane_lo, plane_hi) of a full cube or
 * slab (plane indices local to the set).  Only input planes plane_lo-4 .. plane_hi+3 are read
 * (4 = the band radius of the fused evaluator), so a slab-sharded matvec can compute the
 * planes that need no halo while the halo planes are in flight; the other
 * output planes are not written.  HP_ERR_VALUE outside the fused full-cube class (complex
 * vectors, batch 1, even single-axis bands, at most one x1*x2-type coupling); an empty range
 * only answers that question. */
hp_status hp_apply_polynomial_planes(hp_set_t s, const int32_t* degrees_host, const double* coeffs_host,
                                     int nterms, double halfwidth, int dtype, const void* in_dev,
                                     void* out_dev, int plane_lo, int plane_hi, int flags,
                                     void* workspace_dev, size_t workspace_bytes, void* stream);
/* The same, and dot_dev[0..1] += sum over the output planes [plane_lo, plane_hi) of the rows of
   v^H A v formed inside the kernel (A symmetric: conj(v_p) . row p split at plane p, no second
   read of v).  Summed over the ranks of a slab decomposition (each owning its planes) it is the
   global v^H A v: the Lanczos alpha of sharded_propagate (krylov_propagator.py:81). */
hp_status hp_apply_polynomial_planes_dot(hp_set_t s, const int32_t* degrees_host, const double* coeffs_host,
                                         int nterms, double halfwidth, int dtype, const void* in_dev,
                                         void* out_dev, int plane_lo, int plane_hi, int flags, double* dot_dev,
                                         void* workspace_dev, size_t workspace_bytes, void* stream);

/* The same with the harmonic confinement q * sum_l x_l^2 (fast_apply.py:229-245, error_lab.py:176-183)
 * folded into the fused kernel's single-axis bands, so A(t) v of a harmonic_part != 0 potential stays
 * one launch with its in-kernel dot (slab-sharded propagation). */
hp_status hp_apply_hamiltonian_planes_dot(hp_set_t s, const int32_t* degrees_host, const double* coeffs_host,
                                          int nterms, double halfwidth, double q, int dtype, const void* in_dev,
                                          void* out_dev, int plane_lo, int plane_hi, int flags, double* dot_dev,
                                          void* workspace_dev, size_t workspace_bytes, void* stream);

/* apply_square_sum -- fast_apply.py:202-245 (exact restricted sum_l x_l^2) */
hp_status hp_square_sum(hp_set_t s, int dtype, const void* in_dev, void* out_dev,
                        int64_t batch, void* stream);

/* ---- Lanczos scalars on the device for distributed callers ------------------------
 * The slab-sharded propagation (sharding.sharded_propagate) runs the scaled Lanczos recurrence of
 * krylov_propagator.py:58-104 with every scalar -- alpha_k, beta_k, the basis scales, breakdown
 * (beta <= tol truncates m, :90-93), the QL + exp column (:107-186) -- in an opaque device state,
 * so no iteration waits on the host; cross-rank sums of the per-rank partials are formed by the
 * caller (NCCL all-gather + rank-ordered sum) and handed in as device (re, im) pairs. */
size_t hp_lz_state_bytes(void);
hp_status hp_lz_init(void* state_dev, int m, void* stream);
/* what: 1 = ||y||^2 (sets nrm0, scale_0), 6 = u_k^H A u_k (alpha_k = scale_k^2 re), 7 = ||w_{k+1}||^2
 * (beta_k, scale_{k+1}, or breakdown) */
hp_status hp_lz_set(void* state_dev, int k, int what, const double* value_dev, double tol, void* stream);
/* w_{k+1} = s_k z - alpha_k s_k w_k - beta_{k-1} s_{k-1} w_{k-1} with this rank's ||w_{k+1}||^2
 * partial written to nrm2_out_dev[0]; a no-op past a breakdown.  ws: hp_reduce_workspace_bytes */
hp_status hp_lz_update(int64_t n, const void* z_dev, const void* wk_dev, const void* wkm1_dev, void* wn_dev,
                       const void* state_dev, int k, double* nrm2_out_dev, void* ws, void* stream);
hp_status hp_lz_expm(void* state_dev, double tau, void* stream);
/* out = nrm0 sum_{k < m_eff} col_k s_k w_k over m basis pointers (out may alias vecs[0]) */
hp_status hp_lz_combine(int64_t n, int m, const void* const* vecs_host, const void* state_dev, void* out_dev,
                        void* stream);
/* diag = {m_eff, hermiticity defect, breakdown_at (-1), QL failure}; alpha/beta may be null */
hp_status hp_lz_diag(const void* state_dev, double* diag_dev, double* alpha_dev, double* beta_dev, void* stream);

/* ---- full cube <-> subset maps (index_set.py:296-319, error_lab.py:114-148) ---- */

/* restrict -- index_set.py:308-311: sub[o] = full[pos(o)] for each of `batch` vectors, pos(j) =
 * sum_l j_l (bound+1)^(dim-l) computed on the device from the subset's tables.  `full` must be
 * a full cube (not a slab) of the subset's (dim, bound): HP_ERR_VALUE "target of
 * restrict/extend must be a full cube" / "set mismatch: ..." otherwise. */
hp_status hp_restrict(hp_set_t subset, hp_set_t full, int dtype, const void* full_dev, void* sub_dev,
                      int64_t batch, void* stream);

/* extend -- index_set.py:314-319: full = 0, then full[pos(o)] = sub[o]. */
hp_status hp_extend(hp_set_t subset, hp_set_t full, int dtype, const void* sub_dev, void* full_dev,
                    int64_t batch, void* stream);

/* reduction_error's components -- error_lab.py:114-130: comp[o] = |on_set[o] - on_full[pos(o)]|
 * (float64 out; the restrict and the difference in one pass). */
hp_status hp_reduction_components(hp_set_t subset, hp_set_t full, int dtype, const void* on_set_dev,
                                  const void* on_full_dev, double* comp_dev, void* stream);

/* make_decay_vector's unnormalised entries -- error_lab.py:43-56: out[o] = prod_l max(j_l, 1)^(-beta)
 * (float64, the set's order); HP_ERR_VALUE for beta < 1. */
hp_status hp_decay_vector(hp_set_t s, int beta, double* out_dev, void* stream);

/* reduction_local_mask -- error_lab.py:133-148: mask[o] = 1 iff j(o) + r is in the set for every
 * degree tuple r of the term list (up-walks through the neighbour tables; bound test on cubes).
 * Synchronises the stream. */
hp_status hp_reduction_local_mask(hp_set_t s, const int32_t* degrees_host, int nterms, uint8_t* mask_dev,
                                  void* stream);

/* ---- Lanczos / Magnus (krylov_propagator.py) ---------------------------- */

/* One exponential Magnus step y <- exp(-i h B) y via an m-step Lanczos
 * factorisation (krylov_propagator.py:58-104, 107-186, 215-244), entirely on
 * the device with no host synchronisation.  scheme 0 = midpoint (B = A(t+h/2),
 * terms set 1), 1 = gl2 (two time points, terms sets 1 and 2).
 * A(t) = D + W_pol(t) + q * square_sum (error_lab.py:173-185) with D the
 * oscillator diagonal.  y_dev: complex128 n (in/out).
 * diag_dev (optional, 4 doubles): [m_eff, hermiticity_defect, breakdown_at or -1, ql_failed]. */
size_t hp_magnus_workspace_bytes(hp_set_t s, int scheme, const int32_t* degrees1_host,
                                 int nterms1, const int32_t* degrees2_host, int nterms2,
                                 int krylov_steps);
hp_status hp_magnus_step(hp_set_t s, int scheme, const int32_t* degrees1_host,
                         const double* coeffs1_host, int nterms1, const int32_t* degrees2_host,
                         const double* coeffs2_host, int nterms2, double halfwidth,
                         double harmonic_q, double h, int krylov_steps, int reorthogonalize,
                         void* y_dev, double* diag_dev, void* workspace_dev,
                         size_t workspace_bytes, void* stream);

/* lanczos(matvec, v0, steps) with the polynomial Hamiltonian as matvec --
 * krylov_propagator.py:58-104.  Outputs: basis_dev (steps x n complex128,
 * row k = v_k), alpha_dev (steps), beta_dev (steps-1), diag_dev as above. */
hp_status hp_lanczos(hp_set_t s, const int32_t* degrees_host, const double* coeffs_host,
                     int nterms, double halfwidth, double harmonic_q, const void* v0_dev,
                     int steps, int reorthogonalize, void* basis_dev, double* alpha_dev,
                     double* beta_dev, double* diag_dev, void* workspace_dev,
                     size_t workspace_bytes, void* stream);

/* tridiag_eigh + expm_tridiag_column -- krylov_propagator.py:107-177, on the
 * device (one thread; m <= 64).  col_dev: m complex128. */
hp_status hp_expm_tridiag_column(const double* alpha_dev, const double* beta_dev, int m,
                                 double tau, void* col_dev, int* status_dev, void* stream);

/* tridiag_eigh -- krylov_propagator.py:107-170 on the device (one thread;
 * m <= 48): eigenvalues ascending (stable order) into d_dev (m), eigenvectors
 * as columns of the row-major m x m z_dev; *status_dev = 1 if QL failed to
 * converge within 30 iterations (the reference raises RuntimeError). */
hp_status hp_tridiag_eigh(const double* alpha_dev, const double* beta_dev, int m, double* d_dev,
                          double* z_dev, int* status_dev, void* stream);

/* ---- BLAS-1 building blocks with deterministic reductions --------------- */
size_t hp_reduce_workspace_bytes(int64_t n);
/* out_dev[0..1] = sum conj(a) * b  (complex128), fixed summation order */
hp_status hp_cdot(int64_t n, const void* a_dev, const void* b_dev, double* out_dev,
                  void* workspace_dev, void* stream);
/* out_dev[0] = ||a||_2 (complex128 vector), fixed summation order */
hp_status hp_cnrm2(int64_t n, const void* a_dev, double* out_dev, void* workspace_dev,
                   void* stream);
/* Slab-sharded Lanczos (krylov_propagator.py:86-89): out = a x + b y + c z
   (real a, b, c; z may be NULL) and norm2_dev[0] = ||out||^2 of this rank's part (fixed order;
   the caller sums ranks).  workspace: hp_reduce_workspace_bytes(n). */
hp_status hp_lincomb3_nrm2sq(int64_t n, double a, const void* x_dev, double b, const void* y_dev, double c,
                             const void* z_dev, void* out_dev, double* norm2_dev, void* workspace_dev,
                             void* stream);
/* out = sum_k coef[k] V_k, complex coefficients coef_host[2k], coef_host[2k+1] (m <= 32):
   the basis combine of lanczos_exp_apply (krylov_propagator.py:180-186) */
hp_status hp_lincomb(int64_t n, int m, const void* const* vecs_host, const double* coef_host, void* out_dev,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HPROP_B200_H */
