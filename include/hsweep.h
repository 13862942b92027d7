/*
 * libhsweep -- C ABI of the B200-native TGSP-GMRES hot path.
 *
 * Drop-in boundary for the reference package `helmsweep` (arXiv 1412.0464,
 * /root/reference/pkg/src/helmsweep).  Every entry point replaces one
 * reference interface on the GMRES -> two-grid -> sweep path; the citation is
 * on each declaration.  Plain C types only: opaque handles, device pointers
 * (`void*` to complex128 interleaved re/im, numpy's memory layout), host
 * scalars and host index arrays.  All work is stream-ordered on the context
 * stream (hs_ctx_set_stream); nothing here synchronises unless it says so.
 *
 * Status codes map onto the reference's exception classes:
 *   HS_E_SHAPE / HS_E_ARG -> ValueError     HS_E_ZERO_PIVOT -> ZeroDivisionError
 *   HS_E_ZERO_DIAG -> ZeroDivisionError     HS_E_NONFINITE  -> FloatingPointError
 *   HS_E_BUFFER -> RuntimeError             HS_E_CUDA       -> RuntimeError
 * hs_last_error() returns the message, hs_last_error_index() the row / node.
 */
#ifndef HSWEEP_H
#define HSWEEP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HS_OK = 0,
  HS_E_SHAPE = 1,
  HS_E_ZERO_PIVOT = 2,
  HS_E_ZERO_DIAG = 3,
  HS_E_NONFINITE = 4,
  HS_E_CUDA = 5,
  HS_E_ARG = 6,
  HS_E_BUFFER = 7
};

enum { HS_VARIANT_UD = 0, HS_VARIANT_X = 1 };   /* NX plans get ids >= 2 (hs_sweep_plan_nx) */

typedef struct hs_ctx hs_ctx;
typedef struct hs_stencil hs_stencil;
typedef struct hs_transfer hs_transfer;
typedef struct hs_sweep hs_sweep;
typedef struct hs_cycle hs_cycle;
typedef struct hs_csr hs_csr;

/* ---- context ------------------------------------------------------------ */
int hs_ctx_create(int device, hs_ctx** out);
int hs_ctx_destroy(hs_ctx* ctx);
int hs_ctx_set_stream(hs_ctx* ctx, void* cuda_stream);
/* Face segments per sweep front of the 2-D sweeps this context creates next
 * (two-level partition: one cluster -- 9 CTAs by default -- per segment;
 * 0 = automatic, the widest layout whose clusters co-reside -- the fastest
 * single sweep; 1 = one cluster per front, which leaves room for any number
 * of concurrent sweep lanes; G > 1 allows hs_sweep_max_fronts / 2 lanes). */
int hs_ctx_set_sweep_segments(hs_ctx* ctx, int segments);
/* CTAs (face chunks) per segment's cluster of the 2-D sweeps this context
 * creates next (0 = automatic: 9).  Smaller clusters with more segments pack
 * several concurrent sweeps better: two lockstep batches at C4 run fastest
 * with 5 segments of 6 CTAs per front (DESIGN 5.2). */
int hs_ctx_set_sweep_cluster(hs_ctx* ctx, int ctas);
const char* hs_last_error(hs_ctx* ctx);
long long hs_last_error_index(hs_ctx* ctx);
long long hs_launch_count(hs_ctx* ctx);           /* kernels launched so far */
int hs_synchronize(hs_ctx* ctx);
int hs_version(void);

/* ---- built-in profiler (tracing) -------------------------------
 * When enabled, every launch is bracketed by CUDA events on the context
 * stream and attributed to a kernel class:
 *   0 stencil  1 residual  2 jacobi  3 jacobi2z (2 steps from zero)
 *   4 restrict 5 prolong   6 sweep_gather 7 sweep_front
 *   8 krylov_dot 9 krylov_update 10 krylov_other 11 setup
 *   12 pre_fused 13 post_fused (the fused V-cycle halves of 2-D levels)
 * hs_profile_read synchronises, folds pending events in and copies per-class
 * milliseconds, algorithmic HBM bytes and launch counts (arrays of nclass). */
int hs_profile_enable(hs_ctx* ctx, int on);
int hs_profile_reset(hs_ctx* ctx);
int hs_profile_read(hs_ctx* ctx, int nclass, double* ms, double* bytes, long long* counts);

/* ---- compact-stencil operators ------------------------------------------
 * StencilOperator(shape, coeffs)            reference discretize.py:57-107
 * `offsets`: S x dim int8, row-major; `coeffs`: host pointer to S contiguous
 * arrays of prod(shape) complex128 in the same order.  Uploaded once. */
int hs_stencil_create(hs_ctx* ctx, int dim, const int64_t* shape, int S,
                      const int8_t* offsets, const double* coeffs, hs_stencil** out);
int hs_stencil_destroy(hs_ctx* ctx, hs_stencil* op);
/* copy the S x prod(shape) coefficients back to host memory (synchronises) */
int hs_stencil_download(hs_ctx* ctx, const hs_stencil* op, double* coeffs);

/* ---- operator assembly on the device -----------------
 * The per-axis 1-D arrays come from the host (numpy, the reference's own
 * expressions); every per-node product runs on the device in numpy's
 * operation order and lands in the [S][n] layout, 1/diagonal included.
 * Complex arrays are interleaved (re, im) doubles, per-axis arrays
 * concatenated over the axes.
 *
 * Fine FD operator, _fd_operator / assemble_fine / assemble_sponge
 * (discretize.py:191-253): a_half[a] (N_a = shape[a]+1 complex, alpha at cell
 * midpoints), a_node[a] (N_a - 1 complex, alpha at the unknowns),
 * gamma_nodes[a] (N_a - 1 real sponge damping, or NULL for (k + 0i)^2),
 * k_dev: device float64 wavenumbers at the unknowns.  2*dim+1 offsets. */
int hs_assemble_fd(hs_ctx* ctx, int dim, const int64_t* shape, double h, const double* a_half,
                   const double* a_node, const double* gamma_nodes, const void* k_dev,
                   hs_stencil** out);
/* FE operator with the optimized-table weights, _fe_operator with per-cell
 * wavenumbers (discretize.py:413-506; coarse level :514-537, slabs :685-723):
 * per axis (N_a = shape[a]+1 cells) woa = widths/alpha, aow = alpha/widths,
 * cw = widths*(1/alpha) (complex), gamma_cells (real, or NULL).  k_nodes_dev /
 * k_cells_dev: the GLOBAL level's float64 fields, rows of kn_ld / kc_ld
 * elements; rowmap = {nrow0, nlo, nhi, crow0, clo, chi}: local sweep-axis row
 * r reads global node row clamp(nrow0 + r, nlo, nhi) and cell row
 * clamp(crow0 + r, clo, chi) (a slab's replicated edge rows).  Table:
 * ntab abscissae (1/G) and ntab x ncoef weights; h_ref the table's spacing.
 * 3^dim offsets in itertools.product order. */
int hs_assemble_fe(hs_ctx* ctx, int dim, const int64_t* shape, const double* woa,
                   const double* aow, const double* cw, const double* gamma_cells,
                   const void* k_nodes_dev, int64_t kn_ld, const void* k_cells_dev,
                   int64_t kc_ld, const int32_t* rowmap, double h_ref, int ntab, int ncoef,
                   const double* tab_x, const double* tab_c, hs_stencil** out);
/* y = A x            stencil_apply / fine_csr @ v   discretize.py:110-117, twogrid.py:140-141 */
int hs_stencil_apply(hs_ctx* ctx, const hs_stencil* op, const void* x, void* y, int nrhs);
/* r = f - A u        the residual lines twogrid.py:153, sweepdd.py:343 */
int hs_stencil_residual(hs_ctx* ctx, const hs_stencil* op, const void* f, const void* u,
                        void* r, int nrhs);
/* u <- u + omega (f - A u)/diag, `steps` times (in place);
 * u_is_zero != 0 means u enters as zero (the pre-smoother's start)
 * jacobi_smooth / TwoGridCycle._smooth       twogrid.py:41-50, 143-148 */
int hs_jacobi(hs_ctx* ctx, const hs_stencil* op, void* u, const void* f, double omega,
              int steps, int u_is_zero, int nrhs);

/* ---- tent transfers -----------------------------------------------------
 * CoarseningMap -> prolongation_matrix       mesh.py:107-123, twogrid.py:53-79
 * fp_concat: per-axis fine_point_of_coarse arrays concatenated (lengths in
 * fp_len[dim]); refined_concat: per-axis refined_cell (length fp_len[a]-1). */
int hs_transfer_create(hs_ctx* ctx, int dim, const int64_t* fp_len, const int64_t* fp_concat,
                       const uint8_t* refined_concat, hs_transfer** out);
/* The same maps for one shard of an x-slab (sweep-axis) decomposition
 * (SURVEY 8(e)): window = {fw_lo, fw_hi, cr_lo, cr_hi, fr_lo, fr_hi}, global
 * 0-based indices on the sweep axis.  The fine buffers hold rows [fw_lo,
 * fw_hi) (owned rows plus halo planes); hs_restrict computes coarse rows
 * [cr_lo, cr_hi) into a full-size coarse vector (other rows untouched);
 * hs_prolong_add computes fine rows [fr_lo, fr_hi) from a full-size coarse
 * vector.  HS_E_SHAPE if a computed coarse row reads outside the window. */
int hs_transfer_create_window(hs_ctx* ctx, int dim, const int64_t* fp_len,
                              const int64_t* fp_concat, const uint8_t* refined_concat,
                              const int64_t* window, hs_transfer** out);
int hs_transfer_destroy(hs_ctx* ctx, hs_transfer* t);

/* General sparse matrix (host CSR: indptr [rows+1], indices [nnz], interleaved
 * complex128 values [nnz]) uploaded for y = alpha A x (+ y): the explicit
 * prolongation matrix of a TwoGridCycle built from one (twogrid.py:119-159,
 * `p_matrix @ uc`, `p_matrix.T @ r`); the BASELINE hierarchies use the tent
 * tables (hs_transfer_create) instead. */
int hs_csr_create(hs_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* indptr,
                  const int64_t* indices, const double* vals, hs_csr** out);
int hs_csr_destroy(hs_ctx* ctx, hs_csr* m);
int hs_csr_apply(hs_ctx* ctx, const hs_csr* m, const void* x, void* y, double alpha_re,
                 double alpha_im, int accumulate);
/* rc = scale * P^T r                         twogrid.py:154 (restrict: 89-93 with scale 1) */
int hs_restrict(hs_ctx* ctx, const hs_transfer* t, const void* r_fine, void* rc, double scale,
                int nrhs);
/* rc = scale * P^T (f - A u)                 twogrid.py:153-154 fused */
int hs_restrict_residual(hs_ctx* ctx, const hs_transfer* t, const hs_stencil* op,
                         const void* u, const void* f, void* rc, double scale, int nrhs);
/* u += P uc  (beta = 0: u = P uc)            twogrid.py:156 (prolongate: 82-86) */
int hs_prolong_add(hs_ctx* ctx, const hs_transfer* t, const void* uc, void* u, int accumulate,
                   int nrhs);

/* ---- sweeping preconditioner --------------------------------------------
 * build_partition + per-slab factorize       sweepdd.py:192-218, sparselin.py:40-68
 * coarse: the global level operator (transmission blocks and the mid-sweep
 * residual read it, sweepdd.py:133-141, 175-176).  slab_ops[j]: the slab
 * operators (sweepdd.py:211 / discretize.py:685-723), slab j spanning grid
 * points slab_lo[j]..slab_hi[j] (1-based).  Factorises every slab on the
 * device (batched block-tridiagonal LU); fails with HS_E_ZERO_PIVOT. */
int hs_sweep_create(hs_ctx* ctx, const hs_stencil* coarse, int J, const int64_t* beta,
                    const int64_t* beta_tilde, const int64_t* slab_lo, const int64_t* slab_hi,
                    const hs_stencil* const* slab_ops, hs_sweep** out);
int hs_sweep_destroy(hs_ctx* ctx, hs_sweep* s);
/* u = Sweep(f); variant HS_VARIANT_X (prec_x, sweepdd.py:322-359) or
 * HS_VARIANT_UD (prec_ud, sweepdd.py:312-319).  f and u: device, coarse shape. */
int hs_sweep_apply(hs_ctx* ctx, hs_sweep* s, int variant, const void* f, void* u);
/* nrhs right-hand sides at once (the reference's multi-column
 * Factorization.solve, sparselin.py:58-62; SURVEY 8(b)'s nrhs):
 * right-hand side r at f + r * stride, its result at u + r * stride (stride
 * in complex elements, >= the coarse size).  Groups of up to
 * hs_sweep_rhs_width(s) right-hand sides (4, 2 or 1 by the face length) run
 * through ONE chain of slab solves, every factor block streamed once per
 * group; per right-hand side the result is bitwise hs_sweep_apply's.  3-D
 * levels and the exact solvers (hs_exact_create*) carry the group through
 * their block chains the same way (multi-column Factorization.solve).  The
 * batch's work set (traces, mid-sweep residual, second-pass buffer) belongs
 * to the sweep and is allocated on first use: one caller at a time per
 * hs_sweep; concurrent callers go through lanes (hs_cycle_create_lane), whose
 * work sets are private. */
int hs_sweep_apply_many(hs_ctx* ctx, hs_sweep* s, int variant, int nrhs, const void* f, void* u,
                        long long stride);
int hs_sweep_rhs_width(hs_sweep* s);
/* Sweep fronts whose clusters can be co-resident on the device (2-D levels):
 * concurrent lanes (hs_cycle_create_lane) need 2 fronts each. */
int hs_sweep_max_fronts(hs_sweep* s);
/* NX sweep (prec_nx, sweepdd.py:403-437; NxCells / make_nx_cells :362-401):
 * registers the launch plan of one cell grouping -- j_cell: ncell + 1 cell
 * boundaries with sentinels -1 and J + 1, j_mid: the slab where each cell's
 * sweeps meet -- and returns its variant id (>= 2) for hs_sweep_apply and
 * hs_cycle_create.  The groups' fronts run concurrently (one cluster each).
 * Fails with HS_E_SHAPE on an invalid grouping (NxCells.validate). */
int hs_sweep_plan_nx(hs_ctx* ctx, hs_sweep* s, int ncell, const int64_t* j_cell,
                     const int64_t* j_mid, int* variant);
/* One slab solve outside a schedule: subdom_solve (sweepdd.py:236-268).
 * Slab j (1-based) with right-hand side rows [a, b) of f (global rows,
 * 0-based) plus the transmission of the input traces B1 (forward, used when
 * j > 1) and B3 (backward, j < J) -- each 2 x face, device, or NULL; the
 * solution rows [ta, tb) are ADDED into u (u[ta:tb] += ud); out2 (j < J) /
 * out4 (j > 1), when non-NULL, receive the outgoing 2 x face traces.  On a
 * 2-D level the requested rows must be rows the sweep's schedules read
 * (HS_E_SHAPE otherwise: the device slab solve updates those rows only). */
int hs_sweep_solve_one(hs_ctx* ctx, hs_sweep* s, int j, int64_t a, int64_t b, int64_t ta,
                       int64_t tb, const void* B1, const void* B3, void* out2, void* out4,
                       const void* f, void* u);
/* Exact solve of a whole stencil operator: factorize / Factorization.solve
 * (sparselin.py:40-68) and ExactCoarseSolver (twogrid.py:99-105).  Block LU
 * along the operator's second axis with dense planes of the first (x third)
 * axis -- NB = n0 (2-D) or n0*n2 (3-D) unknowns per block, at most
 * 8 * (SM count); factors: (3 n1 - 2) NB^2 complex128 in HBM.  The handle is
 * an hs_sweep: apply it with hs_sweep_apply(HS_VARIANT_UD), or pass it to
 * hs_cycle_create with HS_VARIANT_UD for a two-grid cycle with an exact
 * coarse solve.  Fails with HS_E_ZERO_PIVOT on a singular pivot block. */
int hs_exact_create(hs_ctx* ctx, const hs_stencil* op, hs_sweep** out);
/* Exact solver of a general sparse n x n matrix given as host CSR (indptr
 * [n+1], indices [nnz], interleaved complex128 values [nnz]) -- replaces
 * Factorization(matrix) / factorize(scipy matrix), sparselin.py:40-68.
 * block >= the matrix bandwidth max|i - j|: the matrix is factorised as
 * block tridiagonal over ceil(n / block) block rows (padded with identity
 * rows); vectors passed to hs_sweep_apply(HS_VARIANT_UD) hold
 * ceil(n / block) * block entries (padding in = 0).  HS_E_ZERO_PIVOT on a
 * singular pivot block, HS_E_SHAPE when the bandwidth exceeds block. */
int hs_exact_create_csr(hs_ctx* ctx, int64_t n, int64_t nnz, const int64_t* indptr,
                        const int64_t* indices, const double* vals, int block, hs_sweep** out);
/* The X plan cut where each front passes from one sweep-axis shard's slabs
 * to the next (slab j on shard (j-1)*shards/J), one launch per shard step:
 * the critical path of a relay in which every GPU owns its region's slabs
 * and the traces hop between GPUs (here through the trace buffers on one
 * device).  Results equal HS_VARIANT_X; *variant is the id to pass to
 * hs_sweep_apply.  (the measured relay vs replication.) */
int hs_sweep_plan_relay(hs_ctx* ctx, hs_sweep* s, int shards, int* variant);
/* bytes of device memory held by the slab factors (diagnostic) */
long long hs_sweep_factor_bytes(hs_sweep* s);
/* slab-solve launches in one application of a variant's plan (diagnostic:
 * the profiler's sweep_front launches per prec_x / prec_ud / prec_nx) */
int hs_sweep_plan_launches(hs_sweep* s, int variant);
/* 2-D slab-solve layout (diagnostic): face segments per front (clusters of
 * the two-level partition, 1 = one cluster) and chunks (CTAs) per segment */
int hs_sweep_segments(hs_sweep* s);
int hs_sweep_chunks(hs_sweep* s);

/* ---- two-grid cycle ------------------------------------------------------
 * TwoGridCycle(fine, P, smoother, SweepCoarseSolver)   twogrid.py:119-164, 196-229 */
int hs_cycle_create(hs_ctx* ctx, const hs_stencil* fine, const hs_transfer* t,
                    const hs_stencil* coarse, hs_sweep* sweep, double omega_jac, int nu,
                    double restrict_scale, int variant, hs_cycle** out);
/* A lane of `base`: the same operators, transfer maps and factorised sweep,
 * with private cycle and sweep scratch, so applications of the two cycles on
 * two contexts / streams run concurrently (several right-hand sides in
 * flight on one GPU; each 2-D sweep front occupies one 16-SM cluster).
 * 2-D levels only (the 3-D slab solve is a cooperative all-SM kernel). */
int hs_cycle_create_lane(hs_ctx* ctx, const hs_cycle* base, hs_cycle** out);
int hs_cycle_destroy(hs_ctx* ctx, hs_cycle* c);
/* u = M f : vcycle / tgsp_apply / as_preconditioner   twogrid.py:150-176 */
int hs_vcycle(hs_ctx* ctx, hs_cycle* c, const void* f, void* u);
/* nrhs cycles u_r = M f_r (twogrid.py:150-176 per column): fine-level halves
 * per right-hand side, the coarse sweeps through hs_sweep_apply_many (a lane,
 * hs_cycle_create_lane, uses its own work set). */
int hs_vcycle_many(hs_ctx* ctx, hs_cycle* c, int nrhs, const void* f, void* u, long long stride);
/* GMRES operator application keeping the preconditioned vector: z = M f,
 * w = A z, in parts like hs_vcycle_apply_a_part (0 pre-coarse into z, 1 the
 * sweep's first launch, 2 the rest and w = A z) or whole (part 3).  With the
 * z of every Arnoldi step kept, the end of a GMRES cycle updates u += Z y
 * instead of applying M once more to V y (M is linear and fixed: the same
 * update, one V-cycle fewer per restart cycle; krylov.py:96-101). */
int hs_vcycle_apply_az_part(hs_ctx* ctx, hs_cycle* c, const void* f, void* z, void* w, int part);
/* w = A M f (the GMRES operator, krylov.py:125-126) */
int hs_vcycle_apply_a(hs_ctx* ctx, hs_cycle* c, const void* f, void* w);
/* The same operator in two halves, so a host pipelining the Arnoldi loop can
 * queue the pre-coarse part of the next iteration before it reads the
 * current Hessenberg column: begin = pre-smoothing, residual, restriction
 * (twogrid.py:152-154); end = sweep, prolongation, post-smoothing and the
 * fine matvec (twogrid.py:155-159, krylov.py:126).  One begin/end pair per
 * cycle handle may be in flight. */
int hs_vcycle_apply_a_begin(hs_ctx* ctx, hs_cycle* c, const void* f);
int hs_vcycle_apply_a_end(hs_ctx* ctx, hs_cycle* c, const void* f, void* w);
/* Finer split for a deeper host pipeline: part 0 = begin; part 1 = the
 * sweep's first launch (X: both pass-1 fronts, prec_x sweepdd.py:331-341);
 * part 2 = the rest of end (w written here).  0, 1, 2 in order == begin+end. */
int hs_vcycle_apply_a_part(hs_ctx* ctx, hs_cycle* c, const void* f, void* w, int part);

/* ---- GMRES vector kernels (krylov.py:46-102) ------------------------------
 * V: device basis, k vectors of length n with leading dimension ldv (elements).
 * Results to device pointers; deterministic two-stage reductions. */
/* h[i] = vdot(V_i, w) (i < k); h[k] = (||w||^2, 0) */
int hs_block_dot(hs_ctx* ctx, const void* V, int64_t ldv, int k, const void* w, int64_t n,
                 void* h);
/* w -= sum_i h[i] V_i (i < k); nrm2[0] = (||w||^2, 0) */
int hs_block_update(hs_ctx* ctx, const void* V, int64_t ldv, int k, const void* h, void* w,
                    int64_t n, void* nrm2);
/* CGS2 step fused (the first pass's update with the second pass's dots,
 * one read of V): w -= sum_i h[i] V_i; h2[i] = vdot(V_i, w) (i < k),
 * h2[k] = nrm2[0] = (||w||^2, 0).  Bitwise equal to hs_block_update followed
 * by hs_block_dot.  1 <= k <= 32. */
int hs_block_update_dot(hs_ctx* ctx, const void* V, int64_t ldv, int k, const void* h, void* w,
                        int64_t n, void* nrm2, void* h2);
/* Second (DGKS) Gram-Schmidt pass gated on the device, krylov.py:67-70 with
 * re-orthogonalisation: runs only when g_after[0].re < thresh * g_before[0].re
 * (||w||^2 after / before the first pass); a closed gate leaves h untouched
 * and copies g_after[0] into nrm2[0]. */
int hs_block_dot_gated(hs_ctx* ctx, const void* V, int64_t ldv, int k, const void* w,
                       int64_t n, void* h, const void* g_after, const void* g_before,
                       double thresh);
int hs_block_update_gated(hs_ctx* ctx, const void* V, int64_t ldv, int k, const void* h,
                          void* w, int64_t n, void* nrm2, const void* g_after,
                          const void* g_before, double thresh);
/* x *= 1 / sqrt(max(s[0].re, 0)): the Arnoldi normalisation v_{k+1} = w / H[k+1,k]
 * (krylov.py:70-72) with the norm read on the device */
int hs_scale_inv_sqrt(hs_ctx* ctx, void* x, int64_t n, const void* s);
/* out = sum_i y[i] V_i  (y: device, k complex) */
int hs_lincomb(hs_ctx* ctx, const void* V, int64_t ldv, int k, const void* y, void* out,
               int64_t n);
/* x = alpha * x (alpha host complex) */
int hs_scale(hs_ctx* ctx, void* x, int64_t n, double alpha_re, double alpha_im);
/* y = a x + b y */
int hs_axpby(hs_ctx* ctx, double a_re, double a_im, const void* x, double b_re, double b_im,
             void* y, int64_t n);
/* out[0] = (||x||^2, nonfinite_count) */
int hs_norm2(hs_ctx* ctx, const void* x, int64_t n, void* out);

#ifdef __cplusplus
}
#endif

#endif /* HSWEEP_H */
