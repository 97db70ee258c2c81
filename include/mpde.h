/*
 * mpde.h -- C ABI of the B200-native NeuRLP-PDE batched solver
 * (Mechanistic PDE Networks, arXiv 2502.18377, §3).
 *
 * The library solves, for a batch of B independent linear space-time PDEs
 *      sum_m c_m(p) u_m(p) = b(p)           (Eq. 1)
 * the least-squares problem min_z ||A z - d||_2 whose rows are the equation
 * (Eq. 3), Dirichlet boundary (Eq. 4), derivative (Eq. 5,
 * P:169-174) and forward/backward Taylor smoothness (Eqs. 6-7)
 * constraints, via the normal equations A^T A z = A^T d (Eq. 9), and the
 * backward pass A^T A d_z = g_z (Eq. 11) with the gradient formulas of
 * P:240 restricted to the encoder outputs c, b, omega.
 *
 * Readings of the paper that fix the operator: the boundary
 * set B is every face of the space-time box; the variables are u_phi plus the first
 * and second pure derivative along every dim (|M| = 1 + 2*ndim, field order
 * phi, d0, d00, d1, d11, ...); derivative rows use 5-point central weights for
 * 2 <= i <= n-3 and one-sided 5-point weights at the two points nearest each edge,
 * with coefficient h^k on the derivative variable (literal Eq. 5); Taylor rows are
 * present in each direction where the neighbour exists.
 *
 * Layout: every per-point tensor is C-contiguous float32 with dim 0 (time) slowest:
 *   coeff  [B][|M|][n0][n1]...      c_m, field-major per PDE
 *   rhs_b  [B][n0][n1]...           b
 *   bnd    [B][n0][n1]...           omega (only entries on B are read)
 *   z, g_z, dz, grad_coeff  [B][|M|][P]
 *   grad_rhs, grad_bnd      [B][P]
 * All tensor pointers passed to mpde_build_hierarchy / mpde_solve_* /
 * mpde_apply_* are DEVICE pointers owned by the caller (PyTorch allocates); the
 * library performs no device allocation in those calls -- all scratch lives in the
 * caller's workspace (size from mpde_workspace_bytes).  Calls enqueue work on
 * `stream` and, unless stated otherwise, return without synchronising.  A handle
 * must not be used from two host threads at once.
 *
 * Errors: every int-returning call returns an MPDE_* code; synchronous failures
 * (bad arguments, unsupported configuration, workspace too small, CUDA launch
 * failure) return non-zero and set a thread-local message (mpde_last_error()).
 * Per-PDE numerical outcomes (not converged, non-finite input, indefinite
 * operator) are asynchronous and reported in mpde_stats.status.
 */
#ifndef MPDE_H_
#define MPDE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mpde_stream_t; /* == cudaStream_t; NULL = legacy default stream */

enum {
  MPDE_OK = 0,
  MPDE_ERR_INVALID_ARG = 1,   /* null pointer, batch < 1, non-finite step, ...        */
  MPDE_ERR_SHAPE = 2,         /* ndim not in {2,3,4}, a dim with fewer than 6 points  */
  MPDE_ERR_UNSUPPORTED = 3,   /* deriv_order != 2, unknown smoother/coarse option     */
  MPDE_ERR_NONFINITE = 4,     /* (status only) non-finite input or residual           */
  MPDE_ERR_NOT_CONVERGED = 5, /* (status only) tolerance not met within the limits    */
  MPDE_ERR_CUDA = 6,          /* a CUDA call failed; message has the CUDA error text  */
  MPDE_ERR_WORKSPACE = 7      /* workspace_bytes smaller than mpde_workspace_bytes()  */
};

/* per-PDE status values in mpde_stats.status */
enum { MPDE_STATUS_CONVERGED = 0, MPDE_STATUS_MAXITER = 1, MPDE_STATUS_NONFINITE = 2,
       MPDE_STATUS_INDEFINITE = 3 };

/* boundary types per face (mpde_problem.bc): "Dirichlet (i.e., boundary conditions
 * on u), Neumann (i.e., boundary conditions on partial derivatives) or mixed types" */
enum { MPDE_BC_DIRICHLET = 0, MPDE_BC_NEUMANN = 1, MPDE_BC_NONE = 2 };

/* Grid, batch and row-group weights.  P:89 (Cartesian grid), P:111-117 (uniform step
 * per dim -- learned per-interval steps are out of scope), P:147-151 (variables). */
typedef struct {
  int32_t ndim;        /* grid dims including time: 2, 3 or 4; dim 0 = time (slowest)   */
  int32_t n[4];        /* points per dim, each >= 6 (5-point one-sided edge stencils)   */
  double  h[4];        /* uniform step per dim, finite, > 0                             */
  int32_t batch;       /* B >= 1 independent PDEs                                        */
  int32_t deriv_order; /* must be 2: M = {phi, d_k, d_kk for every dim}                 */
  float   w_eq, w_bnd, w_deriv, w_smooth; /* row-group weights, > 0 (paper: all 1)      */
  int32_t bc[4][2];    /* boundary type of face (dim d, low = 0 / high = 1 side), MPDE_BC_*:
                          DIRICHLET: w_bnd u_phi(p) = w_bnd omega(p) on every point of the
                            face (one row per point on at least one Dirichlet face);
                          NEUMANN: w_bnd u_{d}(p) = w_bnd omega_n[d](p) (the first-derivative
                            variable along the face's axis; one row per face point);
                          NONE: no boundary row on that face.
                          All zero (the default of a zero-initialised struct) = every face
                          Dirichlet, the paper's Eq. 4 with B = all faces (reading Q1).  */
} mpde_problem;

/* Solver options.  The Krylov method is PCG on the (condensed) normal equations; the
 * preconditioner is one multigrid V-cycle (Alg. 1). */
typedef struct {
  float   tol;        /* stop when ||A^T(d - A z)|| / ||A^T d|| <= tol (fp64 residual)   */
  float   tol_inner;  /* PCG stop per refinement pass: ||r_k|| / ||r_0|| <= tol_inner    */
  int32_t max_iters;  /* PCG iteration cap per refinement pass                          */
  int32_t max_refine; /* fp64-residual refinement passes (>= 1)                          */
  int32_t smoother;   /* 0 = damped Jacobi, 1 = Chebyshev-accelerated Jacobi             */
  int32_t nu;         /* smoothing steps, pre = post (>= 1)                              */
  int32_t coarsest;   /* stop coarsening a dim once it is <= coarsest (8)         */
  int32_t levels_max; /* cap on the number of levels (1 = no multigrid: Jacobi-PCG)      */
  int32_t poll_every; /* host convergence poll interval in PCG iterations (>= 1)         */
  float   jacobi_theta;   /* damped Jacobi: omega = theta / lambda_max(D^-1 S)           */
  float   cheb_ratio;     /* Chebyshev interval [lambda_max/ratio, 1.1 lambda_max]       */
  int32_t lanczos_steps;  /* Lanczos steps (2..32) estimating lambda_max per level+PDE  */
  int32_t precision;  /* arithmetic (storage is fp32): 0 = fp32 everywhere; 1 = fp64 for
                         the condensation / back-substitution (default); 2 = also the
                         PCG operator; 3 = also the V-cycle.  The refinement residual and
                         all dot products are always fp64.                              */
  int32_t use_graphs; /* 1 = replay PCG iterations as a CUDA graph (cached per workspace,
                         problem and options); 0 = plain launches                        */
  float   tol_z;      /* error-based stop: after >= 2 refinement passes, stop when the
                         estimate ||d_k||^2/||d_k-1|| / ||z|| <= tol_z (d_k = correction of
                         pass k); `tol` above is a residual floor that also stops        */
  float   tol_inner2; /* PCG stop for refinement passes >= 2: ||r_k|| / ||r_0|| <= tol_inner2.
                         The first pass must reach tol_inner; later passes only correct it,
                         and the error estimate of pass k >= 2 is ||d_k|| * max(||d_k|| /
                         ||d_k-1||, tol_inner2) / ||z|| (Q14)                    */
  int32_t cf_bf16;    /* 1 = the V-cycle's level-0 S applies read the per-point coefficients
                         of S as bf16 (half the bytes); S~ stays symmetric PSD, so the
                         preconditioner is still a fixed SPD map.  The PCG operator, the
                         refinement residual and the gradients keep fp32 / fp64 (default 1) */
  int32_t krylov;     /* inner Krylov method on the condensed system: 0 = PCG (default; needs
                         the fixed SPD V-cycle), 1 = FGMRES(restart) with the same V-cycle as a
                         flexible right preconditioner -- the paper's method (SURVEY
                         §8(f) N1); its |g_{j+1}| is the true residual ||rt - S x||, so the same
                         tol_inner / max_iters apply; every refinement pass runs to
                         min(tol_inner, tol_inner2) (GMRES minimises the residual, not the
                         error: the PCG-calibrated tol_inner2 left e_z 1.5e-4 at C2)       */
  int32_t restart;    /* FGMRES restart length m, 1..32 (default 30; workspace grows by
                         (2m+1) scalar fields per PDE)                                      */
  int32_t grad_steps; /* 1 = the forward keeps the duals of the derivative and Taylor rows
                         (4*ndim fields per point of workspace) so that mpde_step_gradient
                         can return dl/dh after the backward; default 0        */
  float   tol_adapt;  /* PCG refinement passes >= 3: a PDE whose error estimate after the
                         previous pass is e only needs that error shrunk by tol_z / e, so the
                         pass runs to max(tol_inner2, min(tol_adapt, tol_z / (10 e))) instead
                         of tol_inner2; its error estimate uses that tolerance.  0 = off;
                         default 0.1 (C5 forward -14% iterations, C3 -12%, C2 -12%,
                         DESIGN.md Q14); ignored with krylov = 1                          */
} mpde_options;

/* one per PDE, device memory, written by mpde_solve_fwd / mpde_solve_bwd */
typedef struct {
  int32_t iters;    /* PCG iterations summed over refinement passes                       */
  int32_t refines;  /* refinement passes run                                              */
  int32_t status;   /* MPDE_STATUS_*                                                      */
  float   rel_res;  /* final ||A^T(d - A z)|| / ||A^T d|| (fp64 residual)                 */
  float   err_est;  /* estimated relative error of z (refinement contraction estimate)    */
} mpde_stats;

typedef struct mpde_hierarchy mpde_hierarchy; /* opaque, host-side handle */

/* Defaults: tol_z 1.5e-5 with tol_adapt 0.1 (6.7x below the north_star bar 1e-4; errors
 * against the converged oracle references and over-converged solves are far below it, and
 * the adaptive last pass makes the extra margin cheap: DESIGN.md Q14,
 * profiles/r2_stop_rule.txt), poll_every 4, tol 1e-10, tol_inner 3e-4, tol_inner2 3e-3,
 * max_refine 6, Chebyshev nu = 2, coarsest 8, 16 Lanczos steps, precision 1. */
mpde_options mpde_default_options(void);

/* n_v = |M| * P variables, n_c constraint rows (Eqs. 3-7 counted), levels of the
 * hierarchy for these options.  Any output pointer may be NULL. */
int mpde_sizes(const mpde_problem* prob, const mpde_options* opts, int64_t* n_v,
               int64_t* n_c, int32_t* n_levels);

/* Bytes of device workspace mpde_build_hierarchy needs (0 on invalid input). */
size_t mpde_workspace_bytes(const mpde_problem* prob, const mpde_options* opts);

/* Build the multigrid hierarchy for coefficient fields `coeff` [B][|M|][P] (device):
 * coarse coefficient fields by full-weighting averaging, the diagonal of each
 * level's condensed operator, per-PDE lambda_max estimates and the coarsest-level
 * inverse.  `coeff` and `workspace` must stay valid and unmodified until
 * mpde_destroy_hierarchy.  Asynchronous on `stream`.  *out receives a new handle. */
int mpde_build_hierarchy(const mpde_problem* prob, const mpde_options* opts,
                         const float* coeff, void* workspace, size_t workspace_bytes,
                         mpde_stream_t stream, mpde_hierarchy** out);

/* Forward pass: z* = argmin ||A z - d|| for every PDE of the batch.
 * rhs_b [B][P], bnd [B][P] (device, read);  z [B][|M|][P] (device, written);
 * stats: device array of B mpde_stats or NULL.  Synchronises `stream` only to poll
 * convergence every poll_every iterations. */
int mpde_solve_fwd(mpde_hierarchy* h, const float* rhs_b, const float* bnd, float* z,
                   mpde_stats* stats, mpde_stream_t stream);

/* Forward / backward with Neumann data (faces of type MPDE_BC_NEUMANN):
 * bnd_n [B][ndim][P] (device, read only on the Neumann faces of dim d; NULL = homogeneous
 * Neumann data, omega_n = 0); grad_bnd_n [B][ndim][P] (device, written: dl/domega_n on the
 * Neumann faces of dim d, 0 elsewhere; NULL = not computed).  mpde_solve_fwd / _bwd are these
 * calls with NULL Neumann arguments.
 * lambda_opt (device, written, or NULL): the duals lambda* = d - A z* (Eq. 10 first block row,
 * P:200-214), computed in fp64 from the forward's fp64 solution, in a structured
 * layout [B][2 + 5*ndim][P]: slot 0 the equation row of p (Eq. 3), 1 its Dirichlet row (0 if p
 * has none), 2 + d the Neumann row of dim d (0 off the Neumann faces of d), 2 + ndim + 2d + (k-1)
 * the derivative row (d, k) (Eq. 5), 2 + 3 ndim + 2d + {0 forward, 1 backward} the Taylor rows
 * (Eqs. 6-7; 0 where the neighbour does not exist).  Each slot holds the row's weighted
 * residual, e.g. w_eq (b - sum_m c_m z_m) for slot 0. */
int mpde_solve_fwd_bc(mpde_hierarchy* h, const float* rhs_b, const float* bnd, const float* bnd_n,
                      float* z, float* lambda_opt, mpde_stats* stats, mpde_stream_t stream);
int mpde_solve_bwd_bc(mpde_hierarchy* h, const float* rhs_b, const float* z, const float* g_z,
                      float* grad_coeff, float* grad_rhs, float* grad_bnd, float* grad_bnd_n,
                      float* dz_opt, mpde_stats* stats, mpde_stream_t stream);

/* Backward pass (Eq. 11) for the loss gradient g_z = dl/dz* [B][|M|][P]:
 * solves A^T A d_z = g_z with the same hierarchy and writes
 *   grad_coeff[b][m][p] = dl/dc_m(p),  grad_rhs[b][p] = dl/db(p),
 *   grad_bnd[b][p] = dl/domega(p) (0 off the Dirichlet faces),  dz_opt = d_z (or NULL).
 * z must be the forward solution for the same rhs_b.  If the last mpde_solve_fwd on this
 * handle was called with the same rhs_b pointer, the equation residual b - c.z* it kept
 * (formed from its fp64 solution) is used for grad_coeff; otherwise it is formed from the
 * fp32 z, which loses accuracy where the derivative fields are large. */
int mpde_solve_bwd(mpde_hierarchy* h, const float* rhs_b, const float* z, const float* g_z,
                   float* grad_coeff, float* grad_rhs, float* grad_bnd, float* dz_opt,
                   mpde_stats* stats, mpde_stream_t stream);

/* dl/dh_d, the gradient of the loss with respect to the uniform step of every dim (P:114-126:
 * "step sizes ... are differentiable"), for the loss whose dl/dz* was the g_z of the last
 * mpde_solve_bwd on this handle: the P:240 matrix gradient d_lambda z*^T + lambda* d_z^T
 * contracted with dA/dh_d over the derivative rows (coefficient w_der h^k) and Taylor rows
 * (+-w_sm h, w_sm h^2/2) of dim d.  Needs options.grad_steps = 1 at build (the forward keeps
 * lambda* of those rows) and the forward and backward of the same (rhs_b, z) on this handle.
 * z: the forward's output [B][|M|][P] (device); grad_h: [B][ndim] fp32 (device, written).
 * Deterministic (fixed-order fp64 reduction).  MPDE_ERR_INVALID_ARG without grad_steps or a
 * preceding forward + backward. */
int mpde_step_gradient(mpde_hierarchy* h, const float* z, float* grad_h, mpde_stream_t stream);

/* Release the handle (does not free caller memory). */
int mpde_destroy_hierarchy(mpde_hierarchy* h);

/* Thread-local text of the last synchronous error ("" if none). */
const char* mpde_last_error(void);

/* ---- operator-level entry points (used by the parity tests) ------------------- */

/* q = A^T A z for the fine level of `prob` (Eq. 9), fp64 accumulation, device
 * pointers coeff [B][|M|][P], z [B][|M|][P], q [B][|M|][P]. */
int mpde_apply_normal(const mpde_problem* prob, const float* coeff, const float* z, float* q,
                      mpde_stream_t stream);

/* y = S_l x on level `level` of a built hierarchy, where S_l is the Schur complement of
 * the level's normal matrix onto the u_phi variables.
 * x, y: device [B][P_l]. */
int mpde_apply_schur(mpde_hierarchy* h, int32_t level, const float* x, float* y,
                     mpde_stream_t stream);

/* z = M^-1 r: one V-cycle of the preconditioner (Alg. 1) on the fine level,
 * r, z: device [B][P].  The preconditioner is a fixed symmetric linear map. */
int mpde_apply_precond(mpde_hierarchy* h, const float* r, float* z, mpde_stream_t stream);

/* Copy internal per-level data to the caller (device pointer `dst`):
 *   what = 0: level shape (n0, n1, n2, levels) -> dst is HOST int32[4] (synchronous; 2D/3D)
 *   what = 1: 1/diag(S_l) [B][P_l] fp32        what = 2: lambda_max [B] fp32
 *   what = 3: coarse coefficients [B][|M|][P_l] fp32
 *   what = 4: coarsest-level inverse [B][P_c][P_c] fp32 (level ignored)
 *   what = 5: kernel variants applying S on the level -> dst is HOST int32[4] (synchronous):
 *             [pass 1 of the PCG operator, pass 2 of the PCG operator, pass 2 of the V-cycle
 *             applies, 1 if those read bf16 coefficients]; codes 0 scalar, 1 v4, 2 v4
 *             warp-specialised, 3 t-blocked, 4 t-blocked with compile-time extents,
 *             5 2x2-blocked, 6 smem tile, 7 fused, 8 pass 1 with the y part
 *   what = 6: level shape of any ndim (n0, n1, n2, n3, levels), 0 for dims >= ndim -> dst is
 *             HOST int32[5] (synchronous) */
int mpde_hierarchy_query(mpde_hierarchy* h, int32_t level, int32_t what, void* dst,
                         mpde_stream_t stream);

/* Host-buffer end-to-end call: copies the inputs from HOST memory (pinned for
 * asynchrony) into `device_staging` (>= mpde_host_staging_bytes), builds the
 * hierarchy in `workspace`, runs forward + backward with g_z, and copies z, grad_coeff,
 * grad_rhs, grad_bnd back to HOST memory.  Synchronises `stream` before returning.
 * The H2D of g_z overlaps the build and the forward, and the D2H of z the backward, on a
 * per-thread side stream of the library that is joined back into `stream` (events recorded
 * on `stream` around the call cover every copy). */
size_t mpde_host_staging_bytes(const mpde_problem* prob);
int mpde_fwd_bwd_host(const mpde_problem* prob, const mpde_options* opts,
                      const float* coeff_h, const float* rhs_h, const float* bnd_h,
                      const float* gz_h, float* z_h, float* grad_coeff_h, float* grad_rhs_h,
                      float* grad_bnd_h, void* device_staging, void* workspace,
                      size_t workspace_bytes, mpde_stream_t stream);

/* out[j] = sum_b x[b][j] for x [batch][n] (device, fixed summation order): the
 * batch-summed coefficient gradient that the multi-GPU step all-reduces (NCCL). */
int mpde_batch_sum(const float* x, int32_t batch, int64_t n, float* out, mpde_stream_t stream);

/* ---- polynomial PDE-expression template ----------------------
 * The paper builds the coefficients and the right-hand side from learned polynomials of
 * transformed data fields u~ ("p_1(u~) = theta_0 + theta_1 u~ + theta_2 u~^2";
 * P:520-521 third-degree polynomials of u~, v~ for the u, u_xx, u_yy coefficients and b;
 * P:552 degree 1 for Navier-Stokes).  With F feature fields and total degree G:
 *   c_m(p) = sum_k theta[m][k] Phi_k(u~(p))  (m < |M|),   b(p) = sum_k theta[|M|][k] Phi_k(u~(p))
 * Phi_k = prod_f u~_f^e_f over all exponent tuples with e_0 + ... + e_{F-1} <= G, ordered by
 * total degree, then by tuple in descending lexicographic order (F = 1: 1, u, u^2, ...;
 * F = 2, G = 2: 1, u0, u1, u0^2, u0 u1, u1^2).  A coefficient the paper fixes (c_t = 1) is
 * the constant monomial of its row.  theta is shared by the whole batch.
 * Layouts (device, fp32, C-contiguous): theta [|M|+1][K]; feat [B][F][P]; coeff, grad_coeff
 * [B][|M|][P]; rhs_b, grad_rhs [B][P]; grad_theta [|M|+1][K]; grad_feat [B][F][P].
 * The boundary values omega are not templated (the paper takes them from u~, P:338, P:522:
 * pass the matching feature slice as `bnd` and add grad_bnd to its gradient).
 * Errors: MPDE_ERR_UNSUPPORTED if F not in 1..3 or G not in 0..4; MPDE_ERR_INVALID_ARG for
 * null pointers (grad_feat may be NULL); MPDE_ERR_WORKSPACE if workspace_bytes is short. */
typedef struct {
  int32_t n_feat; /* F: feature fields per PDE, 1..3 */
  int32_t degree; /* G: total polynomial degree, 0..4 */
} mpde_template;

/* K = C(F+G, G) monomials, or -1 for an unsupported template */
int32_t mpde_template_terms(const mpde_template* t);

/* coeff and rhs_b of every PDE from theta and feat (one pointwise kernel). */
int mpde_template_coeff(const mpde_problem* prob, const mpde_template* t, const float* theta,
                        const float* feat, float* coeff, float* rhs_b, mpde_stream_t stream);

/* Device workspace bytes mpde_template_grad needs (fp64 partial sums of grad_theta). */
size_t mpde_template_workspace_bytes(const mpde_problem* prob, const mpde_template* t);

/* Chain rule through the template: from grad_coeff = dl/dc and grad_rhs = dl/db (e.g. the
 * outputs of mpde_solve_bwd) writes grad_theta = dl/dtheta summed over the batch
 * (deterministic fixed-order fp64 reduction) and, if grad_feat != NULL, dl/du~ per PDE
 * (the contribution through c and b only). */
int mpde_template_grad(const mpde_problem* prob, const mpde_template* t, const float* theta,
                       const float* feat, const float* grad_coeff, const float* grad_rhs,
                       float* grad_theta, float* grad_feat, void* workspace,
                       size_t workspace_bytes, mpde_stream_t stream);

/* ---- launch profiler (process-wide, not thread-safe; off by default) ------------
 * Between begin and end every library launch is bracketed by CUDA events on the
 * stream it is launched on.  end() synchronises and returns, per launch class,
 * the summed event time (ms) and the launch count, and pts[0..31], points processed:
 * pts[0..6] by the S pass-2 kernel per epilogue kind on levels >= 1, pts[9..15] the same on
 * level 0, pts[8] / pts[7] by the S pass-1 kernel on levels >= 1 / level 0, pts[16..22] by
 * the one-kernel t-marching S apply per epilogue kind on level 0, pts[24..30] the same on
 * levels >= 1.
 * Classes: 0 S pass 1 (schur_g, levels >= 1), 1 S pass 2 (schur_out, levels >= 1),
 * 2 fp64 residual, 3 condense, 4 back-substitution, 5 grid transfers, 6 PCG/smoother
 * vector ops, 7 per-PDE scalar logic, 8 coarsest solve, 9 hierarchy build,
 * 10 forward/backward epilogues, 11 S pass 2 on level 0, 12 S pass 1 on level 0,
 * 13 t-marching S apply on level 0, 14 t-marching S apply on levels >= 1. */
#define MPDE_PROF_NCLASS 15
/* Number of kernel launches this process has issued through the library so far. */
uint64_t mpde_launch_count(void);
int mpde_profile_begin(void);
int mpde_profile_end(double* ms, int64_t* launches, uint64_t* pts);

#ifdef __cplusplus
}
#endif
#endif /* MPDE_H_ */
