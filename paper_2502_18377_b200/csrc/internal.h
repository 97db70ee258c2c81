// internal.h -- host-visible declarations shared by kernels.cu and mpde.cu
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/mpde.h"
#include "common.cuh"

namespace mpde {

enum {
  EPI_STORE = 0,
  EPI_DOT = 1,
  EPI_POWER = 2,
  EPI_RESID = 3,
  EPI_SMOOTH = 4,
  EPI_SMOOTH_LAST = 5,
  EPI_POST0 = 6
};

enum {
  SC_RHSNORM = 0,
  SC_REFRES = 1,
  SC_PASS_BEGIN = 2,
  SC_INIT = 3,
  SC_RZ0 = 4,
  SC_ALPHA = 5,
  SC_CONV = 6,
  SC_BETA = 7,
  SC_LZ_RESET = 8,
  SC_REACT = 9,
  SC_LZ_ALPHA = 10,
  SC_LZ_BETA = 11,
  SC_LZ_EIG = 12,
  SC_CORR = 13
};

struct EpiArgs {
  float* y = nullptr;        // STORE / DOT / POWER output
  float* res = nullptr;      // smoother residual (in/out)
  float* d_out = nullptr;    // next smoother direction
  float* e = nullptr;        // smoother error accumulator
  const float* dinv = nullptr;
  const float* coef = nullptr;  // per PDE [2*nu] (alpha_k, beta_k)
  int coef_stride = 0;
  int step = 0;
  const float* rdot = nullptr;  // optional dot partner
  double* part = nullptr;       // per (vector, tile) partial sums
  unsigned long long* pts = nullptr;  // profiling: points processed per EPI (or nullptr)
};

// per-PDE device state (arrays of length B)
struct PdeState {
  double* rz;
  double* rr0;
  double* rhsn;
  double* relres;
  double* lmax;
  double* lz;      // [B][64] Lanczos tridiagonal (alpha[0..31], beta[32..63])
  float* alpha;
  float* beta;
  int* act;
  int* done;
  int* iters;
  int* pass_iters;
  int* refines;
  int* status;
  int* inpass;
  int* failed;
  double* dzprev;  // ||delta|| of the previous refinement pass
  double* errest;  // estimated relative error of z after the last pass
  float tol;       // residual floor (stop when ||A^T(d-Az)||/||A^T d|| <= tol)
  float tol_z;     // error-based stop (estimated ||z - z*|| / ||z|| <= tol_z)
  float tol2_later;  // (PCG relative tolerance of refinement passes >= 2)^2
  double* tolp;      // [B] squared relative tolerance of the current pass (passes >= 2)
  float adapt_max;   // passes >= 3: options.tol_adapt (0: off; Q14)
};

// FGMRES(m) (fgmres.cu, opts.krylov = 1): per-PDE Arnoldi state, arrays over the batch
enum { GM_BEGIN = 0, GM_RESTART = 1, GM_DOTS0 = 2, GM_DOTS1 = 3, GM_NORM = 4, GM_SOLVE = 5 };
struct GmState {
  double* H;     // [B][m+1][m] Hessenberg (rotated in place: upper triangle R)
  double* g;     // [B][m+1] rotated residual vector
  double* cs;    // [B][m] Givens cosines
  double* sn;    // [B][m] Givens sines
  double* coef;  // [B][m+1] Gram-Schmidt coefficients of the current step / y at cycle end
  int* k;        // [B] Arnoldi steps of the current cycle
  int* gact;     // [B] PDE iterating at the start of the current cycle
  float* scl;    // [B] 1 / norm of the newest basis vector
};
int gm_tiles(int P);
void launch_gm_mdot(int P, int B, int j1, int m, const float* V, const float* w, double* part,
                    const int* act, cudaStream_t s);
void launch_gm_update(int P, int B, int j1, int m, const float* V, const double* coef, float* w,
                      double* part, const int* act, cudaStream_t s);
void launch_gm_scale(int P, int B, const float* sc, float* y, const int* act, cudaStream_t s);
void launch_gm_resid(int P, int B, int m, const float* rt, float* y, int first, double* part,
                     const int* act, cudaStream_t s);
void launch_gm_xupdate(int P, int B, int m, const float* Z, const GmState& g, float* x,
                       cudaStream_t s);

int ntiles(int P);
extern std::atomic<unsigned long long> g_launch_count;  // host-side count of kernel launches
int coarse_gemv_blocks(int n);
void upload_constants();

void launch_rhs_init(const Geo& G, int B, const float* c, const float* b, const float* om,
                     float* rhs, double* part, cudaStream_t s);
void launch_residual64(const Geo& G, int B, const float* c, const float* rhs, const float* b,
                       const float* om, const float* omn, const double* z64, float* r, double* part,
                       const int* act, cudaStream_t s);
void launch_apply_normal(const Geo& G, int B, const float* c, const float* z, float* q,
                         cudaStream_t s);
void launch_ndd_solve(const Geo& G, int B, const float* c, const float* r, float* t,
                      const int* act, bool f64, cudaStream_t s);
void launch_schur_rhs(const Geo& G, int B, const float* c, const float* r, const float* t,
                      float* rt, const int* act, bool f64, cudaStream_t s);
void launch_backsub(const Geo& G, int B, const float* c, const float* r, const float* dphi,
                    double* z64, const int* act, bool f64, double* part, cudaStream_t s);
// g: per-point scratch, float or double (f64) -- allocate 8 bytes per point
void launch_schur_g(const Geo& G, int nvec, int crep, const float* c, const float* x, void* g,
                    const int* act, unsigned long long* pts, bool f64, cudaStream_t s);
void launch_schur_out(int epi, const Geo& G, int nvec, int crep, const float* c, const float* x,
                      const void* g, const EpiArgs& A, const int* act, bool f64, cudaStream_t s);
// schur.cu: cf = per-point coefficients [B][2+2D][P] of S (from c), dinv = 1/diag(S)
void launch_schur_coef(const Geo& G, int B, const float* c, float* cf, cudaStream_t s);
// number of CTAs (= partial sums per vector) of the S kernels on this level
// partial sums per vector written by the S apply that schur_apply selects for nvec vectors
int schur_tiles(const Geo& G, bool f64, int nvec);
// true when this level applies S with the single fused kernel (launch_schur_fused)
bool schur_fused(const Geo& G, bool f64);
// one-kernel t-marching S apply (march.cu): 3D fp32 levels with n_y in {32,64,128}, n_x = 8k
bool use_march(const Geo& G, bool f64, int nvec);
// mid-size 3D levels (x-y plane <= 1024 points, n_t = 8..32): one launch, a cluster of t-slab
// CTAs per vector exchanging the t halo through distributed shared memory (slab.cu)
bool use_slab(const Geo& G, bool f64);
int slab_ctas(const Geo& G);
void launch_schur_slab(int epi, const Geo& G, int nvec, int crep, const void* cf, bool bf16,
                       const float* x, const EpiArgs& A, const int* act, cudaStream_t s);
// small levels (P <= 4096 per vector): both passes in one launch, one CTA per vector
bool use_small_fused(const Geo& G, bool f64);
void launch_schur_small(int epi, const Geo& G, int nvec, int crep, const float* cf, const float* x,
                        const EpiArgs& A, const int* act, cudaStream_t s);  // also needs 16-byte aligned x
int march_ctas(const Geo& G);
void launch_schur_march(int epi, const Geo& G, int nvec, int crep, const void* cf, bool bf16,
                        const float* x, const EpiArgs& A, const int* act, cudaStream_t s);
void launch_schur_fused(int epi, const Geo& G, int nvec, int crep, const float* cf,
                        const float* x, const EpiArgs& A, const int* act, cudaStream_t s);
void launch_diag_schur(const Geo& G, int B, const float* cf, float* dinv, cudaStream_t s);
// bf16 per-point coefficients (cf16: [B][2+2D][P] __nv_bfloat16) for the V-cycle's applies
// (epilogues RESID / SMOOTH / SMOOTH_LAST / POST0); only where schur_bf16_ok()
bool schur_bf16_ok(const Geo& G, bool f64);
// kernel variants applying S on a level (codes in schur.cu); mpde_hierarchy_query what = 5
void schur_variants(const Geo& G, bool f64, bool bf16_level, int nvec, int32_t out[4]);
void launch_schur_g_bf(const Geo& G, int nvec, int crep, const void* cf16, const float* x, void* g,
                       const int* act, unsigned long long* pts, cudaStream_t s);
void launch_schur_out_bf(int epi, const Geo& G, int nvec, int crep, const void* cf16,
                         const float* x, const void* g, const EpiArgs& A, const int* act,
                         cudaStream_t s);
void launch_f2bf(size_t n, const float* a, void* b, cudaStream_t s);
void launch_restrict(const Geo& Gf, const Geo& Gc, int nvec, int nfield, const float* fine,
                     float* coarse, const int* act, int crep, cudaStream_t s);
void launch_prolong(const Geo& Gf, const Geo& Gc, int nvec, const float* coarse, float* fine,
                    const int* act, cudaStream_t s);
// dense.cu: V-cycle transfers of scalar fields
void launch_restrict1(const Geo& Gf, const Geo& Gc, int nvec, const float* fine, float* coarse,
                      const int* act, cudaStream_t s);
void launch_prolong1(const Geo& Gf, const Geo& Gc, int nvec, const float* coarse, float* fine,
                     const int* act, cudaStream_t s);
void launch_smooth_start(int P, int nvec, const float* r, const float* dinv, const float* coef,
                         int coef_stride, float* res, float* d, float* e, const int* act,
                         cudaStream_t s);
void launch_pcg_update(int P, int nvec, const float* alpha, const float* p, const float* q,
                       float* x, float* r, double* part, const int* act, cudaStream_t s);
void launch_p_update(int P, int nvec, const float* beta, const float* z, float* p,
                     const int* act, cudaStream_t s);
void launch_scale(int P, int nvec, const float* sc, const float* x, float* y, const int* act,
                  cudaStream_t s);
void launch_add(int P, int nvec, const float* x, float* y, const int* act, cudaStream_t s);
void launch_lz_update(int P, int nvec, const float* y, const float* v, float* vprev,
                      const float* dinv, const float* alpha, const float* beta, double* part,
                      cudaStream_t s);
void launch_rand_fill(int P, int nvec, float* y, uint32_t seed, cudaStream_t s);
void launch_identity(int Pc, int nvec, float* x, cudaStream_t s);
void launch_coarse_invert(int n, int B, const float* cols, double* scratch, float* inv,
                          cudaStream_t s);
void launch_coarse_gemv(int n, int nvec, const float* sinv, const float* r, float* e,
                        const float* rdot, double* part, const int* act, cudaStream_t s);
void launch_scalar(int op, int B, const PdeState& st, const double* part, int nt, float tol2,
                   int max_iters, cudaStream_t s);
void launch_gm_scalar(int op, int j, int m, int P, int B, const PdeState& st, const GmState& g,
                      const double* part, float tol2, int max_iters, cudaStream_t s);
void launch_count_active(int B, const int* act, int* out, cudaStream_t s);
void launch_smooth_coef(int B, int nu, int kind, float theta, float ratio, const double* lmax,
                        float* coef, cudaStream_t s);
void launch_row_duals(const Geo& G, int B, const double* z64, float* lam, cudaStream_t s);
int step_grad_tiles(const Geo& G);
void launch_step_grad(const Geo& G, int B, const float* z, const double* dz64, const float* lam,
                      double* part, float* grad_h, cudaStream_t s);
void launch_duals(const Geo& G, int B, const float* c, const float* b, const float* om,
                  const float* omn, const double* z64, float* lam, cudaStream_t s);
void launch_grad(const Geo& G, int B, const float* c, const float* b, const float* z,
                 const float* rho, const double* dz64, float* gc, float* gb, float* gw,
                 float* gwn, float* dz_out, cudaStream_t s);
void launch_fwd_out(const Geo& G, int B, const float* c, const float* b, const double* z64,
                    float* z, float* rho, cudaStream_t s);
void launch_d2f(size_t n, const double* a, float* b, cudaStream_t s);
void launch_batch_sum(const float* x, int B, int64_t n, float* out, cudaStream_t s);
void launch_stats_out(int B, const PdeState& st, mpde_stats* out, cudaStream_t s);
// template.cu: polynomial PDE-expression template (mpde_template_*)
constexpr int kTmplMaxK = 35;  // C(3+4, 4): 3 feature fields, degree 4
constexpr int kTmplMaxR = 8;   // |M| + 1 in 3D
int template_terms(int F, int G);  // K, or -1 if (F, G) is outside 1..3 x 0..4
size_t template_partials(int P, int B, int F, int G, int M);  // fp64 partials of grad_theta
cudaError_t launch_template_coeff(int P, int B, int M, int F, int G, const float* theta,
                                  const float* feat, float* coeff, float* rhs, cudaStream_t s);
cudaError_t launch_template_grad(int P, int B, int M, int F, int G, const float* theta,
                                 const float* feat, const float* gc, const float* gb,
                                 float* gtheta, float* gfeat, double* part, cudaStream_t s);

}  // namespace mpde
