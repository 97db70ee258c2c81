// kernels.cu -- sm_100a kernels of the NeuRLP-PDE batched solve.
//
// Design: the normal matrix N = A^T A of Eq. 9
// is never formed.  Per point p, the derivative variables couple to other
// points only through phi, so N_dd (the derivative-variable block) is block-diagonal
// with one (2D)x(2D) block per point:
//     N_dd(p) = blockdiag_d T_d(i_d) + gamma gamma^T,   gamma = w_eq * c_d(p),
// and the solve is carried out on the Schur complement S = N_pp - N_pd N_dd^-1 N_dp
// over u_phi (one scalar per point) -- the same z* (exact block elimination).
// S phi is applied matrix-free as the phi-component of N zhat, zhat = (phi, -w),
// w = N_dd^-1 N_dp phi, in two passes: schur_g computes the per-point scalar
//     g(p) = sigma(p) (w_eq c_phi phi - sum_d gamma_d . T_d^-1 (K_d phi)(p))
// (the equation-row value of zhat) and schur_out gathers the rows along every axis.
//
// All kernels: grid = (tiles of kThreads points, vectors); a vector v belongs to PDE
// v / crep (crep > 1 only for the coarsest-level probing).  act[pde] == 0 skips the
// whole CTA (converged / failed PDEs).
#include "common.cuh"
#include <cuda_bf16.h>

#include "internal.h"

namespace mpde {

__constant__ float cA[2][5][5];
__constant__ double cAd[2][5][5];

// ----------------------------------------------------------------------------------
// Full normal operator at one point: out = (N z)(p), all 1+2D components.
// z(m, q) returns field m at point q.  T = float or double accumulation.
// Eq. 9 with the rows of Eqs. 3-7.
// ----------------------------------------------------------------------------------
template <int D, typename T, bool WANT_PHI, bool WANT_D, class Z>
__device__ __forceinline__ void normal_point(const Geo& G, const float* __restrict__ cb, Z z,
                                             int p, const int* idx, T* out) {
  constexpr int M = 1 + 2 * D;
  const int P = G.P;
  const T we = G.we, wb = G.wb, wr = G.wr, ws = G.ws;
  T e = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) e += T(cb[m * P + p]) * z(m, p);
  e *= we;
#pragma unroll
  for (int m = 0; m < M; ++m) out[m] = (m == 0 ? WANT_PHI : WANT_D) ? we * T(cb[m * P + p]) * e : T(0);
  if (WANT_PHI && on_boundary<D>(G, idx)) out[0] += wb * wb * z(0, p);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const T h = sizeof(T) == 8 ? T(G.hd[d]) : T(G.h[d]);
    const T h2 = sizeof(T) == 8 ? T(G.h2d[d]) : T(G.h2[d]);
    const int lo = WANT_PHI ? max(0, i - 4) : i, hi = WANT_PHI ? min(n - 1, i + 4) : i;
    for (int ip = lo; ip <= hi; ++ip) {
      const int di = ip - i;
      const int cls = fd_cls(ip, n), st = fd_start(cls), j = i - (ip + st);
      const bool der = (j >= 0) && (j < 5);
      const bool sm = (di >= -1) && (di <= 1);
      if (!der && !sm) continue;
      const int pp = p + di * s;
      T D1 = 0, D2 = 0;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        T zv = z(0, pp + (st + q) * s);
        if (sizeof(T) == 8) {
          D1 += T(cAd[0][cls][q]) * zv;
          D2 += T(cAd[1][cls][q]) * zv;
        } else {
          D1 += T(cA[0][cls][q]) * zv;
          D2 += T(cA[1][cls][q]) * zv;
        }
      }
      const T zd1 = z(1 + 2 * d, pp), zd2 = z(2 + 2 * d, pp);
      const T R1 = wr * (h * zd1 - D1), R2 = wr * (h2 * zd2 - D2);
      if (WANT_PHI && der) {
        if (sizeof(T) == 8)
          out[0] -= wr * (T(cAd[0][cls][j]) * R1 + T(cAd[1][cls][j]) * R2);
        else
          out[0] -= wr * (T(cA[0][cls][j]) * R1 + T(cA[1][cls][j]) * R2);
      }
      if (WANT_D && di == 0) {
        out[1 + 2 * d] += wr * h * R1 + T(neu_w2(G, d, i)) * zd1;  // + Neumann row
        out[2 + 2 * d] += wr * h2 * R2;
      }
      if (sm) {
        const bool fw = ip <= n - 2, bw = ip >= 1;
        const T z0 = z(0, pp);
        const T sp = fw ? ws * (z0 + h * zd1 + T(0.5) * h2 * zd2 - z(0, pp + s)) : T(0);
        const T sn = bw ? ws * (z0 - h * zd1 + T(0.5) * h2 * zd2 - z(0, pp - s)) : T(0);
        if (di == 0) {
          if (WANT_PHI) out[0] += ws * (sp + sn);
          if (WANT_D) {
            out[1 + 2 * d] += ws * h * (sp - sn);
            out[2 + 2 * d] += ws * T(0.5) * h2 * (sp + sn);
          }
        } else if (WANT_PHI && di == -1) {
          out[0] -= ws * sp;
        } else if (WANT_PHI && di == 1) {
          out[0] -= ws * sn;
        }
      }
    }
  }
}

// Apply N_dd(p)^-1 to y (indices 1..2D of a length-M array), Sherman-Morrison on
// blockdiag(T_d) + gamma gamma^T.  Result overwrites y[1..2D].
template <int D, typename T>
__device__ __forceinline__ void ndd_solve(const Geo& G, const float* __restrict__ cb, int p,
                                          const int* idx, T* y) {
  const int P = G.P;
  T u[2 * D], t[2 * D];
  T su = 0, st_ = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int i = idx[d], n = G.n[d];
    T t11, t12, t22;
    tinv<T>(sizeof(T) == 8 ? T(G.hd[d]) : T(G.h[d]), T(G.wr), T(G.ws), i <= n - 2, i >= 1, t11, t12,
            t22, T(neu_w2(G, d, i)));
    const T g1 = T(G.we) * T(cb[(1 + 2 * d) * P + p]), g2 = T(G.we) * T(cb[(2 + 2 * d) * P + p]);
    u[2 * d] = t11 * g1 + t12 * g2;
    u[2 * d + 1] = t12 * g1 + t22 * g2;
    t[2 * d] = t11 * y[1 + 2 * d] + t12 * y[2 + 2 * d];
    t[2 * d + 1] = t12 * y[1 + 2 * d] + t22 * y[2 + 2 * d];
    su += g1 * u[2 * d] + g2 * u[2 * d + 1];
    st_ += g1 * t[2 * d] + g2 * t[2 * d + 1];
  }
  const T f = st_ / (T(1) + su);
#pragma unroll
  for (int q = 0; q < 2 * D; ++q) y[1 + q] = t[q] - u[q] * f;
}

// ----------------------------------------------------------------------------------
// K0 rhs_init: rhs = A^T d, pointwise (Eq. 9 right-hand side; only equation and
// boundary rows have non-zero d).  Also the per-PDE partial of ||rhs||^2.
// ----------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kThreads) k_rhs_init(Geo G, const float* __restrict__ c,
                                                      const float* __restrict__ b,
                                                      const float* __restrict__ om,
                                                      float* __restrict__ rhs, double* part) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double nrm = 0;
  if (p < P) {
    int idx[D];
    unravel<D>(G, p, idx);
    const float* cb = c + (size_t)v * M * P;
    const float bv = b[(size_t)v * P + p];
    const float bnd = on_boundary<D>(G, idx) ? G.wb * G.wb * om[(size_t)v * P + p] : 0.f;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      float r = G.we * G.we * cb[m * P + p] * bv + (m == 0 ? bnd : 0.f);
      rhs[((size_t)v * M + m) * P + p] = r;
      nrm += double(r) * r;
    }
  }
  nrm = block_sum(nrm);
  if (threadIdx.x == 0) part[(size_t)v * gridDim.x + blockIdx.x] = nrm;
}

// ----------------------------------------------------------------------------------
// K9 refine_residual: r = rhs - N z (z fp64, fp64 accumulation), partial ||r||^2.
// z64 == nullptr means z = 0.  rhs == nullptr means rhs = A^T d formed here in fp64
// from (c, b, omega) (K0 fused: forming it in fp32 would perturb z* by cond * 6e-8).
// ----------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kThreads) k_residual64(Geo G, const float* __restrict__ c,
                                                        const float* __restrict__ rhs,
                                                        const float* __restrict__ bb,
                                                        const float* __restrict__ om,
                                                        const float* __restrict__ omn,
                                                        const double* __restrict__ z64,
                                                        float* __restrict__ r, double* part,
                                                        const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double nrm = 0;
  if (p < P) {
    int idx[D];
    unravel<D>(G, p, idx);
    const float* cb = c + (size_t)v * M * P;
    double out[M];
    if (z64) {
      const double* zb = z64 + (size_t)v * M * P;
      auto zf = [&](int m, int q) -> double { return zb[m * P + q]; };
      normal_point<D, double, true, true>(G, cb, zf, p, idx, out);
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) out[m] = 0.0;
    }
    double bv = 0.0, wv = 0.0;
    double nv[D];  // Neumann data rows: w_bnd^2 omega_n[d] on the (d,1) slot
#pragma unroll
    for (int d = 0; d < D; ++d) nv[d] = 0.0;
    if (!rhs) {
      const double we = G.we, wb = G.wb;
      bv = we * we * double(bb[(size_t)v * P + p]);
      wv = on_boundary<D>(G, idx) ? wb * wb * double(om[(size_t)v * P + p]) : 0.0;
      if (omn) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float nw = neu_w2(G, d, idx[d]);
          if (nw != 0.f) nv[d] = double(nw) * double(omn[((size_t)v * D + d) * P + p]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double extra = m == 0 ? wv : 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d)
        if (m == 1 + 2 * d) extra += nv[d];
      const double rh = rhs ? double(rhs[((size_t)v * M + m) * P + p])
                            : double(cb[m * P + p]) * bv + extra;
      double rv = rh - out[m];
      r[((size_t)v * M + m) * P + p] = float(rv);
      nrm += rv * rv;
    }
  }
  nrm = block_sum(nrm);
  if (threadIdx.x == 0) part[(size_t)v * gridDim.x + blockIdx.x] = nrm;
}

// K1 normal_apply for the operator parity test: q = N z (fp32 in/out, fp64 accumulation).
template <int D>
__global__ void __launch_bounds__(kThreads) k_apply_normal(Geo G, const float* __restrict__ c,
                                                          const float* __restrict__ z,
                                                          float* __restrict__ q) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const float* cb = c + (size_t)v * M * P;
  const float* zb = z + (size_t)v * M * P;
  auto zf = [&](int m, int qq) -> double { return double(zb[m * P + qq]); };
  double out[M];
  normal_point<D, double, true, true>(G, cb, zf, p, idx, out);
#pragma unroll
  for (int m = 0; m < M; ++m) q[((size_t)v * M + m) * P + p] = float(out[m]);
}

// ----------------------------------------------------------------------------------
// Condensation of a full right-hand side r (M fields):
//   k_ndd_solve:  t_d = N_dd^-1 r_d (pointwise)
//   k_schur_rhs:  rt = r_phi - (N (0, t))_phi
// ----------------------------------------------------------------------------------
// T = arithmetic type (float or double); storage stays fp32.  With large coefficients
// the per-point Sherman-Morrison cancels (u = T^-1 gamma ~ c/h^4), so the default path
// (mpde_options.precision = 1) runs condensation and the PCG operator in fp64.
template <typename T>
__device__ __forceinline__ T fdw(int k, int cls, int q) {
  return sizeof(T) == 8 ? T(cAd[k][cls][q]) : T(cA[k][cls][q]);
}
template <typename T>
__device__ __forceinline__ T geo_h(const Geo& G, int d) {
  return sizeof(T) == 8 ? T(G.hd[d]) : T(G.h[d]);
}
template <typename T>
__device__ __forceinline__ T geo_h2(const Geo& G, int d) {
  return sizeof(T) == 8 ? T(G.h2d[d]) : T(G.h2[d]);
}

template <int D, typename T>
__global__ void __launch_bounds__(kThreads) k_ndd_solve(Geo G, const float* __restrict__ c,
                                                       const float* __restrict__ r,
                                                       float* __restrict__ t, const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const float* cb = c + (size_t)v * M * P;
  T y[M];
#pragma unroll
  for (int m = 0; m < M; ++m) y[m] = r[((size_t)v * M + m) * P + p];
  ndd_solve<D, T>(G, cb, p, idx, y);
  t[((size_t)v * M) * P + p] = 0.f;
#pragma unroll
  for (int m = 1; m < M; ++m) t[((size_t)v * M + m) * P + p] = float(y[m]);
}

template <int D, typename T>
__global__ void __launch_bounds__(kThreads) k_schur_rhs(Geo G, const float* __restrict__ c,
                                                       const float* __restrict__ r,
                                                       const float* __restrict__ t,
                                                       float* __restrict__ rt, const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const float* cb = c + (size_t)v * M * P;
  const float* tb = t + (size_t)v * M * P;
  auto zf = [&](int m, int q) -> T { return m == 0 ? T(0) : T(tb[m * P + q]); };
  T out[M];
  normal_point<D, T, true, false>(G, cb, zf, p, idx, out);
  rt[(size_t)v * P + p] = float(T(r[((size_t)v * M) * P + p]) - out[0]);
}

// Back-substitution after the condensed solve:
//   delta_d = N_dd^-1 (r_d - (N (dphi, 0))_d);  z64 += (dphi, delta_d)
// Also the per-PDE partials of ||delta||^2 (part) and ||z_new||^2 (part + nvec*tiles) for
// the error-based refinement stop.
template <int D, typename T>
__global__ void __launch_bounds__(kThreads) k_backsub(Geo G, const float* __restrict__ c,
                                                     const float* __restrict__ r,
                                                     const float* __restrict__ dphi,
                                                     double* __restrict__ z64, const int* act,
                                                     double* part) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double dd = 0.0, zz = 0.0;
  if (p < P) {
    int idx[D];
    unravel<D>(G, p, idx);
    const float* cb = c + (size_t)v * M * P;
    const float* xb = dphi + (size_t)v * P;
    auto zf = [&](int m, int q) -> T { return m == 0 ? T(xb[q]) : T(0); };
    T out[M];
    normal_point<D, T, false, true>(G, cb, zf, p, idx, out);
    T y[M];
#pragma unroll
    for (int m = 1; m < M; ++m) y[m] = T(r[((size_t)v * M + m) * P + p]) - out[m];
    ndd_solve<D, T>(G, cb, p, idx, y);
    y[0] = T(xb[p]);
    double* zb = z64 + (size_t)v * M * P;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double dm = double(y[m]);
      const double zn = zb[m * P + p] + dm;
      zb[m * P + p] = zn;
      dd += dm * dm;
      zz += zn * zn;
    }
  }
  dd = block_sum(dd);
  if (threadIdx.x == 0) part[(size_t)v * gridDim.x + blockIdx.x] = dd;
  zz = block_sum(zz);
  if (threadIdx.x == 0) part[(size_t)gridDim.y * gridDim.x + (size_t)v * gridDim.x + blockIdx.x] = zz;
}

// ----------------------------------------------------------------------------------
// Grid transfers.  R = P^T / 2^(coarsened dims)  (full weighting, P:278 / reading Q12)
// ----------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kThreads) k_restrict(Geo Gf, Geo Gc, int nfield,
                                                      const float* __restrict__ fine,
                                                      float* __restrict__ coarse, const int* act,
                                                      int crep) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y, Pc = Gc.P, Pf = Gf.P;
  if (act && !act[v / crep]) return;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= Pc) return;
  int cidx[D];
  unravel<D>(Gc, I, cidx);
  int lo[D], cnt[D];
  float scale = 1.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (Gc.n[d] == Gf.n[d]) {
      lo[d] = cidx[d];
      cnt[d] = 1;
    } else {
      lo[d] = max(0, 2 * cidx[d] - 1);
      cnt[d] = min(Gf.n[d] - 1, 2 * cidx[d] + 2) - lo[d] + 1;
      scale *= 0.5f;
    }
  }
  for (int f = 0; f < nfield; ++f) {
    const float* fb = fine + ((size_t)v * nfield + f) * Pf;
    float acc = 0.f;
    if (D == 2) {
      for (int a = 0; a < cnt[0]; ++a) {
        const int i0 = lo[0] + a;
        const float w0 = pw(i0, cidx[0], Gf.n[0], Gc.n[0]);
        if (w0 == 0.f) continue;
        for (int b2 = 0; b2 < cnt[1]; ++b2) {
          const int i1 = lo[1] + b2;
          const float w1 = pw(i1, cidx[1], Gf.n[1], Gc.n[1]);
          acc += w0 * w1 * fb[i0 * Gf.stride[0] + i1];
        }
      }
    } else if (D == 3) {
      for (int a = 0; a < cnt[0]; ++a) {
        const int i0 = lo[0] + a;
        const float w0 = pw(i0, cidx[0], Gf.n[0], Gc.n[0]);
        if (w0 == 0.f) continue;
        for (int b2 = 0; b2 < cnt[1]; ++b2) {
          const int i1 = lo[1] + b2;
          const float w1 = pw(i1, cidx[1], Gf.n[1], Gc.n[1]);
          if (w1 == 0.f) continue;
          for (int c2 = 0; c2 < cnt[2]; ++c2) {
            const int i2 = lo[2] + c2;
            const float w2 = pw(i2, cidx[2], Gf.n[2], Gc.n[2]);
            acc += w0 * w1 * w2 * fb[i0 * Gf.stride[0] + i1 * Gf.stride[1] + i2];
          }
        }
      }
    } else {  // 4D
      for (int a = 0; a < cnt[0]; ++a) {
        const int i0 = lo[0] + a;
        const float w0 = pw(i0, cidx[0], Gf.n[0], Gc.n[0]);
        if (w0 == 0.f) continue;
        for (int b2 = 0; b2 < cnt[1]; ++b2) {
          const int i1 = lo[1] + b2;
          const float w1 = pw(i1, cidx[1], Gf.n[1], Gc.n[1]);
          if (w1 == 0.f) continue;
          for (int c2 = 0; c2 < cnt[2]; ++c2) {
            const int i2 = lo[2] + c2;
            const float w2 = pw(i2, cidx[2], Gf.n[2], Gc.n[2]);
            if (w2 == 0.f) continue;
            for (int e2 = 0; e2 < cnt[D - 1]; ++e2) {
              const int i3 = lo[D - 1] + e2;
              const float w3 = pw(i3, cidx[D - 1], Gf.n[D - 1], Gc.n[D - 1]);
              acc += w0 * w1 * w2 * w3 * fb[i0 * Gf.stride[0] + i1 * Gf.stride[1] + i2 * Gf.stride[2] + i3];
            }
          }
        }
      }
    }
    coarse[((size_t)v * nfield + f) * Pc + I] = acc * scale;
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_prolong(Geo Gf, Geo Gc, const float* __restrict__ coarse,
                                                     float* __restrict__ fine, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y, Pf = Gf.P, Pc = Gc.P;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= Pf) return;
  int idx[D];
  unravel<D>(Gf, p, idx);
  int I0[D], I1[D];
  float w0[D], w1[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int i = idx[d], nf = Gf.n[d], nc = Gc.n[d];
    if (nf == nc) {
      I0[d] = I1[d] = i;
      w0[d] = 1.f;
      w1[d] = 0.f;
    } else if ((nf & 1) == 0) {
      const int Ii = i >> 1;
      int J = (i & 1) ? Ii + 1 : Ii - 1;
      J = J < 0 ? 0 : (J > nc - 1 ? nc - 1 : J);
      I0[d] = Ii;
      I1[d] = J;
      w0[d] = 0.75f;
      w1[d] = 0.25f;
    } else if ((i & 1) == 0) {
      I0[d] = I1[d] = i >> 1;
      w0[d] = 1.f;
      w1[d] = 0.f;
    } else {
      I0[d] = i >> 1;
      I1[d] = (i >> 1) + 1;
      w0[d] = 0.5f;
      w1[d] = 0.5f;
    }
  }
  const float* cb = coarse + (size_t)v * Pc;
  float acc = 0.f;
#pragma unroll
  for (int mask = 0; mask < (1 << D); ++mask) {
    float w = 1.f;
    int off = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const bool hi = (mask >> d) & 1;
      w *= hi ? w1[d] : w0[d];
      off += (hi ? I1[d] : I0[d]) * Gc.stride[d];
    }
    if (w != 0.f) acc += w * cb[off];
  }
  fine[(size_t)v * Pf + p] = acc;
}

// ----------------------------------------------------------------------------------
// Pointwise vector kernels (PCG, smoother start, power iteration)
// ----------------------------------------------------------------------------------
// V-cycle start on a level: d = beta0 Dinv r; e = d; res = r (res may alias r).
__global__ void __launch_bounds__(kThreads) k_smooth_start(int P, const float* __restrict__ r,
                                                          const float* __restrict__ dinv,
                                                          const float* __restrict__ coef,
                                                          int coef_stride, float* res, float* d,
                                                          float* e, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const size_t o = (size_t)v * P + p;
  const float rv = r[o];
  const float dv = coef[v * coef_stride + 1] * dinv[o] * rv;
  res[o] = rv;
  d[o] = dv;
  e[o] = dv;
}

// x += alpha p; r -= alpha q; partial ||r||^2
__global__ void __launch_bounds__(kThreads) k_pcg_update(int P, const float* __restrict__ alpha,
                                                        const float* __restrict__ p_,
                                                        const float* __restrict__ q, float* x,
                                                        float* r, double* part, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double dot = 0.0;
  if (p < P) {
    const size_t o = (size_t)v * P + p;
    const float a = alpha[v];
    x[o] += a * p_[o];
    const float rv = r[o] - a * q[o];
    r[o] = rv;
    dot = double(rv) * rv;
  }
  dot = block_sum(dot);
  if (threadIdx.x == 0) part[(size_t)v * gridDim.x + blockIdx.x] = dot;
}

// p = z + beta p   (beta == 0 -> copy)
__global__ void __launch_bounds__(kThreads) k_p_update(int P, const float* __restrict__ beta,
                                                      const float* __restrict__ z, float* p_,
                                                      const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const size_t o = (size_t)v * P + p;
  const float b = beta[v];
  p_[o] = b == 0.f ? z[o] : z[o] + b * p_[o];  // p_old may be uninitialised when b == 0
}

// float4 variants of the two copy-like updates (4 points per thread: 4x the bytes in flight
// per load; the 1-point kernels above ran at ~2.6 TB/s on level 0).  Used when P % 4 == 0 and
// every pointer is 16-byte aligned; same arithmetic per point.
__global__ void __launch_bounds__(kThreads) k_smooth_start4(int P4, const float4* __restrict__ r,
                                                           const float4* __restrict__ dinv,
                                                           const float* __restrict__ coef,
                                                           int coef_stride, float4* res, float4* d,
                                                           float4* e, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P4) return;
  const size_t o = (size_t)v * P4 + p;
  const float4 rv = r[o], dn = dinv[o];
  const float c = coef[v * coef_stride + 1];
  const float4 dv = make_float4(c * dn.x * rv.x, c * dn.y * rv.y, c * dn.z * rv.z, c * dn.w * rv.w);
  res[o] = rv;
  d[o] = dv;
  e[o] = dv;
}

// float4 k_pcg_update: one CTA covers 4 of the 1-point kernel's 256-point tiles and writes
// their 4 partials into the same slots (part[v * ntiles(P) + tile]), so the consumers'
// partial count and layout are unchanged
__global__ void __launch_bounds__(kThreads) k_pcg_update4(int P4, int nt,
                                                         const float* __restrict__ alpha,
                                                         const float4* __restrict__ p_,
                                                         const float4* __restrict__ q, float4* x,
                                                         float4* r, double* part, const int* act) {
  MPDE_PDL_ENTRY();
  __shared__ double sh[kThreads / 32];
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double dot = 0.0;
  if (p < P4) {
    const size_t o = (size_t)v * P4 + p;
    const float a = alpha[v];
    const float4 pv = p_[o], qv = q[o];
    float4 xv = x[o], rv = r[o];
    xv.x += a * pv.x; xv.y += a * pv.y; xv.z += a * pv.z; xv.w += a * pv.w;
    rv.x -= a * qv.x; rv.y -= a * qv.y; rv.z -= a * qv.z; rv.w -= a * qv.w;
    x[o] = xv;
    r[o] = rv;
    dot = double(rv.x) * rv.x + double(rv.y) * rv.y + double(rv.z) * rv.z + double(rv.w) * rv.w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = dot;
  __syncthreads();
  // tile k of this CTA = float4 indices [64k, 64k + 64) = warps 2k, 2k + 1
  constexpr int kSub = kThreads / 64;
  if (threadIdx.x < kSub) {
    const int tile = blockIdx.x * kSub + threadIdx.x;
    if (tile < nt) part[(size_t)v * nt + tile] = sh[2 * threadIdx.x] + sh[2 * threadIdx.x + 1];
  }
}

__global__ void __launch_bounds__(kThreads) k_p_update4(int P4, const float* __restrict__ beta,
                                                       const float4* __restrict__ z, float4* p_,
                                                       const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P4) return;
  const size_t o = (size_t)v * P4 + p;
  const float b = beta[v];
  const float4 zv = z[o];
  if (b == 0.f) {
    p_[o] = zv;  // p_old may be uninitialised when b == 0
  } else {
    const float4 pv = p_[o];
    p_[o] = make_float4(zv.x + b * pv.x, zv.y + b * pv.y, zv.z + b * pv.z, zv.w + b * pv.w);
  }
}

// y += x (W-cycle: sum of the two coarse corrections)
__global__ void __launch_bounds__(kThreads) k_add(int P, const float* __restrict__ x, float* y,
                                                 const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const size_t o = (size_t)v * P + p;
  y[o] += x[o];
}

// generic: y = a*x (per-vector scale), or fill
__global__ void __launch_bounds__(kThreads) k_scale(int P, const float* __restrict__ s,
                                                   const float* __restrict__ x, float* y,
                                                   const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const size_t o = (size_t)v * P + p;
  y[o] = s[v] * x[o];
}

// Lanczos three-term update in the D-inner product (D = diag S):
//   w = y - alpha v - beta vprev  (written over vprev),  partial <D w, w>
__global__ void __launch_bounds__(kThreads) k_lz_update(int P, const float* __restrict__ y,
                                                       const float* __restrict__ v, float* vprev,
                                                       const float* __restrict__ dinv,
                                                       const float* __restrict__ alpha,
                                                       const float* __restrict__ beta,
                                                       double* part) {
  MPDE_PDL_ENTRY();
  const int b = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double dot = 0.0;
  if (p < P) {
    const size_t o = (size_t)b * P + p;
    const float w = y[o] - alpha[b] * v[o] - beta[b] * vprev[o];
    vprev[o] = w;
    dot = double(w) * w / dinv[o];
  }
  dot = block_sum(dot);
  if (threadIdx.x == 0) part[(size_t)b * gridDim.x + blockIdx.x] = dot;
}

// deterministic pseudo-random start vector (counter-based hash), values in [-1, 1)
__global__ void __launch_bounds__(kThreads) k_rand_fill(int P, float* y, uint32_t seed) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  // the same start vector for every PDE of the batch (no dependence on the batch position):
  // a PDE's lambda_max estimate, and with it its whole solve, is then bit-identical whether it
  // is solved alone, in a larger batch or in another rank's shard (tests/test_gpu_multirank.py)
  uint32_t h = (uint32_t)p * 0x9E3779B1u ^ seed;
  h ^= h >> 16;
  h *= 0x7FEB352Du;
  h ^= h >> 15;
  h *= 0x846CA68Bu;
  h ^= h >> 16;
  y[(size_t)v * P + p] = -1.0f + (h >> 8) * (2.0f / 16777216.0f);
}

// identity probes: x[(b*Pc + j)][p] = (p == j)
__global__ void __launch_bounds__(kThreads) k_identity(int Pc, float* x) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= Pc) return;
  x[(size_t)v * Pc + p] = (p == (v % Pc)) ? 1.f : 0.f;
}

// ----------------------------------------------------------------------------------
// Per-PDE scalar logic (one thread per PDE).  Sums the CTA partials in a fixed order
// (deterministic) and updates the PCG state.
// ----------------------------------------------------------------------------------
__device__ __forceinline__ double sum_parts(const double* part, int v, int nt) {
  double s = 0.0;
  for (int t = 0; t < nt; ++t) s += part[(size_t)v * nt + t];
  return s;
}

// Flags: done = refinement finished (converged, or failed), inpass = refined in the
// current pass, act = PCG still iterating (subset of inpass), failed = PCG breakdown
// in this pass (indefinite / non-finite) -- its partial result is still applied.
__device__ __forceinline__ void pcg_fail(const PdeState& st, int v, double val) {
  st.status[v] = isfinite(val) ? MPDE_STATUS_INDEFINITE : MPDE_STATUS_NONFINITE;
  st.failed[v] = 1;
  st.act[v] = 0;
}

// one warp per PDE: the warp sums the nt CTA partials (lane-strided, then a fixed
// shuffle tree -- deterministic), lane 0 runs the per-PDE logic.
__global__ void k_scalar(int op, int B, PdeState st, const double* part, int nt, float tol2,
                         int max_iters) {
  MPDE_PDL_ENTRY();
  const int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (v >= B) return;
  double S_ = 0.0;
  for (int t = lane; t < nt; t += 32) S_ += part[(size_t)v * nt + t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) S_ += __shfl_xor_sync(0xffffffffu, S_, o);
  if (lane != 0) return;
#define sum_parts(a, b, c) S_
  if (op == SC_RHSNORM) {  // ||A^T d||, refinement bookkeeping reset
    st.rhsn[v] = sqrt(sum_parts(part, v, nt));
    st.done[v] = st.rhsn[v] == 0.0 ? 1 : 0;
    st.iters[v] = 0;
    st.refines[v] = 0;
    st.failed[v] = 0;
    st.status[v] = st.rhsn[v] == 0.0 ? MPDE_STATUS_CONVERGED : MPDE_STATUS_MAXITER;
    st.relres[v] = st.rhsn[v] == 0.0 ? 0.0 : 1.0;
    st.errest[v] = st.rhsn[v] == 0.0 ? 0.0 : 1.0;
    st.dzprev[v] = 0.0;
    if (!isfinite(st.rhsn[v])) {
      st.status[v] = MPDE_STATUS_NONFINITE;
      st.done[v] = 1;
    }
    return;
  }
  if (op == SC_PASS_BEGIN) {  // PDEs that still need a refinement pass
    st.inpass[v] = st.done[v] ? 0 : 1;
    st.act[v] = st.inpass[v];
    if (st.inpass[v]) st.refines[v] += 1;
    {
      // pass k+1 >= 3 must shrink the error by tol_z / err_k (with a 10x margin), not by
      // tol_inner2: the relative tolerance tau = tol_z / (10 err_k), clamped to
      // [tol_inner2, adapt_max]; the error estimate of the pass then uses tau (SC_CORR)
      double t2 = (double)st.tol2_later;
      if (st.adapt_max > 0.f && st.refines[v] >= 3 && st.errest[v] > 0.0) {
        double tau = (double)st.tol_z / (10.0 * st.errest[v]);
        tau = fmin(tau, (double)st.adapt_max);
        tau = fmax(tau, sqrt((double)st.tol2_later));
        t2 = tau * tau;
      }
      st.tolp[v] = t2;
    }
    st.pass_iters[v] = 0;
    st.failed[v] = 0;
    return;
  }
  if (op == SC_REACT) {  // back-substitution / residual for every PDE of the pass
    st.act[v] = st.inpass[v];
    return;
  }
  if (op == SC_REFRES) {  // after the fp64 refinement residual
    if (!st.inpass[v]) {
      st.act[v] = 0;
      return;
    }
    const double rn = sqrt(sum_parts(part, v, nt));
    const double rel = st.rhsn[v] > 0 ? rn / st.rhsn[v] : 0.0;
    st.relres[v] = rel;
    if (!isfinite(rel) || !isfinite(st.errest[v])) {
      st.status[v] = MPDE_STATUS_NONFINITE;
      st.done[v] = 1;
    } else if (rel <= (double)st.tol ||
               (st.refines[v] >= 2 && st.errest[v] <= (double)st.tol_z)) {
      st.status[v] = MPDE_STATUS_CONVERGED;
      st.done[v] = 1;
    } else if (st.failed[v]) {
      st.done[v] = 1;
    }
    st.act[v] = 0;
    return;
  }
  if (op == SC_CORR) {  // after back-substitution: relative error estimate of z
    if (!st.inpass[v]) return;
    double S2 = 0.0;  // ||z||^2 partials live in the second half of part
    for (int t = 0; t < nt; ++t) S2 += part[(size_t)B * nt + (size_t)v * nt + t];
    const double dz = sqrt(S_), zn = sqrt(S2);
    // geometric refinement: err_k ~ ||d_k|| * rho_k with rho_k the larger of the observed
    // contraction ||d_k|| / ||d_{k-1}|| and the relative tolerance pass k was solved to
    const double est = st.refines[v] >= 2 && st.dzprev[v] > 0
                           ? dz * fmax(dz / st.dzprev[v], sqrt(st.tolp[v]))
                           : dz;
    st.dzprev[v] = dz;
    st.errest[v] = zn > 0 ? est / zn : (dz > 0 ? 1.0 : 0.0);
    return;
  }
  // Lanczos on D^-1 S (self-adjoint in <D.,.>), step index j = max_iters field:
  if (op == SC_LZ_RESET) {
    st.alpha[v] = 0.f;
    st.beta[v] = 0.f;
    return;
  }
  if (op == SC_LZ_ALPHA) {  // alpha_j = <v_j, S v_j>
    const double a = sum_parts(part, v, nt);
    st.lz[(size_t)v * 64 + max_iters] = a;
    st.alpha[v] = float(a);
    return;
  }
  if (op == SC_LZ_BETA) {  // beta_{j+1} = ||w||_D ; alpha <- 1/beta (scale of v_{j+1})
    const double b = sqrt(sum_parts(part, v, nt));
    if (max_iters >= 0) st.lz[(size_t)v * 64 + 32 + max_iters] = b;
    st.beta[v] = max_iters >= 0 ? float(b) : 0.f;
    st.alpha[v] = b > 0 ? float(1.0 / b) : 0.f;
    return;
  }
  if (op == SC_LZ_EIG) {  // largest eigenvalue of the k x k Lanczos tridiagonal (bisection)
    const int k = max_iters;
    const double* a = st.lz + (size_t)v * 64;
    const double* bb = a + 32;  // bb[j] couples j and j+1
    double lo = 1e300, hi = -1e300;
    for (int j = 0; j < k; ++j) {
      const double r = (j > 0 ? fabs(bb[j - 1]) : 0.0) + (j < k - 1 ? fabs(bb[j]) : 0.0);
      lo = fmin(lo, a[j] - r);
      hi = fmax(hi, a[j] + r);
    }
    for (int it = 0; it < 100; ++it) {  // Sturm count of eigenvalues > mid
      const double mid = 0.5 * (lo + hi);
      int cnt = 0;
      double q = 1.0;
      for (int j = 0; j < k; ++j) {
        const double b2 = j > 0 ? bb[j - 1] * bb[j - 1] : 0.0;
        q = a[j] - mid - (j > 0 ? b2 / q : 0.0);
        if (q == 0.0) q = 1e-300;
        if (q < 0) ++cnt;
      }
      if (cnt == k) hi = mid; else lo = mid;  // all eigenvalues < mid -> lmax < mid
    }
    st.lmax[v] = hi;
    return;
  }
  if (!st.act[v]) return;
  if (op == SC_INIT) {  // rr0 = ||r0||^2
    const double rr0 = sum_parts(part, v, nt);
    st.rr0[v] = rr0;
    if (!(rr0 > 0.0)) {
      if (isfinite(rr0))
        st.act[v] = 0;  // nothing left to solve in this pass
      else
        pcg_fail(st, v, rr0);
    }
    st.beta[v] = 0.f;
    return;
  }
  if (op == SC_RZ0) {
    const double rz = sum_parts(part, v, nt);
    st.rz[v] = rz;
    if (!(rz > 0.0)) pcg_fail(st, v, rz);
    st.beta[v] = 0.f;
    return;
  }
  if (op == SC_ALPHA) {
    const double pq = sum_parts(part, v, nt);
    if (!(pq > 0.0)) {
      pcg_fail(st, v, pq);
      st.alpha[v] = 0.f;
      return;
    }
    st.alpha[v] = float(st.rz[v] / pq);
    return;
  }
  if (op == SC_CONV) {
    const double rr = sum_parts(part, v, nt);
    st.iters[v] += 1;
    st.pass_iters[v] += 1;
    if (!isfinite(rr)) {
      pcg_fail(st, v, rr);
    } else if (rr <= (st.refines[v] >= 2 ? st.tolp[v] : (double)tol2) * st.rr0[v] ||
               st.pass_iters[v] >= max_iters ||
               rr <= 0.25 * (double)st.tol * st.tol * st.rhsn[v] * st.rhsn[v]) {
      // pass finished: relative inner tolerance (the fp32 limit) reached, or the outer
      // target itself (after exact back-substitution the full normal residual equals the
      // condensed one, so the last pass need not over-solve)
      st.act[v] = 0;
    }
    return;
  }
  if (op == SC_BETA) {
    const double rz = sum_parts(part, v, nt);
    if (!(rz > 0.0)) {
      pcg_fail(st, v, rz);
      return;
    }
    st.beta[v] = float(rz / st.rz[v]);
    st.rz[v] = rz;
    return;
  }
}

#undef sum_parts

// count of PDEs still active (polled by the host)
__global__ void k_count_active(int B, const int* act, int* out) {
  MPDE_PDL_ENTRY();
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < B; v += blockDim.x)
    if (act[v]) atomicAdd(&s, 1);
  __syncthreads();
  if (threadIdx.x == 0) *out = s;
}

// smoothing coefficients per PDE from lambda_max (damped Jacobi or Chebyshev,
// Saad "Iterative Methods" Alg. 12.1 recurrence): d_k = alpha_k d_{k-1} + beta_k D^-1 res_k
__global__ void k_smooth_coef(int B, int nu, int kind, float theta, float ratio,
                              const double* lmax, float* coef) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B) return;
  const double lm = lmax[v] > 0 ? lmax[v] : 1.0;
  float* cf = coef + (size_t)v * 2 * nu;
  if (kind == 0) {
    for (int k = 0; k < nu; ++k) {
      cf[2 * k] = 0.f;
      cf[2 * k + 1] = float(theta / lm);
    }
    return;
  }
  const double hi = 1.1 * lm, lo = lm / ratio;
  const double th = 0.5 * (hi + lo), de = 0.5 * (hi - lo), s1 = th / de;
  double rho = 1.0 / s1;
  cf[0] = 0.f;
  cf[1] = float(1.0 / th);
  for (int k = 1; k < nu; ++k) {
    const double rn = 1.0 / (2.0 * s1 - rho);
    cf[2 * k] = float(rn * rho);
    cf[2 * k + 1] = float(2.0 * rn / de);
    rho = rn;
  }
}

// ----------------------------------------------------------------------------------
// K10 grad epilogue (a10): rho = b - c.z, gamma = c.dz
//   grad_c = w_eq^2 (rho dz - gamma z), grad_b = w_eq^2 gamma, grad_omega = w_bnd^2 dz_phi on B
// (= P:240's d_lambda z*^T + lambda* d_z^T and -d_lambda restricted to the c, b, omega
//  entries of A and d).
// ----------------------------------------------------------------------------------
// rho: equation residual b - c.z* kept by the forward pass (computed from its fp64 z --
// recomputing it from the fp32 z output would cancel catastrophically, the derivative
// fields being O(1/h^2) larger than the residual); nullptr = recompute from z.
template <int D>
__global__ void __launch_bounds__(kThreads) k_grad(Geo G, const float* __restrict__ c,
                                                  const float* __restrict__ b,
                                                  const float* __restrict__ z,
                                                  const float* __restrict__ rho_in,
                                                  const double* __restrict__ dz64,
                                                  float* __restrict__ gc, float* __restrict__ gb,
                                                  float* __restrict__ gw, float* __restrict__ gwn,
                                                  float* __restrict__ dz_out) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const size_t base = (size_t)v * M * P + p;
  double rho = b[(size_t)v * P + p], gam = 0.0;
  double zz[M], dd[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    zz[m] = z[base + (size_t)m * P];
    dd[m] = dz64[base + (size_t)m * P];
    const double cm = c[base + (size_t)m * P];
    rho -= cm * zz[m];
    gam += cm * dd[m];
  }
  if (rho_in) rho = rho_in[(size_t)v * P + p];
  const double we2 = double(G.we) * G.we;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    gc[base + (size_t)m * P] = float(we2 * (rho * dd[m] - gam * zz[m]));
    if (dz_out) dz_out[base + (size_t)m * P] = float(dd[m]);
  }
  gb[(size_t)v * P + p] = float(we2 * gam);
  gw[(size_t)v * P + p] = on_boundary<D>(G, idx) ? float(double(G.wb) * G.wb * dd[0]) : 0.f;
  if (gwn) {  // dl/domega_n[d] = w_bnd^2 d_z,(d,1) on the Neumann faces of dim d
#pragma unroll
    for (int d = 0; d < D; ++d)
      gwn[((size_t)v * D + d) * P + p] = float(double(neu_w2(G, d, idx[d])) * dd[1 + 2 * d]);
  }
}

// forward epilogue: z = float(z64), rho = b - c.z64 (fp64)
template <int D>
__global__ void __launch_bounds__(kThreads) k_fwd_out(Geo G, const float* __restrict__ c,
                                                     const float* __restrict__ b,
                                                     const double* __restrict__ z64,
                                                     float* __restrict__ z,
                                                     float* __restrict__ rho) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const size_t base = (size_t)v * M * P + p;
  double r = b[(size_t)v * P + p];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double zv = z64[base + (size_t)m * P];
    r -= double(c[base + (size_t)m * P]) * zv;
    z[base + (size_t)m * P] = float(zv);
  }
  rho[(size_t)v * P + p] = float(r);
}

// duals lambda* = d - A z* (Eq. 10 first block row, reading Q8), fp64 from the
// forward's fp64 z, one thread per point writing every row the point owns, structured layout
// [B][2 + 5D][P]: slot 0 equation row (Eq. 3), 1 Dirichlet row (Eq. 4; 0 where the point has
// none), 2..2+D-1 Neumann row of dim d, then derivative rows (d, k = 1, 2) (Eq. 5)
// and smoothness rows (d, forward / backward) (Eqs. 6-7), 0 where a row is absent.
template <int D>
__global__ void __launch_bounds__(kThreads) k_duals(Geo G, const float* __restrict__ c,
                                                   const float* __restrict__ b,
                                                   const float* __restrict__ om,
                                                   const float* __restrict__ omn,
                                                   const double* __restrict__ z64,
                                                   float* __restrict__ lam) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D, NS = 2 + 5 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const double* zb = z64 + (size_t)v * M * P;
  const float* cb = c + (size_t)v * M * P;
  float* out = lam + (size_t)v * NS * P + p;
  double e = double(b[(size_t)v * P + p]);
#pragma unroll
  for (int m = 0; m < M; ++m) e -= double(cb[(size_t)m * P + p]) * zb[(size_t)m * P + p];
  out[0] = float(double(G.we) * e);
  out[(size_t)P] = on_boundary<D>(G, idx) ? float(double(G.wb) * (double(om[(size_t)v * P + p]) - zb[p])) : 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const bool neu = neu_w2(G, d, idx[d]) != 0.f;
    const double dat = (neu && omn) ? double(omn[((size_t)v * D + d) * P + p]) : 0.0;
    out[(size_t)(2 + d) * P] = neu ? float(double(G.wb) * (dat - zb[(size_t)(1 + 2 * d) * P + p])) : 0.f;
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const double h = G.hd[d], h2 = G.h2d[d];
    const int cls = fd_cls(i, n), st = fd_start(cls);
    double D1 = 0.0, D2 = 0.0;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double zv = zb[p + (st + q) * s];
      D1 += cAd[0][cls][q] * zv;
      D2 += cAd[1][cls][q] * zv;
    }
    const double zd1 = zb[(size_t)(1 + 2 * d) * P + p], zd2 = zb[(size_t)(2 + 2 * d) * P + p];
    out[(size_t)(2 + D + 2 * d) * P] = float(-double(G.wr) * (h * zd1 - D1));
    out[(size_t)(2 + D + 2 * d + 1) * P] = float(-double(G.wr) * (h2 * zd2 - D2));
    const double z0 = zb[p];
    out[(size_t)(2 + 3 * D + 2 * d) * P] =
        i <= n - 2 ? float(-double(G.ws) * (z0 + h * zd1 + 0.5 * h2 * zd2 - zb[p + s])) : 0.f;
    out[(size_t)(2 + 3 * D + 2 * d + 1) * P] =
        i >= 1 ? float(-double(G.ws) * (z0 - h * zd1 + 0.5 * h2 * zd2 - zb[p - s])) : 0.f;
  }
}

// duals of the derivative rows (d, k) and Taylor rows (d, fwd/bwd) of the forward solution (fp64
// z*), kept for the step gradient: [B][4D][P], slots 2d+(k-1) then 2D + 2d + {0 fwd, 1 bwd}
template <int D>
__global__ void __launch_bounds__(kThreads) k_row_duals(Geo G, const double* __restrict__ z64,
                                                       float* __restrict__ lam) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const double* zb = z64 + (size_t)v * M * P;
  float* out = lam + (size_t)v * 4 * D * P + p;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const double h = G.hd[d], h2 = G.h2d[d];
    const int cls = fd_cls(i, n), st = fd_start(cls);
    double D1 = 0.0, D2 = 0.0;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double zv = zb[p + (st + q) * s];
      D1 += cAd[0][cls][q] * zv;
      D2 += cAd[1][cls][q] * zv;
    }
    const double zd1 = zb[(size_t)(1 + 2 * d) * P + p], zd2 = zb[(size_t)(2 + 2 * d) * P + p];
    const double z0 = zb[p];
    out[(size_t)(2 * d) * P] = float(-double(G.wr) * (h * zd1 - D1));
    out[(size_t)(2 * d + 1) * P] = float(-double(G.wr) * (h2 * zd2 - D2));
    out[(size_t)(2 * D + 2 * d) * P] = i <= n - 2 ? float(-double(G.ws) * (z0 + h * zd1 + 0.5 * h2 * zd2 - zb[p + s])) : 0.f;
    out[(size_t)(2 * D + 2 * d + 1) * P] = i >= 1 ? float(-double(G.ws) * (z0 - h * zd1 + 0.5 * h2 * zd2 - zb[p - s])) : 0.f;
  }
}

// step gradient, per-point contributions reduced per (PDE, dim, CTA) in fp64: for dim d
//   sum_k (dlam_der zk + lam_der dzk) w_der k h^(k-1)
//   + [fwd row] (dlam_f z1 + lam_f dz1) w_sm + (dlam_f z2 + lam_f dz2) w_sm h
//   + [bwd row] -(dlam_b z1 + lam_b dz1) w_sm + (dlam_b z2 + lam_b dz2) w_sm h
// with d_lambda = -A d_z of those rows (d_z = the backward's fp64 solution) and lambda* kept
// by the forward (k_row_duals).
template <int D>
__global__ void __launch_bounds__(kThreads) k_step_grad(Geo G, const float* __restrict__ z,
                                                       const double* __restrict__ dz64,
                                                       const float* __restrict__ lam,
                                                       double* __restrict__ part) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double contrib[D];
#pragma unroll
  for (int d = 0; d < D; ++d) contrib[d] = 0.0;
  if (p < P) {
    int idx[D];
    unravel<D>(G, p, idx);
    const double* db = dz64 + (size_t)v * M * P;
    const float* zb = z + (size_t)v * M * P;
    const float* lb = lam + (size_t)v * 4 * D * P + p;
    const double wr = G.wr, ws = G.ws;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int n = G.n[d], s = G.stride[d], i = idx[d];
      const double h = G.hd[d], h2 = G.h2d[d];
      const int cls = fd_cls(i, n), st = fd_start(cls);
      double D1 = 0.0, D2 = 0.0;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const double dv = db[p + (st + q) * s];
        D1 += cAd[0][cls][q] * dv;
        D2 += cAd[1][cls][q] * dv;
      }
      const double d0 = db[p], d1 = db[(size_t)(1 + 2 * d) * P + p], d2 = db[(size_t)(2 + 2 * d) * P + p];
      const double z1 = zb[(size_t)(1 + 2 * d) * P + p], z2 = zb[(size_t)(2 + 2 * d) * P + p];
      const double dl1 = -wr * (h * d1 - D1), dl2 = -wr * (h2 * d2 - D2);
      const double l1 = lb[(size_t)(2 * d) * P], l2 = lb[(size_t)(2 * d + 1) * P];
      double c = (dl1 * z1 + l1 * d1) * wr + (dl2 * z2 + l2 * d2) * wr * 2.0 * h;
      if (i <= n - 2) {
        const double dlf = -ws * (d0 + h * d1 + 0.5 * h2 * d2 - db[p + s]);
        const double lf = lb[(size_t)(2 * D + 2 * d) * P];
        c += (dlf * z1 + lf * d1) * ws + (dlf * z2 + lf * d2) * ws * h;
      }
      if (i >= 1) {
        const double dlb = -ws * (d0 - h * d1 + 0.5 * h2 * d2 - db[p - s]);
        const double lbw = lb[(size_t)(2 * D + 2 * d + 1) * P];
        c += -(dlb * z1 + lbw * d1) * ws + (dlb * z2 + lbw * d2) * ws * h;
      }
      contrib[d] = c;
    }
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double sum = block_sum(contrib[d]);
    if (threadIdx.x == 0) part[((size_t)v * D + d) * gridDim.x + blockIdx.x] = sum;
  }
}

// fixed-order sum of the per-CTA partials: grad_h[v][d]
__global__ void k_step_grad_reduce(int nvd, int ntiles, const double* __restrict__ part,
                                   float* __restrict__ out) {
  MPDE_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nvd) return;
  double s = 0.0;
  for (int t = 0; t < ntiles; ++t) s += part[(size_t)i * ntiles + t];
  out[i] = float(s);
}

// out[j] = sum_b x[b][j], fixed summation order (deterministic)
__global__ void __launch_bounds__(kThreads) k_batch_sum(const float* __restrict__ x, int B,
                                                       int64_t n, float* __restrict__ out) {
  MPDE_PDL_ENTRY();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int b = 0; b < B; ++b) acc += x[(size_t)b * n + j];
  out[j] = float(acc);
}

__global__ void __launch_bounds__(kThreads) k_f2bf(size_t n, const float* __restrict__ a,
                                                   __nv_bfloat16* __restrict__ b) {
  MPDE_PDL_ENTRY();
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = __float2bfloat16_rn(a[i]);
}

__global__ void __launch_bounds__(kThreads) k_d2f(size_t n, const double* __restrict__ a, float* __restrict__ b) {
  MPDE_PDL_ENTRY();
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = float(a[i]);
}

__global__ void k_stats_out(int B, PdeState st, mpde_stats* out) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B) return;
  out[v].iters = st.iters[v];
  out[v].refines = st.refines[v];
  out[v].status = st.status[v];
  out[v].rel_res = float(st.relres[v]);
  out[v].err_est = float(st.errest[v]);
}

// ----------------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------------
static inline dim3 grid_for(int P, int nvec) { return dim3((P + kThreads - 1) / kThreads, nvec); }
int ntiles(int P) { return (P + kThreads - 1) / kThreads; }
std::atomic<unsigned long long> g_launch_count{0};

void upload_constants() {
  static bool done = false;
  if (done) return;
  const double fwd[2][5] = {{-25, 48, -36, 16, -3}, {35, -104, 114, -56, 11}};
  const double cen[2][5] = {{1, -8, 0, 8, -1}, {-1, 16, -30, 16, -1}};
  double ad[2][5][5];
  float af[2][5][5];
  for (int k = 0; k < 2; ++k) {
    const double sg = (k == 0) ? -1.0 : 1.0;  // (-1)^order
    for (int m = 0; m < 5; ++m) {
      ad[k][0][m] = ad[k][1][m] = fwd[k][m] / 12.0;
      ad[k][2][m] = cen[k][m] / 12.0;
      ad[k][3][m] = ad[k][4][m] = sg * fwd[k][4 - m] / 12.0;  // offset -4+m = -(4-m)
    }
  }
  for (int k = 0; k < 2; ++k)
    for (int c = 0; c < 5; ++c)
      for (int m = 0; m < 5; ++m) af[k][c][m] = float(ad[k][c][m]);
  cudaMemcpyToSymbol(cA, af, sizeof(af));
  cudaMemcpyToSymbol(cAd, ad, sizeof(ad));
  done = true;
}

#define DISPATCH_D(D_, ...) \
  do {                       \
    if ((D_) == 2) {         \
      constexpr int DD = 2;  \
      __VA_ARGS__;           \
    } else if ((D_) == 3) {  \
      constexpr int DD = 3;  \
      __VA_ARGS__;           \
    } else {                \
      constexpr int DD = 4;  \
      __VA_ARGS__;           \
    }                        \
  } while (0)

void launch_rhs_init(const Geo& G, int B, const float* c, const float* b, const float* om,
                     float* rhs, double* part, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_rhs_init<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, b, om, rhs, part));
}
void launch_residual64(const Geo& G, int B, const float* c, const float* rhs, const float* b,
                       const float* om, const float* omn, const double* z64, float* r, double* part,
                       const int* act, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_residual64<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, rhs, b, om, omn, z64, r, part, act));
}
void launch_apply_normal(const Geo& G, int B, const float* c, const float* z, float* q,
                         cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_apply_normal<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, z, q));
}
void launch_ndd_solve(const Geo& G, int B, const float* c, const float* r, float* t,
                      const int* act, bool f64, cudaStream_t s) {
  ++g_launch_count;
  if (f64)
    DISPATCH_D(G.D, k_ndd_solve<DD, double><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, r, t, act));
  else
    DISPATCH_D(G.D, k_ndd_solve<DD, float><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, r, t, act));
}
void launch_schur_rhs(const Geo& G, int B, const float* c, const float* r, const float* t,
                      float* rt, const int* act, bool f64, cudaStream_t s) {
  ++g_launch_count;
  if (f64)
    DISPATCH_D(G.D, k_schur_rhs<DD, double><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, r, t, rt, act));
  else
    DISPATCH_D(G.D, k_schur_rhs<DD, float><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, r, t, rt, act));
}
void launch_backsub(const Geo& G, int B, const float* c, const float* r, const float* dphi,
                    double* z64, const int* act, bool f64, double* part, cudaStream_t s) {
  ++g_launch_count;
  if (f64)
    DISPATCH_D(G.D, k_backsub<DD, double><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, r, dphi, z64, act, part));
  else
    DISPATCH_D(G.D, k_backsub<DD, float><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, r, dphi, z64, act, part));
}
void launch_restrict(const Geo& Gf, const Geo& Gc, int nvec, int nfield, const float* fine,
                     float* coarse, const int* act, int crep, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(Gf.D, k_restrict<DD><<<grid_for(Gc.P, nvec), kThreads, 0, s>>>(Gf, Gc, nfield, fine, coarse, act, crep));
}
void launch_prolong(const Geo& Gf, const Geo& Gc, int nvec, const float* coarse, float* fine,
                    const int* act, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(Gf.D, k_prolong<DD><<<grid_for(Gf.P, nvec), kThreads, 0, s>>>(Gf, Gc, coarse, fine, act));
}
static inline bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }
template <class... T>
static inline bool vec4_ok(int P, const T*... q) {
  return (P & 3) == 0 && (aligned16(q) && ...);
}
void launch_smooth_start(int P, int nvec, const float* r, const float* dinv, const float* coef,
                         int coef_stride, float* res, float* d, float* e, const int* act,
                         cudaStream_t s) {
  ++g_launch_count;
  if (vec4_ok(P, r, dinv, res, d, e)) {
    k_smooth_start4<<<grid_for(P / 4, nvec), kThreads, 0, s>>>(
        P / 4, (const float4*)r, (const float4*)dinv, coef, coef_stride, (float4*)res, (float4*)d,
        (float4*)e, act);
    return;
  }
  k_smooth_start<<<grid_for(P, nvec), kThreads, 0, s>>>(P, r, dinv, coef, coef_stride, res, d, e, act);
}
void launch_pcg_update(int P, int nvec, const float* alpha, const float* p, const float* q,
                       float* x, float* r, double* part, const int* act, cudaStream_t s) {
  ++g_launch_count;
  if (vec4_ok(P, p, q, x, r)) {
    k_pcg_update4<<<grid_for(P / 4, nvec), kThreads, 0, s>>>(
        P / 4, ntiles(P), alpha, (const float4*)p, (const float4*)q, (float4*)x, (float4*)r, part,
        act);
    return;
  }
  k_pcg_update<<<grid_for(P, nvec), kThreads, 0, s>>>(P, alpha, p, q, x, r, part, act);
}
void launch_p_update(int P, int nvec, const float* beta, const float* z, float* p,
                     const int* act, cudaStream_t s) {
  ++g_launch_count;
  if (vec4_ok(P, z, p)) {
    k_p_update4<<<grid_for(P / 4, nvec), kThreads, 0, s>>>(P / 4, beta, (const float4*)z,
                                                          (float4*)p, act);
    return;
  }
  k_p_update<<<grid_for(P, nvec), kThreads, 0, s>>>(P, beta, z, p, act);
}
void launch_add(int P, int nvec, const float* x, float* y, const int* act, cudaStream_t s) {
  ++g_launch_count;
  k_add<<<grid_for(P, nvec), kThreads, 0, s>>>(P, x, y, act);
}
void launch_scale(int P, int nvec, const float* sc, const float* x, float* y, const int* act,
                  cudaStream_t s) {
  ++g_launch_count;
  k_scale<<<grid_for(P, nvec), kThreads, 0, s>>>(P, sc, x, y, act);
}
void launch_lz_update(int P, int nvec, const float* y, const float* v, float* vprev,
                      const float* dinv, const float* alpha, const float* beta, double* part,
                      cudaStream_t s) {
  ++g_launch_count;
  k_lz_update<<<grid_for(P, nvec), kThreads, 0, s>>>(P, y, v, vprev, dinv, alpha, beta, part);
}
void launch_rand_fill(int P, int nvec, float* y, uint32_t seed, cudaStream_t s) {
  ++g_launch_count;
  k_rand_fill<<<grid_for(P, nvec), kThreads, 0, s>>>(P, y, seed);
}
void launch_identity(int Pc, int nvec, float* x, cudaStream_t s) {
  ++g_launch_count;
  k_identity<<<grid_for(Pc, nvec), kThreads, 0, s>>>(Pc, x);
}
void launch_scalar(int op, int B, const PdeState& st, const double* part, int nt, float tol2,
                   int max_iters, cudaStream_t s) {
  ++g_launch_count;
  k_scalar<<<(B * 32 + 127) / 128, 128, 0, s>>>(op, B, st, part, nt, tol2, max_iters);
}
void launch_count_active(int B, const int* act, int* out, cudaStream_t s) {
  ++g_launch_count;
  k_count_active<<<1, 256, 0, s>>>(B, act, out);
}
void launch_smooth_coef(int B, int nu, int kind, float theta, float ratio, const double* lmax,
                        float* coef, cudaStream_t s) {
  ++g_launch_count;
  k_smooth_coef<<<(B + 127) / 128, 128, 0, s>>>(B, nu, kind, theta, ratio, lmax, coef);
}
void launch_grad(const Geo& G, int B, const float* c, const float* b, const float* z,
                 const float* rho, const double* dz64, float* gc, float* gb, float* gw,
                 float* gwn, float* dz_out, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_grad<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, b, z, rho, dz64, gc, gb, gw, gwn, dz_out));
}
void launch_fwd_out(const Geo& G, int B, const float* c, const float* b, const double* z64,
                    float* z, float* rho, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_fwd_out<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, b, z64, z, rho));
}
void launch_duals(const Geo& G, int B, const float* c, const float* b, const float* om,
                  const float* omn, const double* z64, float* lam, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_duals<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, c, b, om, omn, z64, lam));
}
void launch_row_duals(const Geo& G, int B, const double* z64, float* lam, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D(G.D, k_row_duals<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, z64, lam));
}
int step_grad_tiles(const Geo& G) { return (G.P + kThreads - 1) / kThreads; }
void launch_step_grad(const Geo& G, int B, const float* z, const double* dz64, const float* lam,
                      double* part, float* grad_h, cudaStream_t s) {
  g_launch_count += 2;
  DISPATCH_D(G.D, k_step_grad<DD><<<grid_for(G.P, B), kThreads, 0, s>>>(G, z, dz64, lam, part));
  const int nvd = B * G.D;
  k_step_grad_reduce<<<(nvd + 127) / 128, 128, 0, s>>>(nvd, step_grad_tiles(G), part, grad_h);
}
void launch_batch_sum(const float* x, int B, int64_t n, float* out, cudaStream_t s) {
  ++g_launch_count;
  k_batch_sum<<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(x, B, n, out);
}
void launch_f2bf(size_t n, const float* a, void* b, cudaStream_t s) {
  ++g_launch_count;
  k_f2bf<<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(n, a, (__nv_bfloat16*)b);
}
void launch_d2f(size_t n, const double* a, float* b, cudaStream_t s) {
  ++g_launch_count;
  k_d2f<<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(n, a, b);
}
void launch_stats_out(int B, const PdeState& st, mpde_stats* out, cudaStream_t s) {
  ++g_launch_count;
  k_stats_out<<<(B + 127) / 128, 128, 0, s>>>(B, st, out);
}

}  // namespace mpde
