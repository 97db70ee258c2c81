// schur.cu -- the condensed normal operator S (Schur complement of A^T A onto u_phi).
//
// Exact algebra: with per-point alpha = w_eq c_phi, gamma_d = w_eq c_d,
// u_d = T_d^-1 gamma_d, sigma = 1/(1 + sum_d gamma_d . u_d) and the per-axis 1D operators
//   K_d   : the derivative-variable rows of N applied to phi (der + Taylor rows, Eqs. 5-7)
//   P0_d  = K_pp,d - K_d^T T_d^-1 K_d      (Schur complement of the constant part)
// the operator is
//   h(p)  = (1/sigma) * ( sigma alpha x - sum_d u~_d . (K_d x)(p) ),   u~ = sigma u
//   S x   = sum_d P0_d x - sum_d K_d^T (u~_d h) + sigma alpha h + w_bnd^2 [p in B] x.
// K_d, K_d^T and P0_d depend only on the index along axis d (13 classes near the edges,
// constant inside): their rows are tabulated on the host in fp64 (no run-time
// cancellation of the large h^-k terms) -- kTabRow = 52 floats per (axis, index):
//   [0,18)  Kf[o][k]  coefficient of x(i+o) in (K x)_k(i),      o = -4..4
//   [20,38) KT[o][k]  coefficient of q_k(i+o) in (K^T q)(i),    o = -4..4
//   [40,51) P0[o]     coefficient of x(i+o) in (P0 x)(i),       o = -5..5
// Per point the kernels read cf = [sigma alpha, 1/sigma, u~ (2D)] (2+2D floats).
#include "common.cuh"
#include <cuda_bf16.h>
#include <type_traits>
// A/B build switch: MPDE_B22_MINB = pass-2 CTAs per SM the register allocation targets
// (3: 80 registers; 4 = 64 registers measured slower, profiles/r2_b22_regs_ab.txt)
constexpr int kSmallThreads = 64;  // CTA size of the small-level (<= MPDE_SMALLP points) kernels
#ifndef MPDE_B22_MINB
#define MPDE_B22_MINB 3
#endif

#include "internal.h"

#include <cstdlib>

namespace mpde {

template <int D>
__global__ void __launch_bounds__(kThreads) k_schur_coef(Geo G, const float* __restrict__ c,
                                                        float* __restrict__ cf) {
  MPDE_PDL_ENTRY();
  constexpr int M = 1 + 2 * D, NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const float* cb = c + (size_t)v * M * P;
  float* out = cf + (size_t)v * NC * P;
  const double we = G.we;
  double u[2 * D];
  double s = 1.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double t11, t12, t22;
    tinv<double>(G.hd[d], G.wr, G.ws, idx[d] <= G.n[d] - 2, idx[d] >= 1, t11, t12, t22,
                 double(neu_w2(G, d, idx[d])));
    const double g1 = we * cb[(1 + 2 * d) * P + p], g2 = we * cb[(2 + 2 * d) * P + p];
    u[2 * d] = t11 * g1 + t12 * g2;
    u[2 * d + 1] = t12 * g1 + t22 * g2;
    s += g1 * u[2 * d] + g2 * u[2 * d + 1];
  }
  const double sig = 1.0 / s;
  out[p] = float(sig * we * cb[p]);
  out[P + p] = float(s);
#pragma unroll
  for (int q = 0; q < 2 * D; ++q) out[(size_t)(2 + q) * P + p] = float(sig * u[q]);
}

__device__ __forceinline__ const float* tab_row(const Geo& G, int d, int i) {
  return G.tab + G.tab_off[d] + i * kTabRow;
}

// pass 1: h(p)
template <int D, typename T>
__device__ __forceinline__ T schur_h_point(const Geo& G, const float* __restrict__ cf,
                                           const float* __restrict__ x, int p, const int* idx) {
  const int P = G.P;
  T g = T(cf[p]) * T(x[p]);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const float* row = tab_row(G, d, i);
    T k1 = 0, k2 = 0;
    if (i >= 2 && i <= n - 3) {
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const T xv = x[p + o * s];
        k1 += T(__ldg(row + (o + 4) * 2)) * xv;
        k2 += T(__ldg(row + (o + 4) * 2 + 1)) * xv;
      }
    } else {
      const int lo = max(-4, -i), hi = min(4, n - 1 - i);
      for (int o = lo; o <= hi; ++o) {
        const T xv = x[p + o * s];
        k1 += T(__ldg(row + (o + 4) * 2)) * xv;
        k2 += T(__ldg(row + (o + 4) * 2 + 1)) * xv;
      }
    }
    g -= T(cf[(size_t)(2 + 2 * d) * P + p]) * k1 + T(cf[(size_t)(3 + 2 * d) * P + p]) * k2;
  }
  return T(cf[P + p]) * g;
}

// pass 2: (S x)(p)
template <int D, typename T>
__device__ __forceinline__ T schur_s_point(const Geo& G, const float* __restrict__ cf,
                                           const float* __restrict__ x, const T* __restrict__ hb,
                                           int p, const int* idx) {
  const int P = G.P;
  T acc = T(cf[p]) * hb[p];
  if (on_boundary<D>(G, idx)) acc += T(G.wb) * T(G.wb) * T(x[p]);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const float* row = tab_row(G, d, i);
    const float* u1 = cf + (size_t)(2 + 2 * d) * P;
    const float* u2 = cf + (size_t)(3 + 2 * d) * P;
    if (i >= 7 && i <= n - 8) {  // P0 reach 4 and K^T reach 2 away from the edge classes
#pragma unroll
      for (int o = -4; o <= 4; ++o) acc += T(__ldg(row + kTabP0 + o + 5)) * T(x[p + o * s]);
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const int q = p + o * s;
        acc -= (T(__ldg(row + kTabKT + (o + 4) * 2)) * T(u1[q]) +
                T(__ldg(row + kTabKT + (o + 4) * 2 + 1)) * T(u2[q])) * hb[q];
      }
    } else {
      const int lo = max(-5, -i), hi = min(5, n - 1 - i);
      for (int o = lo; o <= hi; ++o) acc += T(__ldg(row + kTabP0 + o + 5)) * T(x[p + o * s]);
      const int lo2 = max(-4, -i), hi2 = min(4, n - 1 - i);
      for (int o = lo2; o <= hi2; ++o) {
        const int q = p + o * s;
        acc -= (T(__ldg(row + kTabKT + (o + 4) * 2)) * T(u1[q]) +
                T(__ldg(row + kTabKT + (o + 4) * 2 + 1)) * T(u2[q])) * hb[q];
      }
    }
  }
  return acc;
}

template <int D, typename T>
__global__ void __launch_bounds__(kThreads) k_schur_h(Geo G, const float* __restrict__ cf, int crep,
                                                     const float* __restrict__ x,
                                                     T* __restrict__ hout, const int* act,
                                                     unsigned long long* pts) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  hout[(size_t)v * P + p] =
      schur_h_point<D, T>(G, cf + (size_t)pde * NC * P, x + (size_t)v * P, p, idx);
  if (pts && threadIdx.x == 0) atomicAdd(pts, (unsigned long long)min(kThreads, P - p));
}

// pass 2 with the fused PCG / smoother epilogues (same contract as EpiArgs in internal.h)
template <int D, int EPI, typename T>
__global__ void __launch_bounds__(kThreads) k_schur_s(Geo G, const float* __restrict__ cf, int crep,
                                                     const float* __restrict__ x,
                                                     const T* __restrict__ hb, EpiArgs A,
                                                     const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double dot = 0.0;
  if (p < P) {
    int idx[D];
    unravel<D>(G, p, idx);
    const size_t o = (size_t)v * P + p;
    const float q = float(schur_s_point<D, T>(G, cf + (size_t)pde * NC * P, x + (size_t)v * P,
                                              hb + (size_t)v * P, p, idx));
    if (EPI == EPI_STORE) {
      A.y[o] = q;
    } else if (EPI == EPI_DOT) {
      A.y[o] = q;
      dot = double(x[o]) * q;
    } else if (EPI == EPI_POWER) {  // Lanczos step: y = D^-1 S x, partial <x, S x>
      A.y[o] = A.dinv[o] * q;
      dot = double(x[o]) * q;
    } else if (EPI == EPI_RESID) {
      A.res[o] = A.res[o] - q;
    } else if (EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST) {
      const float al = A.coef[pde * A.coef_stride + 2 * A.step];
      const float be = A.coef[pde * A.coef_stride + 2 * A.step + 1];
      const float res = A.res[o] - q;
      const float dn = al * x[o] + be * A.dinv[o] * res;
      const float e = A.e[o] + dn;
      A.e[o] = e;
      if (EPI == EPI_SMOOTH) {
        A.res[o] = res;
        A.d_out[o] = dn;
      }
      if (A.rdot) dot = double(A.rdot[o]) * e;
    } else if (EPI == EPI_POST0) {
      const float be = A.coef[pde * A.coef_stride + 1];
      const float res = A.res[o] - q;
      const float dn = be * A.dinv[o] * res;
      const float e = A.e[o] + x[o] + dn;
      A.e[o] = e;
      A.res[o] = res;
      A.d_out[o] = dn;
      if (A.rdot) dot = double(A.rdot[o]) * e;
    }
  }
  if (A.pts && threadIdx.x == 0 && p < P)
    atomicAdd(A.pts + EPI, (unsigned long long)min(kThreads, P - p));
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (threadIdx.x == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------------
// Small levels (P <= kSmallFusedP points per vector, e.g. the (8,16,16) level of C4): both
// passes in ONE launch, one CTA per vector.  x is staged in shared memory, h is computed for
// every point into shared memory, one barrier, then S x with the fused epilogue.  The
// two-pass kernels need two launches of a few thousand points each on these levels, which
// are launch-latency bound (round-1 launch list: ~10 us per coarse pass for 65 k points).
// ---------------------------------------------------------------------------------
constexpr int kSmallFusedP = 4096;
constexpr int kSmallFusedThreads = 512;

template <int EPI>
__device__ __forceinline__ double point_epilogue(const EpiArgs& A, int pde, size_t o, float xo, float q) {
  double dot = 0.0;
  if (EPI == EPI_STORE) {
    A.y[o] = q;
  } else if (EPI == EPI_DOT) {
    A.y[o] = q;
    dot = double(xo) * q;
  } else if (EPI == EPI_POWER) {
    A.y[o] = A.dinv[o] * q;
    dot = double(xo) * q;
  } else if (EPI == EPI_RESID) {
    A.res[o] = A.res[o] - q;
  } else if (EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST) {
    const float al = A.coef[pde * A.coef_stride + 2 * A.step];
    const float be = A.coef[pde * A.coef_stride + 2 * A.step + 1];
    const float res = A.res[o] - q;
    const float dn = al * xo + be * A.dinv[o] * res;
    const float e = A.e[o] + dn;
    A.e[o] = e;
    if (EPI == EPI_SMOOTH) {
      A.res[o] = res;
      A.d_out[o] = dn;
    }
    if (A.rdot) dot = double(A.rdot[o]) * e;
  } else if (EPI == EPI_POST0) {
    const float be = A.coef[pde * A.coef_stride + 1];
    const float res = A.res[o] - q;
    const float dn = be * A.dinv[o] * res;
    const float e = A.e[o] + xo + dn;
    A.e[o] = e;
    A.res[o] = res;
    A.d_out[o] = dn;
    if (A.rdot) dot = double(A.rdot[o]) * e;
  }
  return dot;
}

template <int D, int EPI>
__global__ void __launch_bounds__(kSmallFusedThreads) k_schur_small(Geo G, const float* __restrict__ cf,
                                                                   int crep, const float* __restrict__ x,
                                                                   EpiArgs A, const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  extern __shared__ __align__(16) float ssm[];
  const int v = blockIdx.x, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  float* xs = ssm;       // [P]
  float* hs = ssm + P;   // [P]
  const float* xb = x + (size_t)v * P;
  const float* cb = cf + (size_t)pde * NC * P;
  for (int p = threadIdx.x; p < P; p += blockDim.x) xs[p] = xb[p];
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int idx[D];
    unravel<D>(G, p, idx);
    hs[p] = schur_h_point<D, float>(G, cb, xs, p, idx);
  }
  __syncthreads();
  double dot = 0.0;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int idx[D];
    unravel<D>(G, p, idx);
    const float q = schur_s_point<D, float>(G, cb, xs, hs, p, idx);
    dot += point_epilogue<EPI>(A, pde, (size_t)v * P + p, xs[p], q);
  }
  if (A.pts && threadIdx.x == 0) atomicAdd(A.pts + EPI, (unsigned long long)P);
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (threadIdx.x == 0) A.part[v] = dot;
  }
}

// 1/diag(S) (smoother diagonal), fp64: diag = sum_d P0_d(i,i) + w_bnd^2 [B]
//   + (sigma alpha) dh(p)/dx(p) - sum_d sum_o sum_k KT[o][k] u~_dk(q) dh(q)/dx(p), q = p + o e_d
template <int D>
__global__ void __launch_bounds__(kThreads) k_schur_diag(Geo G, const float* __restrict__ cf,
                                                        float* __restrict__ dinv) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int idx[D];
  unravel<D>(G, p, idx);
  const float* cb = cf + (size_t)v * NC * P;
  double dhp = cb[p];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float* row = tab_row(G, d, idx[d]);
    dhp -= double(cb[(size_t)(2 + 2 * d) * P + p]) * row[8] + double(cb[(size_t)(3 + 2 * d) * P + p]) * row[9];
  }
  dhp *= double(cb[P + p]);
  double diag = double(cb[p]) * dhp + (on_boundary<D>(G, idx) ? double(G.wb) * G.wb : 0.0);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const float* row = tab_row(G, d, i);
    diag += row[kTabP0 + 5];
    for (int o = max(-4, -i); o <= min(4, n - 1 - i); ++o) {
      const int q = p + o * s;
      double dh;
      if (o == 0) {
        dh = dhp;
      } else {
        const float* rq = tab_row(G, d, i + o);  // coefficient of x(i) in (K x)(i+o)
        dh = -double(cb[(size_t)(2 + 2 * d) * P + q]) * rq[(-o + 4) * 2] -
             double(cb[(size_t)(3 + 2 * d) * P + q]) * rq[(-o + 4) * 2 + 1];
        dh *= double(cb[P + q]);
      }
      diag -= (double(row[kTabKT + (o + 4) * 2]) * cb[(size_t)(2 + 2 * d) * P + q] +
               double(row[kTabKT + (o + 4) * 2 + 1]) * cb[(size_t)(3 + 2 * d) * P + q]) * dh;
    }
  }
  dinv[(size_t)v * P + p] = float(1.0 / diag);
}

// ---------------------------------------------------------------------------------
// Vectorised variants: 4 consecutive points along the contiguous (last) axis per thread
// (requires n_last % 4 == 0).  Non-last axes: one float4 load per stencil offset serves
// the 4 points; last axis: a register window loaded with aligned float4s.  Interior rows
// of the tables come from the constant bank (G.irow); edge rows from the global table.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
// per-point coefficients cf: fp32, or bf16 for the V-cycle's level-0 applies
// (mpde_options.cf_bf16; 4 consecutive points = one 8-byte load, widened by shifts)
__device__ __forceinline__ float4 ldc4(const float* p) { return ld4(p); }
__device__ __forceinline__ float4 ldc4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}
__device__ __forceinline__ void st4(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
template <typename T>
__device__ __forceinline__ void ldT4(const T* p, T* v) {
  if (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}
template <typename T>
__device__ __forceinline__ void stT4(T* p, const T* v) {
  if (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(float(v[0]), float(v[1]), float(v[2]), float(v[3]));
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(double(v[0]), double(v[1]));
    *reinterpret_cast<double2*>(p + 2) = make_double2(double(v[2]), double(v[3]));
  }
}
#define F4(a, j) (j == 0 ? a.x : (j == 1 ? a.y : (j == 2 ? a.z : a.w)))
// Quad updates a[0..3] (+)= ... either as four scalar ops or on the packed fp32x2 pipe
// (FFMA2 / FMUL2 on sm_100a: half the issue slots; each lane is the same single-rounding
// op, so both forms give bit-identical results).  Measured (profiles/r2_ffma2_ab.txt): pass 1
// gains (0.420 -> 0.428 of the HBM peak), pass 2 does not (74.3 -> 75.0 us per level-0
// launch: it waits on L1 wavefronts, not on issue), so pass 2 keeps the scalar form.
// acc[0..3] += c * v
template <bool PACKED>
__device__ __forceinline__ void quad_axpy(float* acc, float c, const float4& v) {
  if constexpr (PACKED) {
    const float2 cc = make_float2(c, c);
    const float2 lo = __ffma2_rn(cc, make_float2(v.x, v.y), make_float2(acc[0], acc[1]));
    const float2 hi = __ffma2_rn(cc, make_float2(v.z, v.w), make_float2(acc[2], acc[3]));
    acc[0] = lo.x; acc[1] = lo.y; acc[2] = hi.x; acc[3] = hi.y;
  } else {
    acc[0] += c * v.x; acc[1] += c * v.y; acc[2] += c * v.z; acc[3] += c * v.w;
  }
}
// acc[0..3] -= (a * va + b * vb) * hv   (the K^T (u~ h) terms)
__device__ __forceinline__ void quad_kt(float* acc, float a, float b, const float4& va, const float4& vb,
                                        const float4& hv) {
  acc[0] -= (a * va.x + b * vb.x) * hv.x; acc[1] -= (a * va.y + b * vb.y) * hv.y;
  acc[2] -= (a * va.z + b * vb.z) * hv.z; acc[3] -= (a * va.w + b * vb.w) * hv.w;
}
// NV 16-byte loads of a table-row segment (rows and segments are 16-byte aligned): one
// vector load per 4 coefficients instead of one scalar load each (L1 wavefronts)
template <int NV>
__device__ __forceinline__ void ldv(const float* p, float* v) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p) + k);
    v[4 * k] = a.x;
    v[4 * k + 1] = a.y;
    v[4 * k + 2] = a.z;
    v[4 * k + 3] = a.w;
  }
}

// Warp-specialised quad mapping along the contiguous axis (NY4 = n_last / 4 a power of two
// <= kThreads): a CTA covers R = kThreads / NY4 whole rows; its first R * NI threads take the
// interior quads 2 .. NY4-3 (ymode 1: constant-bank interior stencils, no per-point branch)
// and the remaining threads the (up to 4) edge quads (ymode 2: table rows for every point),
// so the edge handling never diverges inside a warp.  ymode 0 = per-point test (no remap).
__device__ __forceinline__ void remap_quad(int NY4, int& row, int& q, int& ymode) {
  const int R = kThreads / NY4;
  const int NE = NY4 < 4 ? NY4 : 4, NI = NY4 - NE;
  int k = threadIdx.x;
  if (k < R * NI) {
    row = k / NI;
    q = 2 + k % NI;
    ymode = 1;
  } else {
    k -= R * NI;
    row = k / NE;
    const int e = k % NE;
    q = (NE == 4 && e >= 2) ? NY4 - 4 + e : e;
    ymode = 2;
  }
  row += blockIdx.x * R;
}
// points handled by this CTA (profiling counters)
__device__ __forceinline__ int block_points(int remap, int P, int nlast, int p0_first) {
  if (remap) {
    const int R = kThreads / (nlast >> 2), rows = P / nlast;
    return max(0, min(R, rows - (int)blockIdx.x * R)) * nlast;
  }
  return min(4 * (int)blockDim.x, P - p0_first);
}

template <int D, typename T, typename CF>
__device__ __forceinline__ void schur_h4(const Geo& G, const CF* __restrict__ cb,
                                         const float* __restrict__ xb, int p0, const int* idx,
                                         T* g, int ymode) {
  const int P = G.P;
  {
    const float4 x0 = ld4(xb + p0), c0 = ldc4(cb + p0);
#pragma unroll
    for (int j = 0; j < 4; ++j) g[j] = T(F4(c0, j)) * T(F4(x0, j));
  }
#pragma unroll
  for (int d = 0; d < D - 1; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    T k1[4] = {0, 0, 0, 0}, k2[4] = {0, 0, 0, 0};
    if (i >= 2 && i <= n - 3) {
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const float4 xv = ld4(xb + p0 + o * s);
        if constexpr (std::is_same<T, float>::value) {
          quad_axpy<true>(k1, G.irow[d][(o + 2) * 2], xv);
          quad_axpy<true>(k2, G.irow[d][(o + 2) * 2 + 1], xv);
        } else {
          const T a = G.irow[d][(o + 2) * 2], b = G.irow[d][(o + 2) * 2 + 1];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            k1[j] += a * T(F4(xv, j));
            k2[j] += b * T(F4(xv, j));
          }
        }
      }
    } else {  // edge rows: unrolled, clamped addresses, zero coefficients out of range
      float kf[20];
      ldv<5>(tab_row(G, d, i) + kTabKf, kf);
      const int olo = -i, ohi = n - 1 - i;
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const int oc = o < olo ? olo : (o > ohi ? ohi : o);
        const float4 xv = ld4(xb + p0 + oc * s);
        const T a = kf[(o + 4) * 2], b = kf[(o + 4) * 2 + 1];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          k1[j] += a * T(F4(xv, j));
          k2[j] += b * T(F4(xv, j));
        }
      }
    }
    const float4 ua = ldc4(cb + (size_t)(2 + 2 * d) * P + p0), ub = ldc4(cb + (size_t)(3 + 2 * d) * P + p0);
#pragma unroll
    for (int j = 0; j < 4; ++j) g[j] -= T(F4(ua, j)) * k1[j] + T(F4(ub, j)) * k2[j];
  }
  {  // last axis: window x(i0-4 .. i0+7)
    constexpr int d = D - 1;
    const int n = G.n[d], i0 = idx[d];
    float w[12];
    const float4 wl = i0 >= 4 ? ld4(xb + p0 - 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 wm = ld4(xb + p0);
    const float4 wr = i0 + 4 < n ? ld4(xb + p0 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[j] = F4(wl, j);
      w[4 + j] = F4(wm, j);
      w[8 + j] = F4(wr, j);
    }
    const float4 ua = ldc4(cb + (size_t)(2 + 2 * d) * P + p0), ub = ldc4(cb + (size_t)(3 + 2 * d) * P + p0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      T k1 = 0, k2 = 0;
      if (ymode == 1 || (ymode == 0 && i >= 2 && i <= n - 3)) {
#pragma unroll
        for (int o = -2; o <= 2; ++o) {
          k1 += T(G.irow[d][(o + 2) * 2]) * T(w[4 + j + o]);
          k2 += T(G.irow[d][(o + 2) * 2 + 1]) * T(w[4 + j + o]);
        }
      } else {
        float kf[20];
        ldv<5>(tab_row(G, d, i) + kTabKf, kf);
#pragma unroll
        for (int o = -4; o <= 4; ++o) {  // out-of-range taps have zero coefficients
          if (4 + j + o < 0 || 4 + j + o > 11) continue;
          k1 += T(kf[(o + 4) * 2]) * T(w[4 + j + o]);
          k2 += T(kf[(o + 4) * 2 + 1]) * T(w[4 + j + o]);
        }
      }
      g[j] -= T(F4(ua, j)) * k1 + T(F4(ub, j)) * k2;
    }
  }
  {
    const float4 c1 = ldc4(cb + P + p0);
#pragma unroll
    for (int j = 0; j < 4; ++j) g[j] *= T(F4(c1, j));
  }
}

template <int D, typename T, typename CF>
__device__ __forceinline__ void schur_s4(const Geo& G, const CF* __restrict__ cb,
                                         const float* __restrict__ xb, const T* __restrict__ hb,
                                         int p0, const int* idx, T* acc, int ymode) {
  const int P = G.P;
  {
    T h0[4];
    ldT4<T>(hb + p0, h0);
    const float4 c0 = ldc4(cb + p0);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = T(F4(c0, j)) * h0[j];
    // boundary rows: faces of the non-last axes cover all 4 points; last-axis faces per point
    bool face = false;
#pragma unroll
    for (int d = 0; d < D - 1; ++d) face |= dir_face(G, d, idx[d]);
    const float4 x0 = ld4(xb + p0);
    const T wb2 = T(G.wb) * T(G.wb);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = idx[D - 1] + j;
      if (face || dir_face(G, D - 1, i)) acc[j] += wb2 * T(F4(x0, j));
    }
  }
#pragma unroll
  for (int d = 0; d < D - 1; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
    const CF* u1 = cb + (size_t)(2 + 2 * d) * P;
    const CF* u2 = cb + (size_t)(3 + 2 * d) * P;
    if (i >= 7 && i <= n - 8) {
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const float4 xv = ld4(xb + p0 + o * s);
        const T a = G.irow[d][20 + o + 4];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += a * T(F4(xv, j));
      }
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const int q = p0 + o * s;
        const float4 va = ldc4(u1 + q), vb = ldc4(u2 + q);
        T hv[4];
        ldT4<T>(hb + q, hv);
        const T a = G.irow[d][10 + (o + 2) * 2], b = G.irow[d][10 + (o + 2) * 2 + 1];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] -= (a * T(F4(va, j)) + b * T(F4(vb, j))) * hv[j];
      }
    } else {
      // edge classes: fully unrolled, addresses clamped into the line (the table holds
      // zero coefficients for out-of-range taps) so that every load issues at once
      const float* row = tab_row(G, d, i);
      float p0r[12], ktr[20];
      ldv<3>(row + kTabP0, p0r);
      ldv<5>(row + kTabKT, ktr);
      const int olo = -i, ohi = n - 1 - i;
#pragma unroll
      for (int o = -5; o <= 5; ++o) {
        const int oc = o < olo ? olo : (o > ohi ? ohi : o);
        const float4 xv = ld4(xb + p0 + oc * s);
        const T a = p0r[o + 5];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += a * T(F4(xv, j));
      }
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const int oc = o < olo ? olo : (o > ohi ? ohi : o);
        const int q = p0 + oc * s;
        const float4 va = ldc4(u1 + q), vb = ldc4(u2 + q);
        T hv[4];
        ldT4<T>(hb + q, hv);
        const T a = ktr[(o + 4) * 2], b = ktr[(o + 4) * 2 + 1];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] -= (a * T(F4(va, j)) + b * T(F4(vb, j))) * hv[j];
      }
    }
  }
  {  // last axis: x window (i0-8 .. i0+11), u1/u2/h windows (i0-4 .. i0+7)
    constexpr int d = D - 1;
    const int n = G.n[d], i0 = idx[d];
    const CF* u1 = cb + (size_t)(2 + 2 * d) * P;
    const CF* u2 = cb + (size_t)(3 + 2 * d) * P;
    float xw[20];
    float aw[12], bw[12];
    T hw[12];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int off = -8 + 4 * k;
      const bool ok = (i0 + off >= 0) && (i0 + off < n);
      const float4 v = ok ? ld4(xb + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 4; ++j) xw[4 * k + j] = F4(v, j);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int off = -4 + 4 * k;
      const bool ok = (i0 + off >= 0) && (i0 + off < n);
      const float4 va = ok ? ldc4(u1 + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 vb = ok ? ldc4(u2 + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
      T hv[4] = {0, 0, 0, 0};
      if (ok) ldT4<T>(hb + p0 + off, hv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        aw[4 * k + j] = F4(va, j);
        bw[4 * k + j] = F4(vb, j);
        hw[4 * k + j] = hv[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      if (ymode == 1 || (ymode == 0 && i >= 7 && i <= n - 8)) {
#pragma unroll
        for (int o = -4; o <= 4; ++o) acc[j] += T(G.irow[d][20 + o + 4]) * T(xw[8 + j + o]);
#pragma unroll
        for (int o = -2; o <= 2; ++o)
          acc[j] -= (T(G.irow[d][10 + (o + 2) * 2]) * T(aw[4 + j + o]) +
                     T(G.irow[d][10 + (o + 2) * 2 + 1]) * T(bw[4 + j + o])) * hw[4 + j + o];
      } else {
        const float* row = tab_row(G, d, i);
        float p0r[12], ktr[20];
        ldv<3>(row + kTabP0, p0r);
        ldv<5>(row + kTabKT, ktr);
#pragma unroll
        for (int o = -5; o <= 5; ++o) acc[j] += T(p0r[o + 5]) * T(xw[8 + j + o]);
#pragma unroll
        for (int o = -4; o <= 4; ++o) {
          if (4 + j + o < 0 || 4 + j + o > 11) continue;
          acc[j] -= (T(ktr[(o + 4) * 2]) * T(aw[4 + j + o]) +
                     T(ktr[(o + 4) * 2 + 1]) * T(bw[4 + j + o])) * hw[4 + j + o];
        }
      }
    }
  }
}

// Small-level form of schur_h4 (latency bound: ~2 warps per SM): every x tap of the t / x
// stencils (9, clamped) and every coefficient is loaded before any edge-class branch, so
// the thread pays one memory round trip instead of one per axis.  Interior rows use taps
// -2..2 with irow, edge rows the table (-4..4), in the same order as schur_h4: bit-identical.
template <int D, typename T, typename CF>
__device__ __forceinline__ void schur_h4_lat(const Geo& G, const CF* __restrict__ cb,
                                             const float* __restrict__ xb, int p0, const int* idx,
                                             T* g) {
  const int P = G.P;
  float4 xt[D - 1][9];
#pragma unroll
  for (int d = 0; d < D - 1; ++d) {
    const int n = G.n[d], s = G.stride[d], i = idx[d];
#pragma unroll
    for (int o = -4; o <= 4; ++o) {
      const int oc = min(max(i + o, 0), n - 1) - i;
      xt[d][o + 4] = ld4(xb + p0 + oc * s);
    }
  }
  float4 ua[D], ub[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    ua[d] = ldc4(cb + (size_t)(2 + 2 * d) * P + p0);
    ub[d] = ldc4(cb + (size_t)(3 + 2 * d) * P + p0);
  }
  constexpr int dl = D - 1;
  const int nl = G.n[dl], i0 = idx[dl];
  const float4 wl = i0 >= 4 ? ld4(xb + p0 - 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 wm = ld4(xb + p0);
  const float4 wr = i0 + 4 < nl ? ld4(xb + p0 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 c0 = ldc4(cb + p0), c1 = ldc4(cb + P + p0);
#pragma unroll
  for (int j = 0; j < 4; ++j) g[j] = T(F4(c0, j)) * T(F4(wm, j));
#pragma unroll
  for (int d = 0; d < D - 1; ++d) {
    const int n = G.n[d], i = idx[d];
    T k1[4] = {0, 0, 0, 0}, k2[4] = {0, 0, 0, 0};
    if (i >= 2 && i <= n - 3) {
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const T a = G.irow[d][(o + 2) * 2], b = G.irow[d][(o + 2) * 2 + 1];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          k1[j] += a * T(F4(xt[d][o + 4], j));
          k2[j] += b * T(F4(xt[d][o + 4], j));
        }
      }
    } else {
      float kf[20];
      ldv<5>(tab_row(G, d, i) + kTabKf, kf);
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const T a = kf[(o + 4) * 2], b = kf[(o + 4) * 2 + 1];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          k1[j] += a * T(F4(xt[d][o + 4], j));
          k2[j] += b * T(F4(xt[d][o + 4], j));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) g[j] -= T(F4(ua[d], j)) * k1[j] + T(F4(ub[d], j)) * k2[j];
  }
  {
    float w[12];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[j] = F4(wl, j);
      w[4 + j] = F4(wm, j);
      w[8 + j] = F4(wr, j);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      T k1 = 0, k2 = 0;
      if (i >= 2 && i <= nl - 3) {
#pragma unroll
        for (int o = -2; o <= 2; ++o) {
          k1 += T(G.irow[dl][(o + 2) * 2]) * T(w[4 + j + o]);
          k2 += T(G.irow[dl][(o + 2) * 2 + 1]) * T(w[4 + j + o]);
        }
      } else {
        float kf[20];
        ldv<5>(tab_row(G, dl, i) + kTabKf, kf);
#pragma unroll
        for (int o = -4; o <= 4; ++o) {
          if (4 + j + o < 0 || 4 + j + o > 11) continue;
          k1 += T(kf[(o + 4) * 2]) * T(w[4 + j + o]);
          k2 += T(kf[(o + 4) * 2 + 1]) * T(w[4 + j + o]);
        }
      }
      g[j] -= T(F4(ua[dl], j)) * k1 + T(F4(ub[dl], j)) * k2;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) g[j] *= T(F4(c1, j));
}

template <int D, typename T, typename CF>
__global__ void __launch_bounds__(kSmallThreads) k_schur_h_v4_lat(Geo G, const CF* __restrict__ cf, int crep,
                                                                  const float* __restrict__ x,
                                                                  T* __restrict__ hout, const int* act,
                                                                  unsigned long long* pts) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int nl = G.n[D - 1];
  if (pts && threadIdx.x == 0)
    atomicAdd(pts, (unsigned long long)block_points(0, P, nl, blockIdx.x * blockDim.x * 4));
  const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (p0 >= P) return;
  int idx[D];
  unravel<D>(G, p0, idx);
  T g[4];
  schur_h4_lat<D, T, CF>(G, cf + (size_t)pde * NC * P, x + (size_t)v * P, p0, idx, g);
  stT4<T>(hout + (size_t)v * P + p0, g);
}

template <int D, typename T, typename CF = float>
__global__ void __launch_bounds__(kThreads, 5) k_schur_h_v4(Geo G, const CF* __restrict__ cf, int crep,
                                                        const float* __restrict__ x,
                                                        T* __restrict__ hout, const int* act,
                                                        unsigned long long* pts, int remap) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int nl = G.n[D - 1];
  if (pts && threadIdx.x == 0)
    atomicAdd(pts, (unsigned long long)block_points(remap, P, nl, blockIdx.x * blockDim.x * 4));
  int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4, ymode = 0;
  if (remap) {
    int row, q;
    remap_quad(nl >> 2, row, q, ymode);
    p0 = row * nl + 4 * q;
  }
  if (p0 >= P) return;
  int idx[D];
  unravel<D>(G, p0, idx);
  T g[4];
  schur_h4<D, T, CF>(G, cf + (size_t)pde * NC * P, x + (size_t)v * P, p0, idx, g, ymode);
  stT4<T>(hout + (size_t)v * P + p0, g);
}

template <int D, int EPI, typename T, typename CF = float>
__global__ void __launch_bounds__(kThreads) k_schur_s_v4(Geo G, const CF* __restrict__ cf, int crep,
                                                        const float* __restrict__ x,
                                                        const T* __restrict__ hb, EpiArgs A,
                                                        const int* act, int remap) {
  MPDE_PDL_ENTRY();
  constexpr int NC = 2 + 2 * D;
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int nl = G.n[D - 1];
  int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4, ymode = 0;
  if (remap) {
    int row, q;
    remap_quad(nl >> 2, row, q, ymode);
    p0 = row * nl + 4 * q;
  }
  double dot = 0.0;
  if (p0 < P) {
    int idx[D];
    unravel<D>(G, p0, idx);
    const size_t o = (size_t)v * P + p0;
    T acc[4];
    schur_s4<D, T, CF>(G, cf + (size_t)pde * NC * P, x + (size_t)v * P, hb + (size_t)v * P, p0, idx,
                   acc, ymode);
    float q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = float(acc[j]);
    if (EPI == EPI_STORE) {
      st4(A.y + o, q);
    } else if (EPI == EPI_DOT) {
      st4(A.y + o, q);
      const float4 xv = ld4(x + o);
#pragma unroll
      for (int j = 0; j < 4; ++j) dot += double(F4(xv, j)) * q[j];
    } else if (EPI == EPI_POWER) {
      const float4 xv = ld4(x + o), dv = ld4(A.dinv + o);
      float y[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        y[j] = F4(dv, j) * q[j];
        dot += double(F4(xv, j)) * q[j];
      }
      st4(A.y + o, y);
    } else if (EPI == EPI_RESID) {
      const float4 rv = ld4(A.res + o);
      float r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = F4(rv, j) - q[j];
      st4(A.res + o, r);
    } else if (EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST) {
      const float al = A.coef[pde * A.coef_stride + 2 * A.step];
      const float be = A.coef[pde * A.coef_stride + 2 * A.step + 1];
      const float4 rv = ld4(A.res + o), xv = ld4(x + o), dv = ld4(A.dinv + o), ev = ld4(A.e + o);
      float r[4], dn[4], e[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        r[j] = F4(rv, j) - q[j];
        dn[j] = al * F4(xv, j) + be * F4(dv, j) * r[j];
        e[j] = F4(ev, j) + dn[j];
      }
      st4(A.e + o, e);
      if (EPI == EPI_SMOOTH) {
        st4(A.res + o, r);
        st4(A.d_out + o, dn);
      }
      if (A.rdot) {
        const float4 pv = ld4(A.rdot + o);
#pragma unroll
        for (int j = 0; j < 4; ++j) dot += double(F4(pv, j)) * e[j];
      }
    } else if (EPI == EPI_POST0) {
      const float be = A.coef[pde * A.coef_stride + 1];
      const float4 rv = ld4(A.res + o), xv = ld4(x + o), dv = ld4(A.dinv + o), ev = ld4(A.e + o);
      float r[4], dn[4], e[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        r[j] = F4(rv, j) - q[j];
        dn[j] = be * F4(dv, j) * r[j];
        e[j] = F4(ev, j) + F4(xv, j) + dn[j];
      }
      st4(A.e + o, e);
      st4(A.res + o, r);
      st4(A.d_out + o, dn);
      if (A.rdot) {
        const float4 pv = ld4(A.rdot + o);
#pragma unroll
        for (int j = 0; j < 4; ++j) dot += double(F4(pv, j)) * e[j];
      }
    }
  }
  if (A.pts && threadIdx.x == 0)
    atomicAdd(A.pts + EPI,
              (unsigned long long)block_points(remap, P, nl, blockIdx.x * blockDim.x * 4));
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (threadIdx.x == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------------
// 3D pass 2 with 2x2 register blocking in (t, x): a thread computes the four y-quads at
// (t0+a, x0+b), a, b in {0,1}.  Every t- (x-) neighbour load feeds both t (x) outputs,
// which cuts the L1 gathers per quad by ~30% (the v4 kernel is L1-wavefront bound).
// ---------------------------------------------------------------------------------
// compile-time (x, y) extents (0 = read from G): every stencil offset becomes an immediate
template <int NX, int NY>
__device__ __forceinline__ int dim_n(const Geo& G, int ax) {
  return ax == 0 ? G.n[0] : ax == 1 ? (NX ? NX : G.n[1]) : (NY ? NY : G.n[2]);
}
template <int NX, int NY>
__device__ __forceinline__ int dim_s(const Geo& G, int ax) {
  return ax == 0 ? ((NX && NY) ? NX * NY : G.stride[0]) : ax == 1 ? (NY ? NY : G.stride[1]) : 1;
}

template <int AX, int NX, int NY, typename CF>  // accumulate the AX-axis (0 = t, 1 = x) terms of a 2-output pencil
__device__ __forceinline__ void pencil2(const Geo& G, const CF* __restrict__ cb,
                                        const float* __restrict__ xb, const float* __restrict__ hb,
                                        int pbase, int i0, bool ok1, float* acc0, float* acc1) {
  // pbase: offset of output 0 (index i0 along AX); output 1 is at pbase + s (index i0+1)
  const int P = G.P, n = dim_n<NX, NY>(G, AX), s = dim_s<NX, NY>(G, AX);
  const CF* u1 = cb + (size_t)(2 + 2 * AX) * P;
  const CF* u2 = cb + (size_t)(3 + 2 * AX) * P;
  if (i0 >= 7 && i0 + 1 <= n - 8) {
#pragma unroll
    for (int u = -4; u <= 5; ++u) {
      const float4 xv = ld4(xb + pbase + u * s);
      if (u <= 4) quad_axpy<false>(acc0, G.irow[AX][20 + u + 4], xv);
      if (u >= -3) quad_axpy<false>(acc1, G.irow[AX][20 + u - 1 + 4], xv);
    }
#pragma unroll
    for (int u = -2; u <= 3; ++u) {
      const int q = pbase + u * s;
      const float4 va = ldc4(u1 + q), vb = ldc4(u2 + q), hv = ld4(hb + q);
      if (u <= 2) quad_kt(acc0, G.irow[AX][10 + (u + 2) * 2], G.irow[AX][10 + (u + 2) * 2 + 1], va, vb, hv);
      if (u >= -1) quad_kt(acc1, G.irow[AX][10 + (u + 1) * 2], G.irow[AX][10 + (u + 1) * 2 + 1], va, vb, hv);
    }
    return;
  }
  // edge classes: table rows per output, clamped addresses, zero coefficients out of range
  const float* r0 = tab_row(G, AX, i0);
  const float* r1 = tab_row(G, AX, ok1 ? i0 + 1 : i0);
  const float m1 = ok1 ? 1.f : 0.f;
  float p0a[12], p0b[12];
  ldv<3>(r0 + kTabP0, p0a);
  ldv<3>(r1 + kTabP0, p0b);
#pragma unroll
  for (int u = -5; u <= 6; ++u) {
    const int ic = min(max(i0 + u, 0), n - 1);
    const float4 xv = ld4(xb + pbase + (ic - i0) * s);
    if (u <= 5) quad_axpy<false>(acc0, p0a[u + 5], xv);
    if (u >= -4) quad_axpy<false>(acc1, m1 * p0b[u - 1 + 5], xv);
  }
  float kta[20], ktb[20];
  ldv<5>(r0 + kTabKT, kta);
  ldv<5>(r1 + kTabKT, ktb);
#pragma unroll
  for (int u = -4; u <= 5; ++u) {
    const int ic = min(max(i0 + u, 0), n - 1);
    const int q = pbase + (ic - i0) * s;
    const float4 va = ldc4(u1 + q), vb = ldc4(u2 + q), hv = ld4(hb + q);
    if (u <= 4) quad_kt(acc0, kta[(u + 4) * 2], kta[(u + 4) * 2 + 1], va, vb, hv);
    if (u >= -3) quad_kt(acc1, m1 * ktb[(u + 3) * 2], m1 * ktb[(u + 3) * 2 + 1], va, vb, hv);
  }
}

// one-output version of pencil2 (single quad, AX-axis terms)
template <int AX, int NX, int NY, typename CF>
__device__ __forceinline__ void pencil1(const Geo& G, const CF* __restrict__ cb,
                                        const float* __restrict__ xb, const float* __restrict__ hb,
                                        int p0, int i, float* acc) {
  const int P = G.P, n = dim_n<NX, NY>(G, AX), s = dim_s<NX, NY>(G, AX);
  const CF* u1 = cb + (size_t)(2 + 2 * AX) * P;
  const CF* u2 = cb + (size_t)(3 + 2 * AX) * P;
  if (i >= 7 && i <= n - 8) {
#pragma unroll
    for (int o = -4; o <= 4; ++o) {
      const float4 xv = ld4(xb + p0 + o * s);
      quad_axpy<false>(acc, G.irow[AX][20 + o + 4], xv);
    }
#pragma unroll
    for (int o = -2; o <= 2; ++o) {
      const int q = p0 + o * s;
      const float4 va = ldc4(u1 + q), vb = ldc4(u2 + q), hv = ld4(hb + q);
      quad_kt(acc, G.irow[AX][10 + (o + 2) * 2], G.irow[AX][10 + (o + 2) * 2 + 1], va, vb, hv);
    }
    return;
  }
  const float* row = tab_row(G, AX, i);
  float p0r[12], ktr[20];
  ldv<3>(row + kTabP0, p0r);
  ldv<5>(row + kTabKT, ktr);
  const int olo = -i, ohi = n - 1 - i;
#pragma unroll
  for (int o = -5; o <= 5; ++o) {
    const int oc = o < olo ? olo : (o > ohi ? ohi : o);
    const float4 xv = ld4(xb + p0 + oc * s);
    quad_axpy<false>(acc, p0r[o + 5], xv);
  }
#pragma unroll
  for (int o = -4; o <= 4; ++o) {
    const int oc = o < olo ? olo : (o > ohi ? ohi : o);
    const int q = p0 + oc * s;
    const float4 va = ldc4(u1 + q), vb = ldc4(u2 + q), hv = ld4(hb + q);
    quad_kt(acc, ktr[(o + 4) * 2], ktr[(o + 4) * 2 + 1], va, vb, hv);
  }
}

// y-axis (contiguous) terms + own terms of one quad, as in schur_s4
template <int NX, int NY, typename CF>
__device__ __forceinline__ void quad_y_own(const Geo& G, const CF* __restrict__ cb,
                                           const float* __restrict__ xb,
                                           const float* __restrict__ hb, int p0, int t, int xr,
                                           float* acc, int ymode) {
  const int P = G.P, n = dim_n<NX, NY>(G, 2), i0 = p0 % n;
  {
    const float4 h0 = ld4(hb + p0), c0 = ldc4(cb + p0), x0 = ld4(xb + p0);
    const bool face = dir_face(G, 0, t) | dir_face(G, 1, xr);
    const float wb2 = G.wb * G.wb;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[j] += F4(c0, j) * F4(h0, j);
      if (face || dir_face(G, 2, i0 + j)) acc[j] += wb2 * F4(x0, j);
    }
  }
  const CF* u1 = cb + (size_t)6 * P;
  const CF* u2 = cb + (size_t)7 * P;
  // x window first (P0 taps), then the u~ h windows (K^T taps): fewer values live at once
  // (pass-2 spill 40 -> 8 B, 71.3 -> 69.1 us per level-0 launch; profiles/r2_b22_regs_ab.txt)
  {
    float xw[20];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int off = -8 + 4 * k;
      const bool ok = (i0 + off >= 0) && (i0 + off < n);
      const float4 vv = ok ? ld4(xb + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 4; ++j) xw[4 * k + j] = F4(vv, j);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      if (ymode == 1 || (ymode == 0 && i >= 7 && i <= n - 8)) {
#pragma unroll
        for (int o = -4; o <= 4; ++o) acc[j] += G.irow[2][20 + o + 4] * xw[8 + j + o];
      } else {
        float p0r[12];
        ldv<3>(tab_row(G, 2, i) + kTabP0, p0r);
#pragma unroll
        for (int o = -5; o <= 5; ++o) acc[j] += p0r[o + 5] * xw[8 + j + o];
      }
    }
  }
  {
    float aw[12], bw[12], hw[12];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int off = -4 + 4 * k;
      const bool ok = (i0 + off >= 0) && (i0 + off < n);
      const float4 va = ok ? ldc4(u1 + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 vb = ok ? ldc4(u2 + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 hv = ok ? ld4(hb + p0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        aw[4 * k + j] = F4(va, j);
        bw[4 * k + j] = F4(vb, j);
        hw[4 * k + j] = F4(hv, j);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j;
      if (ymode == 1 || (ymode == 0 && i >= 7 && i <= n - 8)) {
#pragma unroll
        for (int o = -2; o <= 2; ++o)
          acc[j] -= (G.irow[2][10 + (o + 2) * 2] * aw[4 + j + o] +
                     G.irow[2][10 + (o + 2) * 2 + 1] * bw[4 + j + o]) * hw[4 + j + o];
      } else {
        float ktr[20];
        ldv<5>(tab_row(G, 2, i) + kTabKT, ktr);
#pragma unroll
        for (int o = -4; o <= 4; ++o) {
          if (4 + j + o < 0 || 4 + j + o > 11) continue;
          acc[j] -= (ktr[(o + 4) * 2] * aw[4 + j + o] +
                     ktr[(o + 4) * 2 + 1] * bw[4 + j + o]) * hw[4 + j + o];
        }
      }
    }
  }
}

template <int EPI>
__device__ __forceinline__ double quad_epilogue(const EpiArgs& A, int pde, size_t o,
                                                const float* __restrict__ x, const float* q) {
  double dot = 0.0;
  if (EPI == EPI_STORE) {
    st4(A.y + o, q);
  } else if (EPI == EPI_DOT) {
    st4(A.y + o, q);
    const float4 xv = ld4(x + o);
#pragma unroll
    for (int j = 0; j < 4; ++j) dot += double(F4(xv, j)) * q[j];
  } else if (EPI == EPI_POWER) {
    const float4 xv = ld4(x + o), dv = ld4(A.dinv + o);
    float y[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      y[j] = F4(dv, j) * q[j];
      dot += double(F4(xv, j)) * q[j];
    }
    st4(A.y + o, y);
  } else if (EPI == EPI_RESID) {
    const float4 rv = ld4(A.res + o);
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = F4(rv, j) - q[j];
    st4(A.res + o, r);
  } else if (EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST) {
    const float al = A.coef[pde * A.coef_stride + 2 * A.step];
    const float be = A.coef[pde * A.coef_stride + 2 * A.step + 1];
    const float4 rv = ld4(A.res + o), xv = ld4(x + o), dv = ld4(A.dinv + o), ev = ld4(A.e + o);
    float r[4], dn[4], e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      r[j] = F4(rv, j) - q[j];
      dn[j] = al * F4(xv, j) + be * F4(dv, j) * r[j];
      e[j] = F4(ev, j) + dn[j];
    }
    st4(A.e + o, e);
    if (EPI == EPI_SMOOTH) {
      st4(A.res + o, r);
      st4(A.d_out + o, dn);
    }
    if (A.rdot) {
      const float4 pv = ld4(A.rdot + o);
#pragma unroll
      for (int j = 0; j < 4; ++j) dot += double(F4(pv, j)) * e[j];
    }
  } else if (EPI == EPI_POST0) {
    const float be = A.coef[pde * A.coef_stride + 1];
    const float4 rv = ld4(A.res + o), xv = ld4(x + o), dv = ld4(A.dinv + o), ev = ld4(A.e + o);
    float r[4], dn[4], e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      r[j] = F4(rv, j) - q[j];
      dn[j] = be * F4(dv, j) * r[j];
      e[j] = F4(ev, j) + F4(xv, j) + dn[j];
    }
    st4(A.e + o, e);
    st4(A.res + o, r);
    st4(A.d_out + o, dn);
    if (A.rdot) {
      const float4 pv = ld4(A.rdot + o);
#pragma unroll
      for (int j = 0; j < 4; ++j) dot += double(F4(pv, j)) * e[j];
    }
  }
  return dot;
}

template <int EPI, int BX, int NX, int NY, int YP, typename CF = float>
__global__ void __launch_bounds__(kThreads, MPDE_B22_MINB) k_schur_s_b22(Geo G, const CF* __restrict__ cf, int crep,
                                                         const float* __restrict__ x,
                                                         const float* __restrict__ hb, EpiArgs A,
                                                         const int* act, int remap) {
  MPDE_PDL_ENTRY();
  // BX = 1: 2x2 blocking in (t, x); BX = 0: 2x1 blocking in t only (fewer registers)
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int nt = G.n[0], nx = dim_n<NX, NY>(G, 1), ny = dim_n<NX, NY>(G, 2);
  const int NY4 = ny >> 2, NXB = BX ? (nx + 1) >> 1 : nx, NT2 = (nt + 1) >> 1;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int yq = tid % NY4, r2 = tid / NY4, ymode = 0;
  if (remap) remap_quad(NY4, r2, yq, ymode);
  int xp = r2 % NXB, tp = r2 / NXB;
  if (remap > 1) {  // CTA = TPB t-pairs x XPB x-rows (t-neighbour reuse in L1), TPB = remap
    const int R = kThreads / NY4, TPB = remap, XPB = R / TPB, nxb = (NXB + XPB - 1) / XPB;
    const int lr = r2 - (int)blockIdx.x * R, bx = blockIdx.x % nxb, bt = blockIdx.x / nxb;
    xp = bx * XPB + lr % XPB;
    tp = bt * TPB + lr / XPB;
    if (xp >= NXB) tp = NT2;  // outside: skip
  }
  double dot = 0.0;
  int nq = 0;
  if (tp < NT2) {
    const CF* cb = cf + (size_t)pde * 8 * P;
    const float* xb = x + (size_t)v * P;
    const float* hv = hb + (size_t)v * P;
    const int t0 = 2 * tp, x0 = BX ? 2 * xp : xp;
    const bool okt = t0 + 1 < nt, okx = BX && (x0 + 1 < nx);
    const int st = dim_s<NX, NY>(G, 0), sxs = dim_s<NX, NY>(G, 1);
    const int pb = t0 * st + x0 * sxs + 4 * yq;
    float acc[2][BX + 1][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < BX + 1; ++b)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[a][b][j] = 0.f;
    // t pencils (columns x0 [, x0+1]) and x terms (planes t0, t0+1)
    pencil2<0, NX, NY>(G, cb, xb, hv, pb, t0, okt, acc[0][0], acc[1][0]);
    if (BX) {
      if (okx) pencil2<0, NX, NY>(G, cb, xb, hv, pb + sxs, t0, okt, acc[0][BX], acc[1][BX]);
      pencil2<1, NX, NY>(G, cb, xb, hv, pb, x0, okx, acc[0][0], acc[0][BX]);
      if (okt) pencil2<1, NX, NY>(G, cb, xb, hv, pb + st, x0, okx, acc[1][0], acc[1][BX]);
    } else {
      pencil1<1, NX, NY>(G, cb, xb, hv, pb, x0, acc[0][0]);
      if (okt) pencil1<1, NX, NY>(G, cb, xb, hv, pb + st, x0, acc[1][0]);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < BX + 1; ++b) {
        if ((a && !okt) || (b && !okx)) continue;
        const int p0 = pb + a * st + b * sxs;
        if (YP) {  // y-axis and own terms from pass 1 (k_schur_hy)
          const float4 r = ld4(hv + (size_t)gridDim.y * P + p0);
          acc[a][b][0] += r.x;
          acc[a][b][1] += r.y;
          acc[a][b][2] += r.z;
          acc[a][b][3] += r.w;
        } else {
          quad_y_own<NX, NY>(G, cb, xb, hv, p0, t0 + a, x0 + b, acc[a][b], ymode);
        }
        dot += quad_epilogue<EPI>(A, pde, (size_t)v * P + p0, x, acc[a][b]);
        ++nq;
      }
  }
  if (A.pts) {
    __shared__ int sq;
    if (threadIdx.x == 0) sq = 0;
    __syncthreads();
    if (nq) atomicAdd(&sq, 4 * nq);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(A.pts + EPI, (unsigned long long)sq);
  }
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (threadIdx.x == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------------
// Fused S apply for 3D fp32 levels: both passes in one kernel, all neighbour data from
// shared memory.  One CTA per (vector, tile of kFX x-rows x all y), marching along t:
//   step j:  x plane j+5 -> smem ring (cp.async, one plane ahead of use)
//            h(j), Q_d = u~_d h(j) on the tile rows + 2 halo rows (x from the smem ring,
//            cf from HBM), Q_x / Q_y -> smem (this plane only)
//            t-direction terms of S are SCATTERED: x(j) and Q_t(j) add
//              P0_i[j-i] x(j) - KT_i[j-i] . Q_t(j)   to the accumulators of planes
//            i = j-5 .. j+5 (a thread-private smem ring), plus sigma alpha h(j) to plane j
//            x / y terms of plane j (gathered from the smem plane) -> accumulator j
//            plane j-5 is complete -> epilogue (the same EpiArgs contract as pass 2)
// HBM traffic per point: x 4 + cf 32 + the epilogue's vectors (no h round trip, cf read
// once instead of twice).  The t-direction coefficient rows of step j (uniform over the
// CTA) are staged in smem by the first threads.
// ---------------------------------------------------------------------------------
constexpr int kFX = 8;     // x rows per tile
constexpr int kFXR = 10;   // x-plane ring: planes j-4 .. j+5
constexpr int kFAR = 11;   // accumulator ring: planes j-5 .. j+5
constexpr int kFLag = 5;   // plane j - kFLag is output at step j

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void sts4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void f4axpy(float4& a, float c, float4 x) {
  a.x += c * x.x;
  a.y += c * x.y;
  a.z += c * x.z;
  a.w += c * x.w;
}

static inline size_t fused_smem_floats(int n2) {
  return (size_t)kFXR * (kFX + 8) * n2 + (size_t)4 * (kFX + 4) * n2 + (size_t)kFAR * kFX * n2 + 64;
}

template <int EPI>
__global__ void k_schur_fused(Geo G, const float* __restrict__ cf, int crep,
                              const float* __restrict__ x, EpiArgs A, const int* act) {
  MPDE_PDL_ENTRY();
  extern __shared__ __align__(16) float fsm[];
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2], s0 = G.stride[0];
  const int NY4 = n2 >> 2, X0 = blockIdx.x * kFX;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int hr = tid / NY4, q = tid - hr * NY4, y0 = 4 * q;
  const int xg = X0 - 2 + hr;                       // this thread's h row
  const bool hval = xg >= 0 && xg < n1;
  const bool own = hr >= 2 && hr < kFX + 2;         // tile row -> owns an output quad
  const int orow = hr - 2;
  float* xs = fsm;                                   // [kFXR][kFX+8][n2]
  float* qs = xs + (size_t)kFXR * (kFX + 8) * n2;    // [4][kFX+4][n2]
  float* as = qs + (size_t)4 * (kFX + 4) * n2;       // [kFAR][kFX][n2]
  float* ct = as + (size_t)kFAR * kFX * n2;          // [18] Kf_t(j), [33] scatter rows
  const int xrow_sz = (kFX + 8) * n2, qrow_sz = (kFX + 4) * n2, arow_sz = kFX * n2;
  const float* cb = cf + (size_t)pde * 8 * P;
  const float* xb = x + (size_t)v * P;
  const float wb2 = G.wb * G.wb;

  auto load_plane = [&](int k) {
    if (k < n0) {
      float* dst = xs + (k % kFXR) * xrow_sz;
      const float* src = xb + (size_t)k * s0;
      for (int c = tid; c < (kFX + 8) * NY4; c += nthr) {
        const int r = c / NY4, qq = c - r * NY4, xr = X0 - 4 + r;
        if (xr >= 0 && xr < n1) cp_async16(dst + r * n2 + 4 * qq, src + (size_t)xr * n2 + 4 * qq);
      }
    }
    cp_async_commit();
  };
  if (own)
    for (int m = 0; m < kFAR; ++m) sts4(as + m * arow_sz + orow * n2 + y0, make_float4(0.f, 0.f, 0.f, 0.f));
#pragma unroll 1
  for (int k = 0; k < kFLag; ++k) load_plane(k);

  double dot = 0.0;
#pragma unroll 1
  for (int j = 0; j < n0 + kFLag; ++j) {
    if (j < n0) {
      load_plane(j + kFLag);
      // t-direction coefficient rows of this step (uniform): Kf row j, scatter rows i=j-5..j+5
      if (tid < 18) {
        const int o = tid / 2 - 4, k = tid & 1;
        ct[tid] = (j + o >= 0 && j + o < n0) ? __ldg(tab_row(G, 0, j) + kTabKf + (o + 4) * 2 + k) : 0.f;
      } else if (tid < 51) {
        const int m = (tid - 18) / 3, c = (tid - 18) % 3, i = j - kFLag + m, o = j - i;
        float val = 0.f;
        if (i >= 0 && i < n0) {
          const float* row = tab_row(G, 0, i);
          if (c == 0) val = __ldg(row + kTabP0 + o + 5);
          else if (o >= -4 && o <= 4) val = __ldg(row + kTabKT + (o + 4) * 2 + (c - 1));
        }
        ct[tid] = val;
      }
      cp_async_wait1();
      __syncthreads();
      const float* xj = xs + (j % kFXR) * xrow_sz;  // plane j
      // ---- h(j), Q on the h rows --------------------------------------------------------
      float4 qx1 = make_float4(0.f, 0.f, 0.f, 0.f), qx2 = qx1, qy1 = qx1, qy2 = qx1;
      if (hval) {
        const size_t pg = (size_t)j * s0 + (size_t)xg * n2 + y0;
        const float4 csa = ld4(cb + pg), cis = ld4(cb + P + pg);
        const float4 ut1 = ld4(cb + 2 * (size_t)P + pg), ut2 = ld4(cb + 3 * (size_t)P + pg);
        const float4 ux1 = ld4(cb + 4 * (size_t)P + pg), ux2 = ld4(cb + 5 * (size_t)P + pg);
        const float4 uy1 = ld4(cb + 6 * (size_t)P + pg), uy2 = ld4(cb + 7 * (size_t)P + pg);
        const int xrr = hr + 2;  // row of xg in the x ring
        const float4 x0 = lds4(xj + xrr * n2 + y0);
        float g[4] = {csa.x * x0.x, csa.y * x0.y, csa.z * x0.z, csa.w * x0.w};
        {  // t
          float4 k1 = make_float4(0.f, 0.f, 0.f, 0.f), k2 = k1;
          if (j >= 2 && j <= n0 - 3) {
#pragma unroll
            for (int o = -2; o <= 2; ++o) {
              const float4 xv = lds4(xs + ((j + o) % kFXR) * xrow_sz + xrr * n2 + y0);
              f4axpy(k1, G.irow[0][(o + 2) * 2], xv);
              f4axpy(k2, G.irow[0][(o + 2) * 2 + 1], xv);
            }
          } else {
#pragma unroll
            for (int o = -4; o <= 4; ++o) {
              const int pc = min(max(j + o, 0), n0 - 1);
              const float4 xv = lds4(xs + (pc % kFXR) * xrow_sz + xrr * n2 + y0);
              f4axpy(k1, ct[(o + 4) * 2], xv);
              f4axpy(k2, ct[(o + 4) * 2 + 1], xv);
            }
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) g[jj] -= F4(ut1, jj) * F4(k1, jj) + F4(ut2, jj) * F4(k2, jj);
        }
        {  // x
          float4 k1 = make_float4(0.f, 0.f, 0.f, 0.f), k2 = k1;
          if (xg >= 2 && xg <= n1 - 3) {
#pragma unroll
            for (int o = -2; o <= 2; ++o) {
              const float4 xv = lds4(xj + (xrr + o) * n2 + y0);
              f4axpy(k1, G.irow[1][(o + 2) * 2], xv);
              f4axpy(k2, G.irow[1][(o + 2) * 2 + 1], xv);
            }
          } else {
            float kf[20];
            ldv<5>(tab_row(G, 1, xg) + kTabKf, kf);
#pragma unroll
            for (int o = -4; o <= 4; ++o) {
              const int oc = min(max(xg + o, 0), n1 - 1) - xg;
              const float4 xv = lds4(xj + (xrr + oc) * n2 + y0);
              f4axpy(k1, kf[(o + 4) * 2], xv);
              f4axpy(k2, kf[(o + 4) * 2 + 1], xv);
            }
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) g[jj] -= F4(ux1, jj) * F4(k1, jj) + F4(ux2, jj) * F4(k2, jj);
        }
        {  // y: window x(y0-4 .. y0+7) of this row
          const float* xr = xj + xrr * n2;
          float w[12];
          const float4 wl = y0 >= 4 ? lds4(xr + y0 - 4) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 wr = y0 + 4 < n2 ? lds4(xr + y0 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            w[jj] = F4(wl, jj);
            w[4 + jj] = F4(x0, jj);
            w[8 + jj] = F4(wr, jj);
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int i = y0 + jj;
            float k1 = 0.f, k2 = 0.f;
            if (i >= 2 && i <= n2 - 3) {
#pragma unroll
              for (int o = -2; o <= 2; ++o) {
                k1 += G.irow[2][(o + 2) * 2] * w[4 + jj + o];
                k2 += G.irow[2][(o + 2) * 2 + 1] * w[4 + jj + o];
              }
            } else {
              float kf[20];
              ldv<5>(tab_row(G, 2, i) + kTabKf, kf);
#pragma unroll
              for (int o = -4; o <= 4; ++o) {
                if (4 + jj + o < 0 || 4 + jj + o > 11) continue;
                k1 += kf[(o + 4) * 2] * w[4 + jj + o];
                k2 += kf[(o + 4) * 2 + 1] * w[4 + jj + o];
              }
            }
            g[jj] -= F4(uy1, jj) * k1 + F4(uy2, jj) * k2;
          }
        }
        float4 hq;
        hq.x = F4(cis, 0) * g[0];
        hq.y = F4(cis, 1) * g[1];
        hq.z = F4(cis, 2) * g[2];
        hq.w = F4(cis, 3) * g[3];
        qx1 = make_float4(ux1.x * hq.x, ux1.y * hq.y, ux1.z * hq.z, ux1.w * hq.w);
        qx2 = make_float4(ux2.x * hq.x, ux2.y * hq.y, ux2.z * hq.z, ux2.w * hq.w);
        qy1 = make_float4(uy1.x * hq.x, uy1.y * hq.y, uy1.z * hq.z, uy1.w * hq.w);
        qy2 = make_float4(uy2.x * hq.x, uy2.y * hq.y, uy2.z * hq.z, uy2.w * hq.w);
        if (own) {  // scatter the t terms of x(j), Q_t(j) and sigma alpha h(j)
          const float4 qt1 = make_float4(ut1.x * hq.x, ut1.y * hq.y, ut1.z * hq.z, ut1.w * hq.w);
          const float4 qt2 = make_float4(ut2.x * hq.x, ut2.y * hq.y, ut2.z * hq.z, ut2.w * hq.w);
          float* ab = as + orow * n2 + y0;
#pragma unroll
          for (int m = 0; m < 2 * kFLag + 1; ++m) {
            const int i = j - kFLag + m;
            const float cp = ct[18 + 3 * m], ck1 = ct[19 + 3 * m], ck2 = ct[20 + 3 * m];
            if (i < 0 || i >= n0 || (cp == 0.f && ck1 == 0.f && ck2 == 0.f && m != kFLag)) continue;
            float* a = ab + (i % kFAR) * arow_sz;
            float4 av = lds4(a);
            f4axpy(av, cp, x0);
            f4axpy(av, -ck1, qt1);
            f4axpy(av, -ck2, qt2);
            if (m == kFLag) {
              av.x += csa.x * hq.x;
              av.y += csa.y * hq.y;
              av.z += csa.z * hq.z;
              av.w += csa.w * hq.w;
            }
            sts4(a, av);
          }
        }
      }
      sts4(qs + 0 * qrow_sz + hr * n2 + y0, qx1);
      sts4(qs + 1 * qrow_sz + hr * n2 + y0, qx2);
      sts4(qs + 2 * qrow_sz + hr * n2 + y0, qy1);
      sts4(qs + 3 * qrow_sz + hr * n2 + y0, qy2);
      __syncthreads();
      // ---- x / y terms of plane j on the tile rows ----------------------------------------
      if (own) {
        const int xo = X0 + orow, xrr = orow + 4, qrr = orow + 2;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (xo >= 7 && xo <= n1 - 8) {
#pragma unroll
          for (int o = -4; o <= 4; ++o) f4axpy(acc, G.irow[1][20 + o + 4], lds4(xj + (xrr + o) * n2 + y0));
#pragma unroll
          for (int o = -2; o <= 2; ++o) {
            f4axpy(acc, -G.irow[1][10 + (o + 2) * 2], lds4(qs + (qrr + o) * n2 + y0));
            f4axpy(acc, -G.irow[1][10 + (o + 2) * 2 + 1], lds4(qs + qrow_sz + (qrr + o) * n2 + y0));
          }
        } else {
          const float* row = tab_row(G, 1, xo);
          float p0r[12], ktr[20];
          ldv<3>(row + kTabP0, p0r);
          ldv<5>(row + kTabKT, ktr);
#pragma unroll
          for (int o = -5; o <= 5; ++o) {
            const int oc = min(max(xo + o, 0), n1 - 1) - xo;
            f4axpy(acc, p0r[o + 5], lds4(xj + (xrr + oc) * n2 + y0));
          }
#pragma unroll
          for (int o = -4; o <= 4; ++o) {
            const int oc = min(max(xo + o, 0), n1 - 1) - xo;
            const int qr = min(max(qrr + oc, 0), kFX + 3);  // beyond the reach: zero coefficient
            f4axpy(acc, -ktr[(o + 4) * 2], lds4(qs + qr * n2 + y0));
            f4axpy(acc, -ktr[(o + 4) * 2 + 1], lds4(qs + qrow_sz + qr * n2 + y0));
          }
        }
        {  // y terms: x window (y0-8 .. y0+11), Q_y windows (y0-4 .. y0+7)
          const float* xr = xj + xrr * n2;
          const float* q1 = qs + 2 * qrow_sz + qrr * n2;
          const float* q2 = qs + 3 * qrow_sz + qrr * n2;
          float xw[20], aw[12], bw[12];
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int off = -8 + 4 * k;
            const bool ok = (y0 + off >= 0) && (y0 + off < n2);
            const float4 vv = ok ? lds4(xr + y0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) xw[4 * k + jj] = F4(vv, jj);
          }
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int off = -4 + 4 * k;
            const bool ok = (y0 + off >= 0) && (y0 + off < n2);
            const float4 va = ok ? lds4(q1 + y0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 vb = ok ? lds4(q2 + y0 + off) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              aw[4 * k + jj] = F4(va, jj);
              bw[4 * k + jj] = F4(vb, jj);
            }
          }
          float ay[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int i = y0 + jj;
            if (i >= 7 && i <= n2 - 8) {
#pragma unroll
              for (int o = -4; o <= 4; ++o) ay[jj] += G.irow[2][20 + o + 4] * xw[8 + jj + o];
#pragma unroll
              for (int o = -2; o <= 2; ++o)
                ay[jj] -= G.irow[2][10 + (o + 2) * 2] * aw[4 + jj + o] +
                          G.irow[2][10 + (o + 2) * 2 + 1] * bw[4 + jj + o];
            } else {
              const float* row = tab_row(G, 2, i);
              float p0r[12], ktr[20];
              ldv<3>(row + kTabP0, p0r);
              ldv<5>(row + kTabKT, ktr);
#pragma unroll
              for (int o = -5; o <= 5; ++o) ay[jj] += p0r[o + 5] * xw[8 + jj + o];
#pragma unroll
              for (int o = -4; o <= 4; ++o) {
                if (4 + jj + o < 0 || 4 + jj + o > 11) continue;
                ay[jj] -= ktr[(o + 4) * 2] * aw[4 + jj + o] + ktr[(o + 4) * 2 + 1] * bw[4 + jj + o];
              }
            }
          }
          const bool face = dir_face(G, 0, j) | dir_face(G, 1, xo);
          const float4 x0 = lds4(xr + y0);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (face || dir_face(G, 2, y0 + jj)) ay[jj] += wb2 * F4(x0, jj);
          acc.x += ay[0];
          acc.y += ay[1];
          acc.z += ay[2];
          acc.w += ay[3];
        }
        float* a = as + (j % kFAR) * arow_sz + orow * n2 + y0;
        float4 av = lds4(a);
        av.x += acc.x;
        av.y += acc.y;
        av.z += acc.z;
        av.w += acc.w;
        sts4(a, av);
      }
    }
    // ---- plane j - kFLag is complete: epilogue ----------------------------------------------
    if (own && j >= kFLag) {
      const int i = j - kFLag;
      float* a = as + (i % kFAR) * arow_sz + orow * n2 + y0;
      const float4 av = lds4(a);
      sts4(a, make_float4(0.f, 0.f, 0.f, 0.f));
      const float qv[4] = {av.x, av.y, av.z, av.w};
      dot += quad_epilogue<EPI>(A, pde, (size_t)v * P + (size_t)i * s0 + (size_t)(X0 + orow) * n2 + y0, x, qv);
    }
    if (j < n0) __syncthreads();
  }
  if (A.pts && tid == 0) atomicAdd(A.pts + EPI, (unsigned long long)kFX * n2 * n0);
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (tid == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------------
// Pass 2, shared-memory tiled (3D fp32, n_y = NY in {32, 64, 128}): a CTA computes a tile of
// kTT t-planes x kTX x-rows x all y.  Every operand it reads with a halo is staged once in
// shared memory with cp.async (axis-aligned cross halos only: the t column of the tile's
// rows, the x rows of the tile's planes), then each thread evaluates one y-quad from smem
// (no per-tap global address arithmetic, L1-latency operands).  Regions (rows of NY floats):
//   XA x  planes t0-5 .. t0+kTT+4, tile rows        XC x  tile planes, rows X0-5 .. X0+kTX+4
//   HA h  planes t0-4 .. t0+kTT+3, tile rows        HC h  tile planes, rows X0-4 .. X0+kTX+3
//   UT u~_t (2) like HA   UX u~_x (2) like HC   UY u~_y (2), SA sigma alpha: tile planes/rows
// (halos = the largest reach of the edge-class rows: P0 5 (rows 0 <-> 5), K^T 4)
// Out-of-domain rows are zero-filled; their coefficients are zero.
// ---------------------------------------------------------------------------------
constexpr int kTT = 4, kTX = 4;
constexpr int kTPL = kTT + 8;            // planes in the t-column regions of h, u~_t
constexpr int kTPX = kTT + 10;           // planes in the t-column region of x
constexpr int kTRows = kTPX * kTX /*XA*/ + kTT * (kTX + 10) /*XC*/ + kTPL * kTX /*HA*/ +
                       kTT * (kTX + 8) /*HC*/ + 2 * kTPL * kTX /*UT*/ + 2 * kTT * (kTX + 8) /*UX*/ +
                       2 * kTT * kTX /*UY*/ + kTT * kTX /*SA*/;
static inline size_t tile_smem_bytes(int ny) { return sizeof(float) * (size_t)kTRows * ny; }

template <int EPI, int NY>
__global__ void __launch_bounds__(4 * NY) k_schur_s_tile(Geo G, const float* __restrict__ cf, int crep,
                                                        const float* __restrict__ x,
                                                        const float* __restrict__ hb, EpiArgs A,
                                                        const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int NQ = NY / 4, NTH = 4 * NY;  // threads = kTT * kTX * NQ
  extern __shared__ __align__(16) float tsm[];
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int n0 = G.n[0], n1 = G.n[1];
  const int s0 = n1 * NY;
  const int nxt = n1 / kTX;
  const int X0 = (blockIdx.x % nxt) * kTX, t0 = (blockIdx.x / nxt) * kTT;
  float* XA = tsm;
  float* XC = XA + kTPX * kTX * NY;
  float* HA = XC + kTT * (kTX + 10) * NY;
  float* HC = HA + kTPL * kTX * NY;
  float* UT = HC + kTT * (kTX + 8) * NY;
  float* UX = UT + 2 * kTPL * kTX * NY;
  float* UY = UX + 2 * kTT * (kTX + 8) * NY;
  float* SA = UY + 2 * kTT * kTX * NY;
  const float* cb = cf + (size_t)pde * 8 * P;
  const float* xb = x + (size_t)v * P;
  const float* hv = hb + (size_t)v * P;
  const int tid = threadIdx.x;
  // ---- stage: one 16-byte chunk per (row, quad); rows outside the domain -> zeros --------
  auto stage = [&](float* dst, const float* src, int pl0, int npl, int r0, int nr) {
    const int n = npl * nr * NQ;
    for (int c = tid; c < n; c += NTH) {
      const int qq = c % NQ, rr = c / NQ, r = rr % nr, pl = rr / nr;
      const int t = pl0 + pl, xr = r0 + r;
      float* d = dst + (size_t)rr * NY + 4 * qq;
      if (t >= 0 && t < n0 && xr >= 0 && xr < n1)
        cp_async16(d, src + (size_t)t * s0 + (size_t)xr * NY + 4 * qq);
      else
        *reinterpret_cast<float4*>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  stage(XA, xb, t0 - 5, kTPX, X0, kTX);
  stage(XC, xb, t0, kTT, X0 - 5, kTX + 10);
  stage(HA, hv, t0 - 4, kTPL, X0, kTX);
  stage(HC, hv, t0, kTT, X0 - 4, kTX + 8);
  stage(UT, cb + 2 * (size_t)P, t0 - 4, kTPL, X0, kTX);
  stage(UT + kTPL * kTX * NY, cb + 3 * (size_t)P, t0 - 4, kTPL, X0, kTX);
  stage(UX, cb + 4 * (size_t)P, t0, kTT, X0 - 4, kTX + 8);
  stage(UX + kTT * (kTX + 8) * NY, cb + 5 * (size_t)P, t0, kTT, X0 - 4, kTX + 8);
  stage(UY, cb + 6 * (size_t)P, t0, kTT, X0, kTX);
  stage(UY + kTT * kTX * NY, cb + 7 * (size_t)P, t0, kTT, X0, kTX);
  stage(SA, cb, t0, kTT, X0, kTX);
  cp_async_commit();
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();

  // ---- this thread's quad: warp-specialised interior / edge y quads over 16 tile rows ------
  constexpr int NE = NQ < 4 ? NQ : 4, NI = NQ - NE, R = kTT * kTX;
  int rr, q, ymode;
  if (tid < R * NI) {
    rr = tid / NI;
    q = 2 + tid % NI;
    ymode = 1;
  } else {
    const int k = tid - R * NI, e = k % NE;
    rr = k / NE;
    q = (NE == 4 && e >= 2) ? NQ - 4 + e : e;
    ymode = 2;
  }
  const int tt = rr / kTX, xx = rr % kTX, t = t0 + tt, xo = X0 + xx, y0 = 4 * q;
  double dot = 0.0;
  if (t < n0) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const float* xa = XA + xx * NY + y0;             // + plane * kTX * NY
    const float* ha = HA + xx * NY + y0;
    const float* u1a = UT + xx * NY + y0;
    const float* u2a = u1a + kTPL * kTX * NY;
    const int pa = tt + 4, px = tt + 5;              // this plane in the t-column regions
    // t terms
    if (t >= 7 && t <= n0 - 8) {
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const float4 xv = lds4(xa + (px + o) * kTX * NY);
        const float c = G.irow[0][20 + o + 4];
        acc[0] += c * xv.x; acc[1] += c * xv.y; acc[2] += c * xv.z; acc[3] += c * xv.w;
      }
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const int off = (pa + o) * kTX * NY;
        const float4 va = lds4(u1a + off), vb = lds4(u2a + off), hq = lds4(ha + off);
        const float a = G.irow[0][10 + (o + 2) * 2], b = G.irow[0][10 + (o + 2) * 2 + 1];
        acc[0] -= (a * va.x + b * vb.x) * hq.x; acc[1] -= (a * va.y + b * vb.y) * hq.y;
        acc[2] -= (a * va.z + b * vb.z) * hq.z; acc[3] -= (a * va.w + b * vb.w) * hq.w;
      }
    } else {
      const float* row = tab_row(G, 0, t);
      float p0r[12], ktr[20];
      ldv<3>(row + kTabP0, p0r);
      ldv<5>(row + kTabKT, ktr);
#pragma unroll
      for (int o = -5; o <= 5; ++o) {
        const float4 xv = lds4(xa + (px + o) * kTX * NY);
        const float c = p0r[o + 5];
        acc[0] += c * xv.x; acc[1] += c * xv.y; acc[2] += c * xv.z; acc[3] += c * xv.w;
      }
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const int off = (pa + o) * kTX * NY;
        const float4 va = lds4(u1a + off), vb = lds4(u2a + off), hq = lds4(ha + off);
        const float a = ktr[(o + 4) * 2], b = ktr[(o + 4) * 2 + 1];
        acc[0] -= (a * va.x + b * vb.x) * hq.x; acc[1] -= (a * va.y + b * vb.y) * hq.y;
        acc[2] -= (a * va.z + b * vb.z) * hq.z; acc[3] -= (a * va.w + b * vb.w) * hq.w;
      }
    }
    // x terms
    const float* xc = XC + (tt * (kTX + 10) + xx + 5) * NY + y0;
    const float* hc = HC + (tt * (kTX + 8) + xx + 4) * NY + y0;
    const float* u1c = UX + (tt * (kTX + 8) + xx + 4) * NY + y0;
    const float* u2c = u1c + kTT * (kTX + 8) * NY;
    if (xo >= 7 && xo <= n1 - 8) {
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const float4 xv = lds4(xc + o * NY);
        const float c = G.irow[1][20 + o + 4];
        acc[0] += c * xv.x; acc[1] += c * xv.y; acc[2] += c * xv.z; acc[3] += c * xv.w;
      }
#pragma unroll
      for (int o = -2; o <= 2; ++o) {
        const float4 va = lds4(u1c + o * NY), vb = lds4(u2c + o * NY), hq = lds4(hc + o * NY);
        const float a = G.irow[1][10 + (o + 2) * 2], b = G.irow[1][10 + (o + 2) * 2 + 1];
        acc[0] -= (a * va.x + b * vb.x) * hq.x; acc[1] -= (a * va.y + b * vb.y) * hq.y;
        acc[2] -= (a * va.z + b * vb.z) * hq.z; acc[3] -= (a * va.w + b * vb.w) * hq.w;
      }
    } else {
      const float* row = tab_row(G, 1, xo);
      float p0r[12], ktr[20];
      ldv<3>(row + kTabP0, p0r);
      ldv<5>(row + kTabKT, ktr);
#pragma unroll
      for (int o = -5; o <= 5; ++o) {
        const float4 xv = lds4(xc + o * NY);
        const float c = p0r[o + 5];
        acc[0] += c * xv.x; acc[1] += c * xv.y; acc[2] += c * xv.z; acc[3] += c * xv.w;
      }
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        const float4 va = lds4(u1c + o * NY), vb = lds4(u2c + o * NY), hq = lds4(hc + o * NY);
        const float a = ktr[(o + 4) * 2], b = ktr[(o + 4) * 2 + 1];
        acc[0] -= (a * va.x + b * vb.x) * hq.x; acc[1] -= (a * va.y + b * vb.y) * hq.y;
        acc[2] -= (a * va.z + b * vb.z) * hq.z; acc[3] -= (a * va.w + b * vb.w) * hq.w;
      }
    }
    // y terms and own terms
    {
      const float* u1y = UY + (tt * kTX + xx) * NY;
      const float* u2y = u1y + kTT * kTX * NY;
      const float* xr = xc - y0;
      const float* hr = hc - y0;
      float xw[20], aw[12], bw[12], hw[12];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int off = y0 - 8 + 4 * k;
        const bool ok = ymode == 1 || (off >= 0 && off < NY);
        const float4 vv = ok ? lds4(xr + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        xw[4 * k] = vv.x; xw[4 * k + 1] = vv.y; xw[4 * k + 2] = vv.z; xw[4 * k + 3] = vv.w;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int off = y0 - 4 + 4 * k;
        const bool ok = ymode == 1 || (off >= 0 && off < NY);
        const float4 va = ok ? lds4(u1y + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 vb = ok ? lds4(u2y + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 hq = ok ? lds4(hr + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        aw[4 * k] = va.x; aw[4 * k + 1] = va.y; aw[4 * k + 2] = va.z; aw[4 * k + 3] = va.w;
        bw[4 * k] = vb.x; bw[4 * k + 1] = vb.y; bw[4 * k + 2] = vb.z; bw[4 * k + 3] = vb.w;
        hw[4 * k] = hq.x; hw[4 * k + 1] = hq.y; hw[4 * k + 2] = hq.z; hw[4 * k + 3] = hq.w;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (ymode == 1) {
#pragma unroll
          for (int o = -4; o <= 4; ++o) acc[j] += G.irow[2][20 + o + 4] * xw[8 + j + o];
#pragma unroll
          for (int o = -2; o <= 2; ++o)
            acc[j] -= (G.irow[2][10 + (o + 2) * 2] * aw[4 + j + o] +
                       G.irow[2][10 + (o + 2) * 2 + 1] * bw[4 + j + o]) * hw[4 + j + o];
        } else {
          const float* row = tab_row(G, 2, y0 + j);
          float p0r[12], ktr[20];
          ldv<3>(row + kTabP0, p0r);
          ldv<5>(row + kTabKT, ktr);
#pragma unroll
          for (int o = -5; o <= 5; ++o) acc[j] += p0r[o + 5] * xw[8 + j + o];
#pragma unroll
          for (int o = -4; o <= 4; ++o) {
            if (4 + j + o < 0 || 4 + j + o > 11) continue;
            acc[j] -= (ktr[(o + 4) * 2] * aw[4 + j + o] + ktr[(o + 4) * 2 + 1] * bw[4 + j + o]) *
                      hw[4 + j + o];
          }
        }
      }
      const float4 sa = lds4(SA + (tt * kTX + xx) * NY + y0);
      const bool face = dir_face(G, 0, t) | dir_face(G, 1, xo);
      const float wb2 = G.wb * G.wb;
      const float sav[4] = {sa.x, sa.y, sa.z, sa.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[j] += sav[j] * hw[4 + j];
        if (face || dir_face(G, 2, y0 + j)) acc[j] += wb2 * xw[8 + j];
      }
    }
    dot = quad_epilogue<EPI>(A, pde, (size_t)v * P + (size_t)t * s0 + (size_t)xo * NY + y0, x, acc);
  }
  if (A.pts && tid == 0) {
    const int nt = min(kTT, n0 - t0);
    atomicAdd(A.pts + EPI, (unsigned long long)nt * kTX * NY);
  }
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (tid == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

// ---------------------------------------------------------------------------------
// 3D fp32 pass 1 with the y-axis (contiguous) part of S folded in ("hy"): a CTA covers
// R = kThreads / (n_y/4) whole rows (remap_quad mapping).  Each thread computes h of its
// quad, parks x, u~_y1 h, u~_y2 h of the quad in shared memory, and after one barrier
// evaluates  r_y = P0_y x - K_y^T (u~_y h) + sigma alpha h + w_bnd^2 [B] x  from the smem rows
// (no neighbour h from HBM).  Writes h and r_y (second half of the 8-byte-per-point g
// buffer); pass 2 then needs only the t and x axes (fewer registers, no y windows).
// ---------------------------------------------------------------------------------
template <int NX, int NY>
__global__ void __launch_bounds__(kThreads) k_schur_hy(Geo G, const float* __restrict__ cf, int crep,
                                                      const float* __restrict__ x,
                                                      float* __restrict__ gout, const int* act,
                                                      unsigned long long* pts) {
  MPDE_PDL_ENTRY();
  __shared__ __align__(16) float sx[4 * kThreads], sw1[4 * kThreads], sw2[4 * kThreads],
      sh[4 * kThreads];
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;
  const int nl = dim_n<NX, NY>(G, 2), NY4 = nl >> 2;
  if (pts && threadIdx.x == 0) atomicAdd(pts, (unsigned long long)block_points(1, P, nl, 0));
  const float* cb = cf + (size_t)pde * 8 * P;
  const float* xb = x + (size_t)v * P;
  {  // phase 1, natural mapping (coalesced): h of this thread's quad -> HBM and smem
    const int pn = (blockIdx.x * kThreads + threadIdx.x) * 4;
    if (pn < P) {
      int id[3];
      unravel<3>(G, pn, id);
      float hn[4];
      schur_h4<3, float>(G, cb, xb, pn, id, hn, 0);
      st4(gout + (size_t)v * P + pn, hn);
      const float4 u1 = ld4(cb + 6 * (size_t)P + pn), u2 = ld4(cb + 7 * (size_t)P + pn);
      const int so = 4 * threadIdx.x;  // CTA rows are contiguous: smem index = pn - CTA base
      sts4(sx + so, ld4(xb + pn));
      sts4(sh + so, make_float4(hn[0], hn[1], hn[2], hn[3]));
      sts4(sw1 + so, make_float4(u1.x * hn[0], u1.y * hn[1], u1.z * hn[2], u1.w * hn[3]));
      sts4(sw2 + so, make_float4(u2.x * hn[0], u2.y * hn[1], u2.z * hn[2], u2.w * hn[3]));
    }
  }
  __syncthreads();
  // phase 2, warp-specialised mapping (interior / edge y quads), operands from smem
  int row, q, ymode;
  remap_quad(NY4, row, q, ymode);
  const int lr = row - (int)blockIdx.x * (kThreads / NY4), y0 = 4 * q;
  const int p0 = row * nl + y0;
  if (p0 >= P) return;
  int idx[3];
  unravel<3>(G, p0, idx);
  const float* sxr = sx + lr * nl;
  const float* sw1r = sw1 + lr * nl;
  const float* sw2r = sw2 + lr * nl;
  const float4 hv4 = lds4(sh + lr * nl + y0), csa = ld4(cb + p0);
  const float hq[4] = {hv4.x, hv4.y, hv4.z, hv4.w};
  float xw[20], aw[12], bw[12];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int off = y0 - 8 + 4 * k;
    const bool ok = ymode == 1 || (off >= 0 && off < nl);
    const float4 vv = ok ? lds4(sxr + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    xw[4 * k] = vv.x; xw[4 * k + 1] = vv.y; xw[4 * k + 2] = vv.z; xw[4 * k + 3] = vv.w;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int off = y0 - 4 + 4 * k;
    const bool ok = ymode == 1 || (off >= 0 && off < nl);
    const float4 va = ok ? lds4(sw1r + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 vb = ok ? lds4(sw2r + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    aw[4 * k] = va.x; aw[4 * k + 1] = va.y; aw[4 * k + 2] = va.z; aw[4 * k + 3] = va.w;
    bw[4 * k] = vb.x; bw[4 * k + 1] = vb.y; bw[4 * k + 2] = vb.z; bw[4 * k + 3] = vb.w;
  }
  float ry[4];
  const bool face = dir_face(G, 0, idx[0]) | dir_face(G, 1, idx[1]);
  const float wb2 = G.wb * G.wb;
  const float sav[4] = {csa.x, csa.y, csa.z, csa.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float a = sav[j] * hq[j];
    if (face || dir_face(G, 2, y0 + j)) a += wb2 * xw[8 + j];
    if (ymode == 1) {
#pragma unroll
      for (int o = -4; o <= 4; ++o) a += G.irow[2][20 + o + 4] * xw[8 + j + o];
#pragma unroll
      for (int o = -2; o <= 2; ++o)
        a -= G.irow[2][10 + (o + 2) * 2] * aw[4 + j + o] + G.irow[2][10 + (o + 2) * 2 + 1] * bw[4 + j + o];
    } else {
      const float* rowp = tab_row(G, 2, y0 + j);
      float p0r[12], ktr[20];
      ldv<3>(rowp + kTabP0, p0r);
      ldv<5>(rowp + kTabKT, ktr);
#pragma unroll
      for (int o = -5; o <= 5; ++o) a += p0r[o + 5] * xw[8 + j + o];
#pragma unroll
      for (int o = -4; o <= 4; ++o) {
        if (4 + j + o < 0 || 4 + j + o > 11) continue;
        a -= ktr[(o + 4) * 2] * aw[4 + j + o] + ktr[(o + 4) * 2 + 1] * bw[4 + j + o];
      }
    }
    ry[j] = a;
  }
  st4(gout + (size_t)gridDim.y * P + (size_t)v * P + p0, ry);
}

// ------------------------------------------------------------------------- launchers
static inline dim3 grid2(int P, int nvec) { return dim3((P + kThreads - 1) / kThreads, nvec); }

#define DISPATCH_D2(D_, ...) \
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

void launch_schur_coef(const Geo& G, int B, const float* c, float* cf, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D2(G.D, k_schur_coef<DD><<<grid2(G.P, B), kThreads, 0, s>>>(G, c, cf));
}

static inline bool small_level(const Geo& G);
static int g_small_scalar = -1;  // env MPDE_SMALL_SCALAR=1: 1-point-per-thread kernels on small levels
static inline bool use_v4(const Geo& G) {
  if (g_small_scalar < 0) {
    const char* e = getenv("MPDE_SMALL_SCALAR");
    g_small_scalar = e ? atoi(e) : 0;
  }
  if (g_small_scalar && small_level(G)) return false;
  return (G.n[G.D - 1] & 3) == 0;
}
// small levels (<= 16384 points per vector): 4-points-per-thread kernels in 64-thread CTAs
// (a 256-thread CTA per PDE leaves most SMs idle at the coarse levels)
static int g_small_p = -1;  // points-per-vector threshold (env MPDE_SMALLP, default 16384)
static inline bool small_level(const Geo& G) {
  if (g_small_p < 0) {
    const char* e = getenv("MPDE_SMALLP");
    g_small_p = e ? atoi(e) : 16384;
  }
  return G.P <= g_small_p;
}
static inline int v4_threads(const Geo& G) { return small_level(G) ? kSmallThreads : kThreads; }
static int g_small_lat = -1;  // env MPDE_SMALL_LAT=0: small-level pass 1 with the per-axis load phases
static inline bool small_lat(const Geo& G) {
  if (g_small_lat < 0) {
    const char* e = getenv("MPDE_SMALL_LAT");
    g_small_lat = e ? atoi(e) : 1;
  }
  return g_small_lat && small_level(G) && use_v4(G);
}
// warp-specialised interior / edge quads (remap_quad): NY4 a power of two dividing kThreads
static int g_remap = -1;  // env MPDE_REMAP=1: warp-specialised interior / edge quad mapping
static inline int use_remap(const Geo& G) {
  if (g_remap < 0) {
    const char* e = getenv("MPDE_REMAP");
    g_remap = e ? atoi(e) : 0;  // default natural: see DESIGN.md §4 tuning table
  }
  const int q = G.n[G.D - 1] >> 2;
  return g_remap && use_v4(G) && !small_level(G) && q > 0 && (q & (q - 1)) == 0 && q <= kThreads;
}
// 2x2 (t,x)-blocked pass 2: 3D, fp32, n_y % 4 == 0
static int g_block_mode = -1;  // 0: v4, 1: 2x1 (t), 2: 2x2 (t,x); env MPDE_SCHUR_BLOCK
static inline int block_mode() {
  if (g_block_mode < 0) {
    const char* e = getenv("MPDE_SCHUR_BLOCK");
    g_block_mode = e ? atoi(e) : 1;
  }
  return g_block_mode;
}
static inline bool use_b22(const Geo& G, bool f64) {
  return G.D == 3 && !f64 && use_v4(G) && !small_level(G) && block_mode() > 0;
}
static inline int b22_threads(const Geo& G) {
  const int bx = block_mode() == 2;
  return ((G.n[0] + 1) / 2) * (bx ? (G.n[1] + 1) / 2 : G.n[1]) * (G.n[2] / 4);
}
// t-pairs per CTA of the t-blocked pass 2 (env MPDE_B22_TP, default 1 = one x-row strip;
// 2/4/8 measured 3-10% slower at C4)
static int g_b22_tp = -1;
static inline int b22_tp(const Geo& G) {
  if (g_b22_tp < 0) {
    const char* e = getenv("MPDE_B22_TP");
    g_b22_tp = e ? atoi(e) : 1;
  }
  const int R = kThreads / (G.n[2] / 4);
  if (!use_remap(G) || block_mode() != 1 || g_b22_tp <= 1 || R % g_b22_tp) return 1;
  return g_b22_tp;
}
static inline int b22_ctas(const Geo& G) {
  const int tp = b22_tp(G);
  if (tp <= 1) return (b22_threads(G) + kThreads - 1) / kThreads;
  const int R = kThreads / (G.n[2] / 4), XPB = R / tp;
  return ((G.n[0] + 1) / 2 + tp - 1) / tp * ((G.n[1] + XPB - 1) / XPB);
}
// pass 1 with the y part folded in (k_schur_hy) + pass 2 on t and x only: the t-blocked
// pass-2 levels with the warp-specialised mapping (env MPDE_HY=0 disables)
static int g_hy = -1;
static inline bool use_hy(const Geo& G, bool f64) {
  if (g_hy < 0) {
    const char* e = getenv("MPDE_HY");
    g_hy = e ? atoi(e) : 0;
  }
  return g_hy && use_b22(G, f64) && block_mode() == 1 && use_remap(G);
}
// fused single-kernel S apply (k_schur_fused): 3D fp32 levels with full-row tiles
static int g_fused = -1;  // env MPDE_FUSED=1 enables (default off: slower)
static inline bool use_fused(const Geo& G, bool f64) {
  if (g_fused < 0) {
    const char* e = getenv("MPDE_FUSED");
    g_fused = e ? atoi(e) : 0;
  }
  const int n1 = G.D == 3 ? G.n[1] : 0, n2 = G.D == 3 ? G.n[2] : 0;
  return g_fused && G.D == 3 && !f64 && !small_level(G) && n2 % 4 == 0 && n2 >= 32 && n2 <= 128 &&
         n1 % kFX == 0 && n1 >= 2 * kFX;
}
bool schur_fused(const Geo& G, bool f64) { return use_fused(G, f64); }
// smem-tiled pass 2 (k_schur_s_tile): 3D fp32, n_y in {32, 64, 128}, n_x % kTX == 0
static int g_tile = -1;  // env MPDE_TILE=1 enables (default off: slower)
static inline bool use_tile(const Geo& G, bool f64) {
  if (g_tile < 0) {
    const char* e = getenv("MPDE_TILE");
    g_tile = e ? atoi(e) : 0;
  }
  if (!g_tile || G.D != 3 || f64 || small_level(G)) return false;
  const int n2 = G.n[2];
  if (g_tile == 2 && n2 > 32) return false;  // 2: only the n_y = 32 levels
  return (n2 == 32 || n2 == 64 || n2 == 128) && G.n[1] % kTX == 0 && G.n[1] >= 2 * kTX;
}
static inline int tile_ctas(const Geo& G) { return ((G.n[0] + kTT - 1) / kTT) * (G.n[1] / kTX); }
// CTAs per vector of the two-pass pass-2 kernel (grid x of its launches)
static int schur_tiles2p(const Geo& G, bool f64) {
  if (use_fused(G, f64)) return G.n[1] / kFX;
  if (use_tile(G, f64)) return tile_ctas(G);
  if (use_b22(G, f64)) return b22_ctas(G);
  if (use_v4(G)) {
    const int th = v4_threads(G);
    return (G.P + 4 * th - 1) / (4 * th);
  }
  return (G.P + kThreads - 1) / kThreads;
}

int schur_tiles(const Geo& G, bool f64, int nvec) {
  if (use_march(G, f64, nvec)) return march_ctas(G);
  if (use_slab(G, f64)) return slab_ctas(G);
  if (use_small_fused(G, f64)) return 1;
  return schur_tiles2p(G, f64);
}

// warp-specialised interior / edge y quads in pass 1 too (env MPDE_P1_REMAP=1 enables)
static int g_p1_remap = -1;
static inline int pass1_remap(const Geo& G) {
  if (g_p1_remap < 0) {
    const char* e = getenv("MPDE_P1_REMAP");
    g_p1_remap = e ? atoi(e) : 0;  // opt-in: 48.9 vs 49.5 ms per C4 step (no gain)
  }
  return g_p1_remap && use_remap(G) ? 1 : 0;
}

void launch_schur_g(const Geo& G, int nvec, int crep, const float* cf, const float* x, void* g,
                    const int* act, unsigned long long* pts, bool f64, cudaStream_t s) {
  ++g_launch_count;
  if (use_hy(G, f64)) {
    const dim3 gr((G.P + 4 * kThreads - 1) / (4 * kThreads), nvec);
    if (G.n[1] == 64 && G.n[2] == 64)
      k_schur_hy<64, 64><<<gr, kThreads, 0, s>>>(G, cf, crep, x, (float*)g, act, pts);
    else if (G.n[1] == 32 && G.n[2] == 32)
      k_schur_hy<32, 32><<<gr, kThreads, 0, s>>>(G, cf, crep, x, (float*)g, act, pts);
    else if (G.n[1] == 128 && G.n[2] == 128)
      k_schur_hy<128, 128><<<gr, kThreads, 0, s>>>(G, cf, crep, x, (float*)g, act, pts);
    else
      k_schur_hy<0, 0><<<gr, kThreads, 0, s>>>(G, cf, crep, x, (float*)g, act, pts);
    return;
  }
  if (use_v4(G)) {
    const int th = v4_threads(G);
    dim3 gr((G.P + 4 * th - 1) / (4 * th), nvec);
    if (small_lat(G)) {  // latency-bound small level: all loads before the edge branches
      if (f64)
        DISPATCH_D2(G.D, k_schur_h_v4_lat<DD, double, float><<<gr, th, 0, s>>>(G, cf, crep, x, (double*)g, act, pts));
      else
        DISPATCH_D2(G.D, k_schur_h_v4_lat<DD, float, float><<<gr, th, 0, s>>>(G, cf, crep, x, (float*)g, act, pts));
      return;
    }
    if (f64)
      DISPATCH_D2(G.D, k_schur_h_v4<DD, double><<<gr, th, 0, s>>>(G, cf, crep, x, (double*)g, act, pts, 0));
    else
      DISPATCH_D2(G.D, k_schur_h_v4<DD, float><<<gr, th, 0, s>>>(G, cf, crep, x, (float*)g, act, pts,
                                                                  pass1_remap(G)));
    return;
  }
  if (f64)
    DISPATCH_D2(G.D, k_schur_h<DD, double><<<grid2(G.P, nvec), kThreads, 0, s>>>(G, cf, crep, x, (double*)g, act, pts));
  else
    DISPATCH_D2(G.D, k_schur_h<DD, float><<<grid2(G.P, nvec), kThreads, 0, s>>>(G, cf, crep, x, (float*)g, act, pts));
}

void launch_schur_out(int epi, const Geo& G, int nvec, int crep, const float* cf, const float* x,
                      const void* g, const EpiArgs& A, const int* act, bool f64, cudaStream_t s) {
  ++g_launch_count;
  if (use_tile(G, f64)) {
    const dim3 gt(tile_ctas(G), nvec);
    const size_t smem = tile_smem_bytes(G.n[2]);
#define TILE_LAUNCH(E, NYv)                                                                  \
  {                                                                                          \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      cudaFuncSetAttribute(k_schur_s_tile<E, NYv>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)tile_smem_bytes(NYv));                                       \
      attr = true;                                                                           \
    }                                                                                        \
    k_schur_s_tile<E, NYv><<<gt, 4 * NYv, smem, s>>>(G, cf, crep, x, (const float*)g, A, act); \
  }
#define TILE_CASE(E)                                                                         \
  case E:                                                                                    \
    if (G.n[2] == 64) TILE_LAUNCH(E, 64)                                                     \
    else if (G.n[2] == 32) TILE_LAUNCH(E, 32)                                                \
    else TILE_LAUNCH(E, 128)                                                                 \
    break;
    switch (epi) {
      TILE_CASE(EPI_STORE)
      TILE_CASE(EPI_DOT)
      TILE_CASE(EPI_POWER)
      TILE_CASE(EPI_RESID)
      TILE_CASE(EPI_SMOOTH)
      TILE_CASE(EPI_SMOOTH_LAST)
      TILE_CASE(EPI_POST0)
    }
#undef TILE_CASE
#undef TILE_LAUNCH
    return;
  }
  if (use_b22(G, f64)) {
    const dim3 gb(schur_tiles2p(G, f64), nvec);
    const int rm = use_remap(G) ? b22_tp(G) : 0;  // >1: t-pair tiling (remap implied)
#define B22_LAUNCH(E, BXv, YPv)                                                              \
  if (G.n[1] == 64 && G.n[2] == 64)                                                          \
    k_schur_s_b22<E, BXv, 64, 64, YPv><<<gb, kThreads, 0, s>>>(G, cf, crep, x, (const float*)g, A, act, rm); \
  else if (G.n[1] == 32 && G.n[2] == 32)                                                     \
    k_schur_s_b22<E, BXv, 32, 32, YPv><<<gb, kThreads, 0, s>>>(G, cf, crep, x, (const float*)g, A, act, rm); \
  else if (G.n[1] == 128 && G.n[2] == 128)                                                   \
    k_schur_s_b22<E, BXv, 128, 128, YPv><<<gb, kThreads, 0, s>>>(G, cf, crep, x, (const float*)g, A, act, rm); \
  else                                                                                       \
    k_schur_s_b22<E, BXv, 0, 0, YPv><<<gb, kThreads, 0, s>>>(G, cf, crep, x, (const float*)g, A, act, rm);
#define B22_CASE(E)                                                                          \
  case E:                                                                                    \
    if (block_mode() == 2) {                                                                 \
      B22_LAUNCH(E, 1, 0)                                                                    \
    } else if (use_hy(G, f64)) {                                                             \
      B22_LAUNCH(E, 0, 1)                                                                    \
    } else {                                                                                 \
      B22_LAUNCH(E, 0, 0)                                                                    \
    }                                                                                        \
    break;
    switch (epi) {
      B22_CASE(EPI_STORE)
      B22_CASE(EPI_DOT)
      B22_CASE(EPI_POWER)
      B22_CASE(EPI_RESID)
      B22_CASE(EPI_SMOOTH)
      B22_CASE(EPI_SMOOTH_LAST)
      B22_CASE(EPI_POST0)
    }
#undef B22_CASE
#undef B22_LAUNCH
    return;
  }
  const bool v4 = use_v4(G);
  const int rm = use_remap(G);
  const int th = v4 ? v4_threads(G) : kThreads;
  dim3 gr(schur_tiles2p(G, f64), nvec);
#define EPI_CASE2(E)                                                                              \
  case E:                                                                                         \
    if (v4) {                                                                                     \
      if (f64)                                                                                    \
        DISPATCH_D2(G.D, k_schur_s_v4<DD, E, double><<<gr, th, 0, s>>>(G, cf, crep, x, (const double*)g, A, act, rm)); \
      else                                                                                        \
        DISPATCH_D2(G.D, k_schur_s_v4<DD, E, float><<<gr, th, 0, s>>>(G, cf, crep, x, (const float*)g, A, act, rm)); \
    } else if (f64)                                                                               \
      DISPATCH_D2(G.D, k_schur_s<DD, E, double><<<gr, kThreads, 0, s>>>(G, cf, crep, x, (const double*)g, A, act)); \
    else                                                                                          \
      DISPATCH_D2(G.D, k_schur_s<DD, E, float><<<gr, kThreads, 0, s>>>(G, cf, crep, x, (const float*)g, A, act)); \
    break;
  switch (epi) {
    EPI_CASE2(EPI_STORE)
    EPI_CASE2(EPI_DOT)
    EPI_CASE2(EPI_POWER)
    EPI_CASE2(EPI_RESID)
    EPI_CASE2(EPI_SMOOTH)
    EPI_CASE2(EPI_SMOOTH_LAST)
    EPI_CASE2(EPI_POST0)
  }
#undef EPI_CASE2
}

// ---- bf16-coefficient variants (V-cycle applies on level 0, mpde_options.cf_bf16) ----------
bool schur_bf16_ok(const Geo& G, bool f64) {
  return !f64 && use_v4(G) && !use_hy(G, f64) && !use_tile(G, f64) && !use_fused(G, f64) &&
         !(use_b22(G, f64) && block_mode() == 2);
}

void launch_schur_g_bf(const Geo& G, int nvec, int crep, const void* cf16, const float* x, void* g,
                       const int* act, unsigned long long* pts, cudaStream_t s) {
  ++g_launch_count;
  const __nv_bfloat16* cf = static_cast<const __nv_bfloat16*>(cf16);
  const int th = v4_threads(G);
  dim3 gr((G.P + 4 * th - 1) / (4 * th), nvec);
  DISPATCH_D2(G.D, (k_schur_h_v4<DD, float, __nv_bfloat16><<<gr, th, 0, s>>>(G, cf, crep, x, (float*)g, act, pts,
                                                                            pass1_remap(G))));
}

void launch_schur_out_bf(int epi, const Geo& G, int nvec, int crep, const void* cf16, const float* x,
                         const void* g, const EpiArgs& A, const int* act, cudaStream_t s) {
  ++g_launch_count;
  const __nv_bfloat16* cf = static_cast<const __nv_bfloat16*>(cf16);
  const float* gf = static_cast<const float*>(g);
  if (use_b22(G, false)) {
    const dim3 gb(schur_tiles2p(G, false), nvec);
    const int rm = use_remap(G) ? b22_tp(G) : 0;
#define B22BF(E)                                                                                  \
  case E:                                                                                         \
    if (G.n[1] == 64 && G.n[2] == 64)                                                             \
      k_schur_s_b22<E, 0, 64, 64, 0, __nv_bfloat16><<<gb, kThreads, 0, s>>>(G, cf, crep, x, gf, A, act, rm); \
    else if (G.n[1] == 32 && G.n[2] == 32)                                                        \
      k_schur_s_b22<E, 0, 32, 32, 0, __nv_bfloat16><<<gb, kThreads, 0, s>>>(G, cf, crep, x, gf, A, act, rm); \
    else if (G.n[1] == 128 && G.n[2] == 128)                                                      \
      k_schur_s_b22<E, 0, 128, 128, 0, __nv_bfloat16><<<gb, kThreads, 0, s>>>(G, cf, crep, x, gf, A, act, rm); \
    else                                                                                          \
      k_schur_s_b22<E, 0, 0, 0, 0, __nv_bfloat16><<<gb, kThreads, 0, s>>>(G, cf, crep, x, gf, A, act, rm); \
    break;
    switch (epi) {
      B22BF(EPI_RESID)
      B22BF(EPI_SMOOTH)
      B22BF(EPI_SMOOTH_LAST)
      B22BF(EPI_POST0)
    }
#undef B22BF
    return;
  }
  const int rm = use_remap(G);
  const int th = v4_threads(G);
  dim3 gr(schur_tiles2p(G, false), nvec);
#define V4BF(E)                                                                                   \
  case E:                                                                                         \
    DISPATCH_D2(G.D, (k_schur_s_v4<DD, E, float, __nv_bfloat16><<<gr, th, 0, s>>>(G, cf, crep, x, gf, A, act, rm))); \
    break;
  switch (epi) {
    V4BF(EPI_RESID)
    V4BF(EPI_SMOOTH)
    V4BF(EPI_SMOOTH_LAST)
    V4BF(EPI_POST0)
  }
#undef V4BF
}

// small levels: one fused launch per apply (env MPDE_SMALL_FUSED=1 enables; at C4 level 2 it
// took 22 us per apply against ~22 us for the two passes -- one CTA per PDE is too little parallelism)
static int g_small_fused = -1;
bool use_small_fused(const Geo& G, bool f64) {
  if (g_small_fused < 0) {
    const char* e = getenv("MPDE_SMALL_FUSED");
    g_small_fused = e ? atoi(e) : 0;  // opt-in: one CTA per PDE measured slower than the two passes
  }
  return g_small_fused && !f64 && G.P <= kSmallFusedP;
}

void launch_schur_small(int epi, const Geo& G, int nvec, int crep, const float* cf, const float* x,
                        const EpiArgs& A, const int* act, cudaStream_t s) {
  ++g_launch_count;
  const size_t smem = sizeof(float) * 2 * (size_t)G.P;
#define SMALL_CASE(E)                                                                             \
  case E:                                                                                         \
    DISPATCH_D2(G.D, (k_schur_small<DD, E><<<nvec, kSmallFusedThreads, smem, s>>>(G, cf, crep, x, A, act))); \
    break;
  switch (epi) {
    SMALL_CASE(EPI_STORE)
    SMALL_CASE(EPI_DOT)
    SMALL_CASE(EPI_POWER)
    SMALL_CASE(EPI_RESID)
    SMALL_CASE(EPI_SMOOTH)
    SMALL_CASE(EPI_SMOOTH_LAST)
    SMALL_CASE(EPI_POST0)
  }
#undef SMALL_CASE
}

void launch_schur_fused(int epi, const Geo& G, int nvec, int crep, const float* cf,
                        const float* x, const EpiArgs& A, const int* act, cudaStream_t s) {
  ++g_launch_count;
  const dim3 gr(G.n[1] / kFX, nvec);
  const int thr = (kFX + 4) * (G.n[2] / 4);
  const size_t smem = sizeof(float) * fused_smem_floats(G.n[2]);
#define FUSED_CASE(E)                                                                          \
  case E: {                                                                                    \
    static size_t attr = 0;                                                                    \
    if (smem > attr) {                                                                         \
      cudaFuncSetAttribute(k_schur_fused<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           (int)smem);                                                         \
      attr = smem;                                                                             \
    }                                                                                          \
    k_schur_fused<E><<<gr, thr, smem, s>>>(G, cf, crep, x, A, act);                            \
  } break;
  switch (epi) {
    FUSED_CASE(EPI_STORE)
    FUSED_CASE(EPI_DOT)
    FUSED_CASE(EPI_POWER)
    FUSED_CASE(EPI_RESID)
    FUSED_CASE(EPI_SMOOTH)
    FUSED_CASE(EPI_SMOOTH_LAST)
    FUSED_CASE(EPI_POST0)
  }
#undef FUSED_CASE
}

// Kernel variants that apply S on a level (mpde_hierarchy_query what = 5; the tests assert the
// selection so that a parity case really exercises the kernel it names):
//   out[0] pass 1 of the PCG operator, out[1] pass 2 of the PCG operator,
//   out[2] pass 2 of the V-cycle applies, out[3] 1 if those read bf16 coefficients.
// Codes: 0 scalar, 1 v4, 2 v4 warp-specialised, 3 t-blocked (runtime extents),
// 4 t-blocked (compile-time extents), 5 2x2-blocked, 6 smem tile, 7 fused, 8 pass 1 with y part,
// 9 one-kernel t-marching apply (march.cu), 10 one-CTA-per-vector fused apply (small levels),
// 11 one-launch t-slab cluster apply (slab.cu, mid-size levels).
static int pass2_kind(const Geo& G, bool f64) {
  if (use_fused(G, f64)) return 7;
  if (use_tile(G, f64)) return 6;
  if (use_b22(G, f64)) {
    if (block_mode() == 2) return 5;
    const bool ct = (G.n[1] == G.n[2]) && (G.n[2] == 32 || G.n[2] == 64 || G.n[2] == 128);
    return ct ? 4 : 3;
  }
  if (use_v4(G)) return use_remap(G) ? 2 : 1;
  return 0;
}
void schur_variants(const Geo& G, bool f64, bool bf16_level, int nvec, int32_t out[4]) {
  if (use_slab(G, f64) && !use_march(G, f64, nvec)) {  // one launch per apply, t-slab clusters
    out[0] = out[1] = out[2] = 11;
    out[3] = bf16_level ? 1 : 0;
    return;
  }
  if (use_small_fused(G, f64) && !use_march(G, f64, nvec)) {  // one launch per apply, fp32 cf
    out[0] = out[1] = out[2] = 10;
    out[3] = 0;
    return;
  }
  if (use_march(G, f64, nvec)) {  // one kernel for every apply; V-cycle applies read bf16 cf if kept
    out[0] = out[1] = out[2] = 9;
    out[3] = bf16_level ? 1 : 0;
    return;
  }
  out[0] = use_fused(G, f64) ? 7 : use_hy(G, f64) ? 8 : use_v4(G) ? 1 : 0;
  out[1] = pass2_kind(G, f64);
  const bool bf = bf16_level && schur_bf16_ok(G, f64);
  out[2] = bf ? (use_b22(G, false) ? pass2_kind(G, false) : (use_remap(G) ? 2 : 1)) : pass2_kind(G, f64);
  out[3] = bf ? 1 : 0;
}

void launch_diag_schur(const Geo& G, int B, const float* cf, float* dinv, cudaStream_t s) {
  ++g_launch_count;
  DISPATCH_D2(G.D, k_schur_diag<DD><<<grid2(G.P, B), kThreads, 0, s>>>(G, cf, dinv));
}

}  // namespace mpde
