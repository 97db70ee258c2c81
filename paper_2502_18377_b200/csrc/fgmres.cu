// fgmres.cu -- FGMRES(m) on the condensed system S x = rt with the V-cycle as the (right,
// flexible) preconditioner: the paper's own Krylov method ("FGMRES with a multigrid
// preconditioner").  Batched over independent PDEs (blockIdx.y = PDE);
// every PDE keeps its own Arnoldi basis, Hessenberg matrix and Givens rotations.
//
// Per Arnoldi step j (Saad, flexible GMRES):  Z_j = V(V_j);  w = S Z_j;
//   classical Gram-Schmidt with one re-orthogonalisation (CGS2):  h_ij = <w, V_i>,
//   w -= sum_i h_ij V_i  (twice, the coefficients summed into H);  h_{j+1,j} = ||w||;
//   V_{j+1} = w / h_{j+1,j};  Givens rotations keep |g_{j+1}| = ||rt - S x_j|| (the true,
//   unpreconditioned residual: right preconditioning).
// End of a cycle: R y = g (back substitution), x += sum_i y_i Z_i;  restart from
// r = rt - S x.  Dot products are fp64 partial sums per (PDE, tile), reduced in a fixed
// order (deterministic).
#include <cuda_runtime.h>

#include "internal.h"

namespace mpde {

constexpr int kGmTile = 2048;  // points per CTA of the Arnoldi vector kernels (256 x 2 float4)

int gm_tiles(int P) { return (P + kGmTile - 1) / kGmTile; }

// P % 4 == 0 is not required: the vector kernels handle the tail point by point.
__device__ __forceinline__ double gm_block_sum(double v) { return block_sum(v); }

// part[(v * (m+1) + i) * nt + tile] = <w_v, V_i,v> over the tile, i < j1.  Each thread keeps
// its kGmTile / kThreads points of w in registers; every V_i is read once (coalesced), its
// per-thread partial reduced by warp shuffles into smem [warp][i]; one barrier at the end.
__global__ void __launch_bounds__(kThreads) k_gm_mdot(int P, int j1, int m1, const float* V,
                                                      size_t BP, const float* w, double* part,
                                                      const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int kPer = kGmTile / kThreads;
  __shared__ double red[kThreads / 32][33];
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int nt = gridDim.x;
  const int p0 = blockIdx.x * kGmTile + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* wv = w + (size_t)v * P;
  float wr[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int p = p0 + k * kThreads;
    wr[k] = p < P ? wv[p] : 0.f;
  }
  for (int i = 0; i < j1; ++i) {
    const float* Vi = V + i * BP + (size_t)v * P;
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int p = p0 + k * kThreads;
      if (p < P) d += double(wr[k]) * double(Vi[p]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) red[warp][i] = d;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < j1; i += kThreads) {
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < kThreads / 32; ++k) d += red[k][i];
    part[((size_t)v * m1 + i) * nt + blockIdx.x] = d;
  }
}

// w -= sum_{i < j1} coef[v][i] V_i ; part[(v*(m+1)) * nt + tile] = ||w||^2 over the tile.
// w stays in registers (kPer points per thread); per basis vector one coefficient load and
// kPer independent coalesced loads (memory-level parallelism instead of a per-point chain).
__global__ void __launch_bounds__(kThreads) k_gm_update(int P, int j1, int m1, const float* V,
                                                        size_t BP, const double* coef, float* w,
                                                        double* part, const int* act) {
  MPDE_PDL_ENTRY();
  constexpr int kPer = kGmTile / kThreads;
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int nt = gridDim.x;
  const int p0 = blockIdx.x * kGmTile + threadIdx.x;
  float* wv = w + (size_t)v * P;
  const double* cv = coef + (size_t)v * m1;
  float a[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int p = p0 + k * kThreads;
    a[k] = p < P ? wv[p] : 0.f;
  }
  for (int i = 0; i < j1; ++i) {
    const float c = float(cv[i]);
    const float* Vi = V + i * BP + (size_t)v * P;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int p = p0 + k * kThreads;
      if (p < P) a[k] -= c * Vi[p];
    }
  }
  double d = 0.0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int p = p0 + k * kThreads;
    if (p < P) {
      wv[p] = a[k];
      d += double(a[k]) * a[k];
    }
  }
  d = gm_block_sum(d);
  if (threadIdx.x == 0) part[(size_t)v * m1 * nt + blockIdx.x] = d;
}

// y = sc[v] * y  (sc = 1/||.||; 0 for a finished PDE)
__global__ void __launch_bounds__(kThreads) k_gm_scale(int P, const float* sc, float* y,
                                                       const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) y[(size_t)v * P + p] *= sc[v];
}

// y = rt - y (y holds S x), or y = rt when first; part = ||y||^2 per tile
__global__ void __launch_bounds__(kThreads) k_gm_resid(int P, int m1, const float* rt, float* y,
                                                       int first, double* part, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int nt = gridDim.x;
  const int p0 = blockIdx.x * kGmTile;
  const int p1 = min(P, p0 + kGmTile);
  double d = 0.0;
  for (int p = p0 + threadIdx.x; p < p1; p += kThreads) {
    const size_t o = (size_t)v * P + p;
    const float a = first ? rt[o] : rt[o] - y[o];
    y[o] = a;
    d += double(a) * a;
  }
  d = gm_block_sum(d);
  if (threadIdx.x == 0) part[(size_t)v * m1 * nt + blockIdx.x] = d;
}

// x += sum_{i < k[v]} y_i Z_i  for the PDEs of the cycle (gact); register tile as k_gm_update
__global__ void __launch_bounds__(kThreads) k_gm_xupdate(int P, int m1, const float* Z, size_t BP,
                                                         const double* y, const int* k, float* x,
                                                         const int* gact) {
  MPDE_PDL_ENTRY();
  constexpr int kPer = kGmTile / kThreads;
  const int v = blockIdx.y;
  if (!gact[v]) return;
  const int p0 = blockIdx.x * kGmTile + threadIdx.x;
  const int kv = k[v];
  const double* yv = y + (size_t)v * m1;
  float* xv = x + (size_t)v * P;
  float a[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int p = p0 + q * kThreads;
    a[q] = p < P ? xv[p] : 0.f;
  }
  for (int i = 0; i < kv; ++i) {
    const float c = float(yv[i]);
    const float* Zi = Z + i * BP + (size_t)v * P;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int p = p0 + q * kThreads;
      if (p < P) a[q] += c * Zi[p];
    }
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int p = p0 + q * kThreads;
    if (p < P) xv[p] = a[q];
  }
}

// one CTA per PDE: warps reduce the per-tile partials of the j1 values (fixed order), thread 0
// runs the per-PDE FGMRES logic.
__global__ void __launch_bounds__(kThreads) k_gm_scalar(int op, int j, int m, int nt, PdeState st,
                                                        GmState g, const double* part, float tol2,
                                                        int max_iters) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.x;
  const int m1 = m + 1;
  __shared__ double red[33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nval = (op == GM_DOTS0 || op == GM_DOTS1) ? j + 1 : 1;
  const bool need = op != GM_SOLVE && st.act[v];
  if (need && part) {
    for (int i = warp; i < nval; i += kThreads / 32) {
      double s = 0.0;
      for (int t = lane; t < nt; t += 32) s += part[((size_t)v * m1 + i) * nt + t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[i] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double* H = g.H + (size_t)v * m1 * m;  // H[i * m + col]
  double* gv = g.g + (size_t)v * m1;
  double* cs = g.cs + (size_t)v * m;
  double* sn = g.sn + (size_t)v * m;
  double* cf = g.coef + (size_t)v * m1;
  auto fail = [&](double val) {
    st.status[v] = isfinite(val) ? MPDE_STATUS_INDEFINITE : MPDE_STATUS_NONFINITE;
    st.failed[v] = 1;
    st.act[v] = 0;
  };
  if (op == GM_BEGIN || op == GM_RESTART) {
    if (!st.act[v]) {
      g.gact[v] = 0;
      return;
    }
    const double rr = red[0];
    if (op == GM_BEGIN) st.rr0[v] = rr;
    const double nrm = sqrt(rr);
    g.k[v] = 0;
    if (!(nrm > 0.0)) {
      if (isfinite(nrm)) st.act[v] = 0; else fail(nrm);
      g.gact[v] = 0;
      g.scl[v] = 0.f;
      return;
    }
    gv[0] = nrm;
    g.scl[v] = float(1.0 / nrm);
    g.gact[v] = 1;
    return;
  }
  if (op == GM_DOTS0 || op == GM_DOTS1) {
    if (!st.act[v]) return;
    for (int i = 0; i <= j; ++i) {
      cf[i] = red[i];
      H[i * m + j] = (op == GM_DOTS0 ? 0.0 : H[i * m + j]) + red[i];
    }
    return;
  }
  if (op == GM_NORM) {
    if (!st.act[v]) return;
    const double hn = sqrt(red[0]);
    if (!isfinite(hn)) {
      fail(hn);
      return;  // k stays j: the broken column is not used
    }
    for (int i = 0; i < j; ++i) {  // previous rotations
      const double a = H[i * m + j], b = H[(i + 1) * m + j];
      H[i * m + j] = cs[i] * a + sn[i] * b;
      H[(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
    }
    const double a = H[j * m + j], b = hn;
    const double r = sqrt(a * a + b * b);
    if (!(r > 0.0)) {  // S Z_j in span(V_0..V_{j-1}) with a zero projection: breakdown
      fail(r);
      return;
    }
    cs[j] = a / r;
    sn[j] = b / r;
    H[j * m + j] = r;
    H[(j + 1) * m + j] = 0.0;
    gv[j + 1] = -sn[j] * gv[j];
    gv[j] = cs[j] * gv[j];
    g.k[v] = j + 1;
    st.iters[v] += 1;
    st.pass_iters[v] += 1;
    const double res2 = gv[j + 1] * gv[j + 1];
    const double t2 = st.refines[v] >= 2 ? (double)st.tol2_later : (double)tol2;
    if (res2 <= t2 * st.rr0[v] || st.pass_iters[v] >= max_iters || hn == 0.0 ||
        res2 <= 0.25 * (double)st.tol * st.tol * st.rhsn[v] * st.rhsn[v])
      st.act[v] = 0;  // converged (or happy breakdown / iteration cap): x updated at cycle end
    g.scl[v] = hn > 0.0 ? float(1.0 / hn) : 0.f;
    return;
  }
  if (op == GM_SOLVE) {  // R y = g, R = the rotated Hessenberg's upper triangle
    if (!g.gact[v]) return;
    const int k = g.k[v];
    for (int i = k - 1; i >= 0; --i) {
      double s = gv[i];
      for (int l = i + 1; l < k; ++l) s -= H[i * m + l] * cf[l];
      cf[i] = s / H[i * m + i];
    }
    return;
  }
}

void launch_gm_mdot(int P, int B, int j1, int m, const float* V, const float* w, double* part,
                    const int* act, cudaStream_t s) {
  ++g_launch_count;
  k_gm_mdot<<<dim3(gm_tiles(P), B), kThreads, 0, s>>>(P, j1, m + 1, V, (size_t)B * P, w, part, act);
}
void launch_gm_update(int P, int B, int j1, int m, const float* V, const double* coef, float* w,
                      double* part, const int* act, cudaStream_t s) {
  ++g_launch_count;
  k_gm_update<<<dim3(gm_tiles(P), B), kThreads, 0, s>>>(P, j1, m + 1, V, (size_t)B * P, coef, w,
                                                       part, act);
}
void launch_gm_scale(int P, int B, const float* sc, float* y, const int* act, cudaStream_t s) {
  ++g_launch_count;
  k_gm_scale<<<dim3((P + kThreads - 1) / kThreads, B), kThreads, 0, s>>>(P, sc, y, act);
}
void launch_gm_resid(int P, int B, int m, const float* rt, float* y, int first, double* part,
                     const int* act, cudaStream_t s) {
  ++g_launch_count;
  k_gm_resid<<<dim3(gm_tiles(P), B), kThreads, 0, s>>>(P, m + 1, rt, y, first, part, act);
}
void launch_gm_xupdate(int P, int B, int m, const float* Z, const GmState& g, float* x,
                       cudaStream_t s) {
  ++g_launch_count;
  k_gm_xupdate<<<dim3(gm_tiles(P), B), kThreads, 0, s>>>(
      P, m + 1, Z, (size_t)B * P, g.coef, g.k, x, g.gact);
}
void launch_gm_scalar(int op, int j, int m, int P, int B, const PdeState& st, const GmState& g,
                      const double* part, float tol2, int max_iters, cudaStream_t s) {
  ++g_launch_count;
  k_gm_scalar<<<B, kThreads, 0, s>>>(op, j, m, gm_tiles(P), st, g, part, tol2, max_iters);
}

}  // namespace mpde
