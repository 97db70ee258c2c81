// dense.cu -- coarsest-level exact solve ("solve for the exact error", Alg. 1):
// batched in-place blocked Gauss-Jordan inversion of the SPD coarse operators S_c (fp64,
// 32-column panels, no pivoting -- S_c is SPD), then a symmetrised fp32 copy applied by a
// batched GEMV in every V-cycle.
//
// Block step K (P = A_KK^-1):  A_Kj <- P A_Kj (j != K);  A_ij -= A_iK A_Kj (i, j != K);
//                              A_iK <- -A_iK P (i != K);  A_KK <- P.
#include "common.cuh"
#include "internal.h"

namespace mpde {

constexpr int NB = 32;

// symmetrise the probed columns: a = (Y + Y^T)/2, Y[j] = S_c e_j
__global__ void k_gj_init(int n, const float* __restrict__ cols, double* __restrict__ a) {
  MPDE_PDL_ENTRY();
  const int b = blockIdx.z;
  const int i = blockIdx.y * 32 + threadIdx.y, j = blockIdx.x * 32 + threadIdx.x;
  if (i >= n || j >= n) return;
  const float* cb = cols + (size_t)b * n * n;
  a[(size_t)b * n * n + (size_t)i * n + j] =
      0.5 * (double(cb[(size_t)j * n + i]) + double(cb[(size_t)i * n + j]));
}

__global__ void __launch_bounds__(1024) k_gj_diag(int n, int k0, double* __restrict__ a) {
  MPDE_PDL_ENTRY();
  __shared__ double M[NB][NB + 1];
  const int b = blockIdx.x, ty = threadIdx.y, tx = threadIdx.x;
  const int kb = min(NB, n - k0);
  double* A = a + (size_t)b * n * n;
  if (ty < kb && tx < kb) M[ty][tx] = A[(size_t)(k0 + ty) * n + k0 + tx];
  for (int k = 0; k < kb; ++k) {
    __syncthreads();
    const double piv = 1.0 / M[k][k];
    const double rk = (tx < kb) ? M[k][tx] * piv : 0.0;
    const double ck = (ty < kb) ? M[ty][k] : 0.0;
    const double old = (ty < kb && tx < kb) ? M[ty][tx] : 0.0;
    __syncthreads();
    if (ty < kb && tx < kb) {
      double v;
      if (ty == k)
        v = (tx == k) ? piv : rk;
      else
        v = (tx == k) ? -ck * piv : old - ck * rk;
      M[ty][tx] = v;
    }
  }
  __syncthreads();
  if (ty < kb && tx < kb) A[(size_t)(k0 + ty) * n + k0 + tx] = M[ty][tx];
}

// mode 0: row panel   A_Kj <- P A_Kj          (grid.x = column blocks)
// mode 1: column panel A_iK <- -A_iK P        (grid.x = row blocks)
__global__ void __launch_bounds__(1024) k_gj_panel(int n, int k0, int mode, double* __restrict__ a) {
  MPDE_PDL_ENTRY();
  __shared__ double Pm[NB][NB + 1];
  __shared__ double T[NB][NB + 1];
  const int b = blockIdx.y, ty = threadIdx.y, tx = threadIdx.x;
  const int kb = min(NB, n - k0);
  const int o0 = blockIdx.x * NB;
  if (o0 == k0) return;
  double* A = a + (size_t)b * n * n;
  const int ob = min(NB, n - o0);
  if (ty < kb && tx < kb) Pm[ty][tx] = A[(size_t)(k0 + ty) * n + k0 + tx];
  if (mode == 0) {
    if (ty < kb && tx < ob) T[ty][tx] = A[(size_t)(k0 + ty) * n + o0 + tx];
  } else {
    if (ty < ob && tx < kb) T[ty][tx] = A[(size_t)(o0 + ty) * n + k0 + tx];
  }
  __syncthreads();
  if (mode == 0) {
    if (ty < kb && tx < ob) {
      double s = 0.0;
      for (int k = 0; k < kb; ++k) s += Pm[ty][k] * T[k][tx];
      A[(size_t)(k0 + ty) * n + o0 + tx] = s;
    }
  } else {
    if (ty < ob && tx < kb) {
      double s = 0.0;
      for (int k = 0; k < kb; ++k) s += T[ty][k] * Pm[k][tx];
      A[(size_t)(o0 + ty) * n + k0 + tx] = -s;
    }
  }
}

// trailing update A_ij -= A_iK A_Kj for i, j != K (A_Kj already scaled by P)
__global__ void __launch_bounds__(1024) k_gj_trail(int n, int k0, double* __restrict__ a) {
  MPDE_PDL_ENTRY();
  __shared__ double L[NB][NB + 1];
  __shared__ double R[NB][NB + 1];
  const int b = blockIdx.z, ty = threadIdx.y, tx = threadIdx.x;
  const int i0 = blockIdx.y * NB, j0 = blockIdx.x * NB;
  if (i0 == k0 || j0 == k0) return;
  const int kb = min(NB, n - k0);
  double* A = a + (size_t)b * n * n;
  const int i = i0 + ty, j = j0 + tx;
  L[ty][tx] = (i < n && tx < kb) ? A[(size_t)i * n + k0 + tx] : 0.0;
  R[ty][tx] = (ty < kb && j < n) ? A[(size_t)(k0 + ty) * n + j] : 0.0;
  __syncthreads();
  if (i < n && j < n) {
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < NB; ++k) s += L[ty][k] * R[k][tx];
    A[(size_t)i * n + j] -= s;
  }
}

__global__ void k_gj_final(int n, const double* __restrict__ a, float* __restrict__ inv) {
  MPDE_PDL_ENTRY();
  const int b = blockIdx.z;
  const int i = blockIdx.y * 32 + threadIdx.y, j = blockIdx.x * 32 + threadIdx.x;
  if (i >= n || j >= n) return;
  const double* A = a + (size_t)b * n * n;
  inv[(size_t)b * n * n + (size_t)i * n + j] =
      float(0.5 * (A[(size_t)i * n + j] + A[(size_t)j * n + i]));
}

void launch_coarse_invert(int n, int B, const float* cols, double* scratch, float* inv,
                          cudaStream_t s) {
  const int nbk = (n + NB - 1) / NB;
  const dim3 t(32, 32);
  g_launch_count += 2 + 4 * (size_t)nbk;
  k_gj_init<<<dim3(nbk, nbk, B), t, 0, s>>>(n, cols, scratch);
  for (int K = 0; K < nbk; ++K) {
    const int k0 = K * NB;
    k_gj_diag<<<B, t, 0, s>>>(n, k0, scratch);
    k_gj_panel<<<dim3(nbk, B), t, 0, s>>>(n, k0, 0, scratch);
    k_gj_trail<<<dim3(nbk, nbk, B), t, 0, s>>>(n, k0, scratch);
    k_gj_panel<<<dim3(nbk, B), t, 0, s>>>(n, k0, 1, scratch);
  }
  k_gj_final<<<dim3(nbk, nbk, B), t, 0, s>>>(n, scratch, inv);
}

// e = S_c^-1 r on the coarsest level: one warp per (row, vector), float4 over the row;
// optional partial <rdot, e> per CTA.
__global__ void __launch_bounds__(256) k_coarse_gemv4(int n, const float* __restrict__ sinv,
                                                     const float* __restrict__ r, float* e,
                                                     const float* rdot, double* part,
                                                     const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y;
  if (act && !act[v]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  const float* S = sinv + (size_t)v * n * n;
  const float* rv = r + (size_t)v * n;
  double dot = 0.0;
  if (row < n) {
    float acc = 0.f;
    if ((n & 3) == 0) {
      const float4* Sr = reinterpret_cast<const float4*>(S + (size_t)row * n);
      const float4* r4 = reinterpret_cast<const float4*>(rv);
      for (int j = lane; j < n / 4; j += 32) {
        const float4 m = Sr[j], x = r4[j];
        acc += m.x * x.x + m.y * x.y + m.z * x.z + m.w * x.w;
      }
    } else {
      for (int j = lane; j < n; j += 32) acc += S[(size_t)row * n + j] * rv[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      e[(size_t)v * n + row] = acc;
      if (rdot) dot = double(rdot[(size_t)v * n + row]) * acc;
    }
  }
  if (part) {
    dot = block_sum(dot);
    if (threadIdx.x == 0) part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

int coarse_gemv_blocks(int n) { return (n + 7) / 8; }

// ---------------------------------------------------------------------------------
// Grid transfers of scalar fields (the V-cycle hot path).  P:278 "linear interpolation";
// R = P^T / 2^(coarsened dims) (reading Q12).  Per axis, coarse I gathers fine
// 2I-1 .. 2I+2 (even n, cell-centred 1/4,3/4,3/4,1/4 with constant end extrapolation),
// 2I-1 .. 2I+1 (odd n, vertex-centred 1/2,1,1/2) or I itself (axis not coarsened).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void restrict_axis(int I, int nf, int nc, int* f, float* w) {
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    f[a] = 0;
    w[a] = 0.f;
  }
  if (nc == nf) {
    f[0] = I;
    w[0] = 1.f;
    return;
  }
  if (nf & 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int i = 2 * I - 1 + a;
      if (i >= 0 && i < nf) {
        f[a] = i;
        w[a] = 0.5f * (a == 1 ? 1.f : 0.5f);
      }
    }
    return;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = 2 * I - 1 + a;
    if (i < 0 || i >= nf) continue;
    // P[i, I]: i = 2I or 2I+1 -> 3/4 (+1/4 if its other neighbour is clamped onto I);
    // i = 2I-1 or 2I+2 -> 1/4
    float p = (a == 1 || a == 2) ? 0.75f : 0.25f;
    if (a == 1 && I == 0) p = 1.f;          // fine 0: 3/4 I + 1/4 clamp(I-1)=I
    if (a == 2 && I == nc - 1) p = 1.f;     // fine nf-1: 3/4 I + 1/4 clamp(I+1)=I
    f[a] = i;
    w[a] = 0.5f * p;
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_restrict1(Geo Gf, Geo Gc, const float* __restrict__ fine,
                                                  float* __restrict__ coarse, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y, Pc = Gc.P, Pf = Gf.P;
  if (act && !act[v]) return;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= Pc) return;
  int cidx[D];
  unravel<D>(Gc, I, cidx);
  int f[D][4];
  float w[D][4];
#pragma unroll
  for (int d = 0; d < D; ++d) restrict_axis(cidx[d], Gf.n[d], Gc.n[d], f[d], w[d]);
  const float* fb = fine + (size_t)v * Pf;
  float acc = 0.f;
  if (D == 2) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (w[0][a] == 0.f) continue;
      const float* row = fb + f[0][a] * Gf.stride[0];
      float s = 0.f;
#pragma unroll
      for (int b = 0; b < 4; ++b) s += w[D - 1][b] * __ldg(row + f[D - 1][b]);
      acc += w[0][a] * s;
    }
  } else if (D == 3) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (w[0][a] == 0.f) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (w[1][b] == 0.f) continue;
        const float* row = fb + f[0][a] * Gf.stride[0] + f[1][b] * Gf.stride[1];
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) s += w[2][c] * __ldg(row + f[2][c]);
        acc += w[0][a] * w[1][b] * s;
      }
    }
  } else {  // 4D: the same tensor-product full weighting over the fourth axis
    for (int a = 0; a < 4; ++a) {
      if (w[0][a] == 0.f) continue;
      for (int b = 0; b < 4; ++b) {
        if (w[1][b] == 0.f) continue;
        for (int c = 0; c < 4; ++c) {
          if (w[2][c] == 0.f) continue;
          const float* row = fb + f[0][a] * Gf.stride[0] + f[1][b] * Gf.stride[1] + f[2][c] * Gf.stride[2];
          float s = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) s += w[D - 1][e] * __ldg(row + f[D - 1][e]);
          acc += w[0][a] * w[1][b] * w[2][c] * s;
        }
      }
    }
  }
  coarse[(size_t)v * Pc + I] = acc;
}

// prolongation: fine point i_d -> coarse (I0, w0), (I1, w1) per axis
__device__ __forceinline__ void prolong_axis(int i, int nf, int nc, int& I0, int& I1, float& w0,
                                             float& w1) {
  if (nf == nc) {
    I0 = I1 = i;
    w0 = 1.f;
    w1 = 0.f;
  } else if ((nf & 1) == 0) {
    const int Ii = i >> 1;
    int J = (i & 1) ? Ii + 1 : Ii - 1;
    J = J < 0 ? 0 : (J > nc - 1 ? nc - 1 : J);
    I0 = Ii;
    I1 = J;
    w0 = 0.75f;
    w1 = 0.25f;
  } else if ((i & 1) == 0) {
    I0 = I1 = i >> 1;
    w0 = 1.f;
    w1 = 0.f;
  } else {
    I0 = i >> 1;
    I1 = (i >> 1) + 1;
    w0 = w1 = 0.5f;
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_prolong1(Geo Gf, Geo Gc, const float* __restrict__ coarse,
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
  for (int d = 0; d < D; ++d) prolong_axis(idx[d], Gf.n[d], Gc.n[d], I0[d], I1[d], w0[d], w1[d]);
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
    if (w != 0.f) acc += w * __ldg(cb + off);
  }
  fine[(size_t)v * Pf + p] = acc;
}

// Quad versions (4 consecutive points of the last axis per thread, float4 stores): the
// weights of the non-last axes are computed once per quad and the last-axis taps come from
// a small window with static offsets (same arithmetic as the scalar kernels above).
template <int D>
__global__ void __launch_bounds__(256) k_restrict1q(Geo Gf, Geo Gc, const float* __restrict__ fine,
                                                   float* __restrict__ coarse, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y, Pc = Gc.P, Pf = Gf.P;
  if (act && !act[v]) return;
  const int I0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (I0 >= Pc) return;
  int cidx[D];
  unravel<D>(Gc, I0, cidx);
  constexpr int L = D - 1;
  const int nfy = Gf.n[L], ncy = Gc.n[L], Yq = cidx[L];  // Yq = 4 * quad index
  int f[D - 1][4];
  float w[D - 1][4];
#pragma unroll
  for (int d = 0; d < D - 1; ++d) restrict_axis(cidx[d], Gf.n[d], Gc.n[d], f[d], w[d]);
  float wy[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int fj[4];
    restrict_axis(Yq + j, nfy, ncy, fj, wy[j]);
  }
  const float* fb = fine + (size_t)v * Pf;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const bool ycoarse = nfy != ncy;
  const int ylo = 2 * Yq - 4;  // window fine y ylo .. ylo+15 (coarsened y)
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    if (w[0][a] == 0.f) continue;
#pragma unroll
    for (int b = 0; b < (D == 3 ? 4 : 1); ++b) {
      float wab = w[0][a];
      const float* row = fb + (size_t)f[0][a] * Gf.stride[0];
      if (D == 3) {
        if (w[D - 2][b] == 0.f) continue;
        wab *= w[D - 2][b];
        row += (size_t)f[D - 2][b] * Gf.stride[D - 2];
      }
      if (ycoarse) {
        float win[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int y = ylo + 4 * k;
          const float4 t = (y >= 0 && y < nfy) ? *reinterpret_cast<const float4*>(row + y)
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
          win[4 * k] = t.x; win[4 * k + 1] = t.y; win[4 * k + 2] = t.z; win[4 * k + 3] = t.w;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // fine 2(Yq+j)-1+c = ylo + 2j + 3 + c
          float sy = 0.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) sy += wy[j][c] * win[2 * j + 3 + c];
          acc[j] += wab * sy;
        }
      } else {
        const float4 t = *reinterpret_cast<const float4*>(row + Yq);
        acc[0] += wab * t.x; acc[1] += wab * t.y; acc[2] += wab * t.z; acc[3] += wab * t.w;
      }
    }
  }
  *reinterpret_cast<float4*>(coarse + (size_t)v * Pc + I0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
}

template <int D>
__global__ void __launch_bounds__(256) k_prolong1q(Geo Gf, Geo Gc, const float* __restrict__ coarse,
                                                  float* __restrict__ fine, const int* act) {
  MPDE_PDL_ENTRY();
  const int v = blockIdx.y, Pf = Gf.P, Pc = Gc.P;
  if (act && !act[v]) return;
  const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (p0 >= Pf) return;
  int idx[D];
  unravel<D>(Gf, p0, idx);
  constexpr int L = D - 1;
  const int nfy = Gf.n[L], ncy = Gc.n[L], y0 = idx[L];
  int I0[D - 1], I1[D - 1];
  float w0[D - 1], w1[D - 1];
#pragma unroll
  for (int d = 0; d < D - 1; ++d) prolong_axis(idx[d], Gf.n[d], Gc.n[d], I0[d], I1[d], w0[d], w1[d]);
  const float* cb = coarse + (size_t)v * Pc;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int q2 = y0 >> 1;  // 2q
#pragma unroll
  for (int mask = 0; mask < (1 << (D - 1)); ++mask) {
    float w = 1.f;
    int off = 0;
#pragma unroll
    for (int d = 0; d < D - 1; ++d) {
      const bool hi = (mask >> d) & 1;
      w *= hi ? w1[d] : w0[d];
      off += (hi ? I1[d] : I0[d]) * Gc.stride[d];
    }
    if (w == 0.f) continue;
    const float* row = cb + off;
    if (nfy == ncy) {
      const float4 t = *reinterpret_cast<const float4*>(row + y0);
      acc[0] += w * t.x; acc[1] += w * t.y; acc[2] += w * t.z; acc[3] += w * t.w;
    } else if ((nfy & 1) == 0) {  // cell-centred: window 2q-1 .. 2q+2, clamped
      const float c0 = __ldg(row + max(q2 - 1, 0)), c1 = __ldg(row + q2);
      const float c2 = __ldg(row + min(q2 + 1, ncy - 1)), c3 = __ldg(row + min(q2 + 2, ncy - 1));
      acc[0] += w * (0.75f * c1 + 0.25f * c0);
      acc[1] += w * (0.75f * c1 + 0.25f * c2);
      acc[2] += w * (0.75f * c2 + 0.25f * c1);
      acc[3] += w * (0.75f * c2 + 0.25f * c3);
    } else {  // vertex-centred: window 2q .. 2q+2
      const float c0 = __ldg(row + q2), c1 = __ldg(row + min(q2 + 1, ncy - 1));
      const float c2 = __ldg(row + min(q2 + 2, ncy - 1));
      acc[0] += w * c0;
      acc[1] += w * 0.5f * (c0 + c1);
      acc[2] += w * c1;
      acc[3] += w * 0.5f * (c1 + c2);
    }
  }
  *reinterpret_cast<float4*>(fine + (size_t)v * Pf + p0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
}

// quad kernels need the last axis % 4 == 0 on the output side (and on the fine side for the
// restriction's float4 window)
static inline bool transfer_quads(const Geo& Gf, const Geo& Gc) {
  const int L = Gf.D - 1;
  return Gf.D <= 3 && (Gf.n[L] % 4 == 0) && (Gc.n[L] % 4 == 0);  // 4D: the generic kernels
}

void launch_restrict1(const Geo& Gf, const Geo& Gc, int nvec, const float* fine, float* coarse,
                      const int* act, cudaStream_t s) {
  ++g_launch_count;
  if (transfer_quads(Gf, Gc)) {
    const dim3 gq((Gc.P / 4 + 255) / 256, nvec);
    if (Gf.D == 2)
      k_restrict1q<2><<<gq, 256, 0, s>>>(Gf, Gc, fine, coarse, act);
    else
      k_restrict1q<3><<<gq, 256, 0, s>>>(Gf, Gc, fine, coarse, act);
    return;
  }
  const dim3 g((Gc.P + 255) / 256, nvec);
  if (Gf.D == 2)
    k_restrict1<2><<<g, 256, 0, s>>>(Gf, Gc, fine, coarse, act);
  else if (Gf.D == 4)
    k_restrict1<4><<<g, 256, 0, s>>>(Gf, Gc, fine, coarse, act);
  else
    k_restrict1<3><<<g, 256, 0, s>>>(Gf, Gc, fine, coarse, act);
}

void launch_prolong1(const Geo& Gf, const Geo& Gc, int nvec, const float* coarse, float* fine,
                     const int* act, cudaStream_t s) {
  ++g_launch_count;
  if (transfer_quads(Gf, Gc)) {
    const dim3 gq((Gf.P / 4 + 255) / 256, nvec);
    if (Gf.D == 2)
      k_prolong1q<2><<<gq, 256, 0, s>>>(Gf, Gc, coarse, fine, act);
    else
      k_prolong1q<3><<<gq, 256, 0, s>>>(Gf, Gc, coarse, fine, act);
    return;
  }
  const dim3 g((Gf.P + 255) / 256, nvec);
  if (Gf.D == 2)
    k_prolong1<2><<<g, 256, 0, s>>>(Gf, Gc, coarse, fine, act);
  else if (Gf.D == 4)
    k_prolong1<4><<<g, 256, 0, s>>>(Gf, Gc, coarse, fine, act);
  else
    k_prolong1<3><<<g, 256, 0, s>>>(Gf, Gc, coarse, fine, act);
}

void launch_coarse_gemv(int n, int nvec, const float* sinv, const float* r, float* e,
                        const float* rdot, double* part, const int* act, cudaStream_t s) {
  ++g_launch_count;
  k_coarse_gemv4<<<dim3(coarse_gemv_blocks(n), nvec), 256, 0, s>>>(n, sinv, r, e, rdot, part, act);
}

}  // namespace mpde
