// common.cuh -- device-side geometry, stencil tables and helpers shared by the
// NeuRLP-PDE kernels (B200 / sm_100a).  Nothing here is shared with oracle/.
//
// Operator (§3): for one PDE on a level with sizes n[d], steps h[d]:
//   equation rows   w_eq * sum_m c_m(p) z_m(p)                       (Eq. 3)
//   boundary rows   w_bnd * z_phi(p), p on any face                  (Eq. 4)
//   derivative rows w_der * (h^k z_dk(p) - sum_j a^k_j z_phi(p+o_j))  (Eq. 5)
//   smoothness rows w_sm * (z_phi(p) +- h z_d1(p) + h^2/2 z_d2(p) - z_phi(p +- e_d))
//                                                                   (Eqs. 6-7)
// Field order per PDE: phi, d0, d00, d1, d11, d2, d22 (field f = 1+2d+(k-1)).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Programmatic dependent launch (PDL).  Inside the PCG iteration graphs every kernel ->
// kernel edge is programmatic (mpde.cu, chunk_graph): a kernel's CTAs may be scheduled once
// every CTA of its predecessor has started, so its launch overlaps the predecessor's tail.
// Every kernel therefore first waits for its predecessor grid to complete and flush
// (griddepcontrol.wait -- before ANY memory access, so read-after-write and write-after-read
// both stay ordered), then lets its own dependents be scheduled.  Without PDL both
// instructions are no-ops.
#define MPDE_PDL_ENTRY() \
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

namespace mpde {

constexpr int kMaxD = 4;  // grid dims incl. time (mpde.h: ndim 2..4)
constexpr int kThreads = 256;
constexpr int kTabRow = 52;  // floats per (axis, index) row of the condensed-operator tables
constexpr int kTabKf = 0;   // row segments, 16-byte aligned: Kf [0,18), KT [20,38), P0 [40,51)
constexpr int kTabKT = 20;
constexpr int kTabP0 = 40;

// Per-level geometry, passed by value to every kernel.
struct Geo {
  int D;
  int n[kMaxD];
  int stride[kMaxD];
  int P;
  float h[kMaxD], h2[kMaxD];      // h, h^2 (fp32)
  double hd[kMaxD], h2d[kMaxD];   // h, h^2 (fp64)
  float we, wb, wr, ws;           // row-group weights
  const float* tab;               // device: per-axis row tables of S (schur.cu)
  int tab_off[kMaxD];             // offset of axis d's rows in tab
  // interior rows of the tables (identical for 7 <= i <= n-8), kept in the constant bank:
  // [0,10) Kf o=-2..2 x k, [10,20) KT o=-2..2 x k, [20,29) P0 o=-4..4
  float irow[kMaxD][32];
  // boundary types per face (mpde_problem.bc): 0 Dirichlet, 1 Neumann, 2 none;
  // nb2 = w_bnd^2 on the Neumann faces (the Neumann row's N_dd entry), 0 otherwise
  int bc[kMaxD][2];
  float nb2[kMaxD][2];
};

// point index i of axis d lies on a Dirichlet face (Eq. 4 rows; reading Q1 / B1)
__device__ __forceinline__ bool dir_face(const Geo& G, int d, int i) {
  return (i == 0 && G.bc[d][0] == 0) || (i == G.n[d] - 1 && G.bc[d][1] == 0);
}
// w_bnd^2 of the Neumann row(s) of the first-derivative variable along d at index i
__device__ __forceinline__ float neu_w2(const Geo& G, int d, int i) {
  return (i == 0 ? G.nb2[d][0] : 0.f) + (i == G.n[d] - 1 ? G.nb2[d][1] : 0.f);
}

// 5-point FD weights for the unit-spaced grid, per class and ascending offset.
// class 0,1: forward (offsets 0..4), 2: central (-2..2), 3,4: backward (-4..0).
// P:174 "5 point central differences and ... forward, backward finite differences at
// the edges" (reading Q4 in DESIGN.md).
// (the weight tables cA / cAd live in kernels.cu, the only translation unit using them)

__device__ __forceinline__ int fd_cls(int i, int n) {
  return i < 2 ? i : (i > n - 3 ? (i == n - 2 ? 3 : 4) : 2);
}
__device__ __forceinline__ int fd_start(int cls) { return cls < 2 ? 0 : (cls == 2 ? -2 : -4); }

// 2x2 block T_d(i) of N_dd from derivative + smoothness rows along axis d at index i:
//   T11 = wr^2 h^2 + ws^2 h^2 (f+b) + nb, T12 = ws^2 h^3/2 (f-b), T22 = wr^2 h^4 + ws^2 h^4/4 (f+b)
// with f = [i <= n-2] (forward row present), b = [i >= 1] (backward row present) and nb the
// w_bnd^2 of a Neumann row on the first-derivative variable (neu_w2).
template <typename T>
__device__ __forceinline__ void tinv(T h, T wr, T ws, bool f, bool b, T& t11, T& t12, T& t22,
                                     T nb = T(0)) {
  T h2 = h * h;
  T fb = T(f) + T(b), fmb = T(f) - T(b);
  T a11 = wr * wr * h2 + ws * ws * h2 * fb + nb;
  T a12 = ws * ws * h2 * h * T(0.5) * fmb;
  T a22 = wr * wr * h2 * h2 + ws * ws * h2 * h2 * T(0.25) * fb;
  T det = a11 * a22 - a12 * a12;
  T id = T(1) / det;
  t11 = a22 * id;
  t12 = -a12 * id;
  t22 = a11 * id;
}

template <int D>
__device__ __forceinline__ void unravel(const Geo& G, int p, int* idx) {
  if (D == 2) {
    idx[0] = p / G.n[1];
    idx[1] = p - idx[0] * G.n[1];
  } else if (D == 3) {
    int nn = G.n[1] * G.n[2];
    idx[0] = p / nn;
    int r = p - idx[0] * nn;
    idx[1] = r / G.n[2];
    idx[2] = r - idx[1] * G.n[2];
  } else {
#pragma unroll
    for (int d = D - 1; d > 0; --d) {
      const int q = p / G.n[d];
      idx[d] = p - q * G.n[d];
      p = q;
    }
    idx[0] = p;
  }
}

// the point carries a Dirichlet row: it lies on at least one Dirichlet face
template <int D>
__device__ __forceinline__ bool on_boundary(const Geo& G, const int* idx) {
  bool onb = false;
#pragma unroll
  for (int d = 0; d < D; ++d) onb |= dir_face(G, d, idx[d]);
  return onb;
}

// Prolongation weight P[i, I] along one axis, fine size nf -> coarse size nc.
// Even nf: cell-centred linear interpolation (3/4, 1/4) with constant end
// extrapolation; odd nf: vertex-centred (1 | 1/2,1/2); nc == nf: identity.
// P:272 / P:278 ("linear interpolation"), reading Q10.
__device__ __forceinline__ float pw(int i, int I, int nf, int nc) {
  if (nc == nf) return i == I ? 1.f : 0.f;
  if ((nf & 1) == 0) {
    int Ii = i >> 1;
    int J = (i & 1) ? Ii + 1 : Ii - 1;
    J = J < 0 ? 0 : (J > nc - 1 ? nc - 1 : J);
    float w = 0.f;
    if (I == Ii) w += 0.75f;
    if (I == J) w += 0.25f;
    return w;
  }
  if ((i & 1) == 0) return (I == (i >> 1)) ? 1.f : 0.f;
  return (I == (i >> 1) || I == (i >> 1) + 1) ? 0.5f : 0.f;
}

// Block-wide sum of a double; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    v = l < nw ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

}  // namespace mpde
