// slab.cu -- the condensed operator S applied in ONE launch on mid-size 3D levels (a t-x-y grid
// whose x-y plane has <= 1024 points, e.g. the (16,32,32) level of C4 and the (32,32,32) fine
// level of C3), B200 / sm_100a.
//
// Operator (schur.cu header; Eq. 9 P:193-196 condensed onto u_phi):
//   h(p) = (1/sigma)(sigma alpha x - sum_d u~_d . (K_d x)(p))
//   S x  = sum_d P0_d x - sum_d K_d^T (u~_d h) + sigma alpha h + w_bnd^2 [p Dirichlet] x
// The two-pass kernels need two launches of ~0.5 M points on these levels and run at 12-15% of
// HBM bandwidth (round-2 kernel table: 9.5 + 20 us per apply at C4 level 1), latency bound.
//
// Decomposition: one thread-block cluster per vector, one CTA per slab of kSTS = 4 t-planes
// (cluster size n_t / 4 <= 8).  Each CTA
//   1. stages x on its planes +- 5 (the P0 / K reach along t) in shared memory;
//   2. computes, for its own points, h and the products q_t = u~_t h, q_x = u~_x h, q_y = u~_y h
//      and sigma alpha h into shared memory (the per-point coefficients are read once, here);
//   3. one cluster barrier: the q_t of the neighbouring slabs become readable through
//      distributed shared memory (the t-direction K^T reaches at most 4 planes = one slab);
//   4. evaluates S x at its own points from shared memory only (P0 terms from the staged x,
//      K^T terms from the q planes, the t halo from the neighbours' shared memory) and applies
//      the fused PCG / smoother epilogue (EpiArgs contract).
// Bytes per point: x 4 (+ halo re-reads from L2) + cf 32 (16 as bf16) + the epilogue: one
// read of the coefficients instead of the two-pass kernels' two and no h round trip.
#include <cuda_bf16.h>

#include "internal.h"

namespace mpde {
namespace {

constexpr int kSTS = 4;          // t-planes per CTA
constexpr int kSHalo = 5;        // staged x planes on each side (P0 reach at the t-edge classes)
constexpr int kSThreads = 512;
constexpr int kSMaxPlane = 1024; // x-y points per plane

__device__ __forceinline__ const float* srow(const Geo& G, int d, int i) {
  return G.tab + G.tab_off[d] + i * kTabRow;
}
template <typename CF>
__device__ __forceinline__ float ldcf(const CF* p);
template <>
__device__ __forceinline__ float ldcf<float>(const float* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float ldcf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t s_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(s_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_cluster(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t s_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void s_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int EPI>
__device__ __forceinline__ double slab_epilogue(const EpiArgs& A, int pde, size_t o, float xo, float q) {
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

// 1-D K (2 outputs) at index i of axis d applied to values v(o) = x(i+o), o = -4..4 (zero
// outside the axis); interior rows from the kernel-parameter bank
template <class V>
__device__ __forceinline__ void kf_axis(const Geo& G, int d, int i, V v, float& k1, float& k2) {
  const int n = G.n[d];
  k1 = 0.f;
  k2 = 0.f;
  if (i >= 2 && i <= n - 3) {
#pragma unroll
    for (int o = -2; o <= 2; ++o) {
      const float xv = v(o);
      k1 = fmaf(G.irow[d][(o + 2) * 2], xv, k1);
      k2 = fmaf(G.irow[d][(o + 2) * 2 + 1], xv, k2);
    }
  } else {
    const float* row = srow(G, d, i);
    const int lo = max(-4, -i), hi = min(4, n - 1 - i);
    for (int o = lo; o <= hi; ++o) {
      const float xv = v(o);
      k1 = fmaf(__ldg(row + kTabKf + (o + 4) * 2), xv, k1);
      k2 = fmaf(__ldg(row + kTabKf + (o + 4) * 2 + 1), xv, k2);
    }
  }
}

// (P0_d x)(i) - (K_d^T q)(i) along axis d: xv(o) = x(i+o), q1v(o) / q2v(o) = q_d(i+o)
template <class VX, class VQ1, class VQ2>
__device__ __forceinline__ float p0kt_axis(const Geo& G, int d, int i, VX xv, VQ1 q1v, VQ2 q2v) {
  const int n = G.n[d];
  float a = 0.f;
  if (i >= 7 && i <= n - 8) {
#pragma unroll
    for (int o = -4; o <= 4; ++o) a = fmaf(G.irow[d][20 + o + 4], xv(o), a);
#pragma unroll
    for (int o = -2; o <= 2; ++o)
      a -= G.irow[d][10 + (o + 2) * 2] * q1v(o) + G.irow[d][10 + (o + 2) * 2 + 1] * q2v(o);
  } else {
    const float* row = srow(G, d, i);
    const int lo = max(-5, -i), hi = min(5, n - 1 - i);
    for (int o = lo; o <= hi; ++o) a = fmaf(__ldg(row + kTabP0 + o + 5), xv(o), a);
    const int lo2 = max(-4, -i), hi2 = min(4, n - 1 - i);
    for (int o = lo2; o <= hi2; ++o)
      a -= __ldg(row + kTabKT + (o + 4) * 2) * q1v(o) + __ldg(row + kTabKT + (o + 4) * 2 + 1) * q2v(o);
  }
  return a;
}

template <int EPI, typename CF>
__global__ void __launch_bounds__(kSThreads) k_schur_slab(Geo G, const CF* __restrict__ cf, int crep,
                                                          const float* __restrict__ x, EpiArgs A,
                                                          const int* act) {
  MPDE_PDL_ENTRY();
  extern __shared__ __align__(16) float ssl[];
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;  // uniform over the cluster (same vector)
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2], NXY = n1 * n2;
  const int t0 = blockIdx.x * kSTS;
  const int NOWN = kSTS * NXY;
  float* xs = ssl;                                // [kSTS + 2 kSHalo][NXY]
  float* qs = ssl + (kSTS + 2 * kSHalo) * NXY;    // [7][kSTS][NXY]: q_t1 q_t2 q_x1 q_x2 q_y1 q_y2 sah
  const float* xb = x + (size_t)v * P;
  const CF* cb = cf + (size_t)pde * 8 * P;

  // 1. x on planes t0-5 .. t0+kSTS+4 (zero outside the domain), 16-byte loads
  {
    const int nq = (kSTS + 2 * kSHalo) * NXY / 4;
    for (int k = threadIdx.x; k < nq; k += kSThreads) {
      const int e = 4 * k, pl = e / NXY, t = t0 - kSHalo + pl;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t >= 0 && t < n0) val = __ldg(reinterpret_cast<const float4*>(xb + (size_t)t * NXY + (e - pl * NXY)));
      *reinterpret_cast<float4*>(xs + e) = val;
    }
  }
  __syncthreads();
  // 2. h and the q products at the own points
  for (int k = threadIdx.x; k < NOWN; k += kSThreads) {
    const int jl = k / NXY, r = k - jl * NXY, t = t0 + jl;
    const int ix = r / n2, iy = r - ix * n2;
    const size_t pg = (size_t)t * NXY + r;
    const float* xc = xs + (jl + kSHalo) * NXY + r;  // x at this point in the staged planes
    const float csa = ldcf(cb + pg), cis = ldcf(cb + P + pg);
    float g = csa * xc[0];
    float u[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) u[f] = ldcf(cb + (size_t)(2 + f) * P + pg);
    float k1, k2;
    kf_axis(G, 0, t, [&](int o) { return xc[o * NXY]; }, k1, k2);
    g -= u[0] * k1 + u[1] * k2;
    kf_axis(G, 1, ix, [&](int o) { return xc[o * n2]; }, k1, k2);
    g -= u[2] * k1 + u[3] * k2;
    kf_axis(G, 2, iy, [&](int o) { return xc[o]; }, k1, k2);
    g -= u[4] * k1 + u[5] * k2;
    const float h = cis * g;
#pragma unroll
    for (int f = 0; f < 6; ++f) qs[f * NOWN + k] = u[f] * h;
    qs[6 * NOWN + k] = csa * h;
  }
  // 3. every slab's q planes written: the t halo is read from the neighbours' shared memory
  s_cluster_sync();
  const uint32_t rank = s_rank();
  const int CL = gridDim.x;
  const uint32_t q_lo = rank > 0 ? s_map(qs, rank - 1) : 0u;
  const uint32_t q_hi = (int)rank < CL - 1 ? s_map(qs, rank + 1) : 0u;
  // 4. S x at the own points + epilogue
  double dot = 0.0;
  const float wb2 = G.wb * G.wb;
  for (int k = threadIdx.x; k < NOWN; k += kSThreads) {
    const int jl = k / NXY, r = k - jl * NXY, t = t0 + jl;
    const int ix = r / n2, iy = r - ix * n2;
    const float* xc = xs + (jl + kSHalo) * NXY + r;
    const float x0 = xc[0];
    float acc = qs[6 * NOWN + k];
    if (dir_face(G, 0, t) | dir_face(G, 1, ix) | dir_face(G, 2, iy)) acc += wb2 * x0;
    // q_t at plane t+o: own slab, or the neighbouring slab's shared memory (|o| <= 4 < kSTS+1)
    auto qt = [&](int f, int o) -> float {
      const int jj = jl + o;
      if (jj >= 0 && jj < kSTS) return qs[f * NOWN + jj * NXY + r];
      if (jj < 0) return ld_cluster(q_lo + (uint32_t)(sizeof(float) * (f * NOWN + (jj + kSTS) * NXY + r)));
      return ld_cluster(q_hi + (uint32_t)(sizeof(float) * (f * NOWN + (jj - kSTS) * NXY + r)));
    };
    acc += p0kt_axis(G, 0, t, [&](int o) { return xc[o * NXY]; }, [&](int o) { return qt(0, o); },
                     [&](int o) { return qt(1, o); });
    const float* q2 = qs + 2 * NOWN + k;
    const float* q3 = qs + 3 * NOWN + k;
    acc += p0kt_axis(G, 1, ix, [&](int o) { return xc[o * n2]; }, [&](int o) { return q2[o * n2]; },
                     [&](int o) { return q3[o * n2]; });
    const float* q4 = qs + 4 * NOWN + k;
    const float* q5 = qs + 5 * NOWN + k;
    acc += p0kt_axis(G, 2, iy, [&](int o) { return xc[o]; }, [&](int o) { return q4[o]; },
                     [&](int o) { return q5[o]; });
    dot += slab_epilogue<EPI>(A, pde, (size_t)v * P + (size_t)t * NXY + r, x0, acc);
  }
  if (A.pts && threadIdx.x == 0) atomicAdd(A.pts + EPI, (unsigned long long)NOWN);
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (threadIdx.x == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
  s_cluster_sync();  // no CTA leaves while a neighbour may still read its q planes
}

int g_slab = -1;  // env MPDE_SLAB=1 enables the one-launch slab apply (default off)
}  // namespace

// mid-size 3D fp32 levels: x-y plane <= 1024 points, n_t = 4 * (2..8) slabs
bool use_slab(const Geo& G, bool f64) {
  if (g_slab < 0) {
    const char* e = getenv("MPDE_SLAB");
    g_slab = e ? atoi(e) : 0;  // opt-in: measured 3x slower than the two passes
  }
  if (!g_slab || f64 || G.D != 3) return false;
  const int nxy = G.n[1] * G.n[2];
  if (nxy > kSMaxPlane || (nxy & 3) || G.n[0] % kSTS) return false;
  const int cl = G.n[0] / kSTS;
  return cl >= 2 && cl <= 8;
}
int slab_ctas(const Geo& G) { return G.n[0] / kSTS; }

template <int EPI, typename CF>
static cudaError_t launch_slab_t(const Geo& G, int nvec, int crep, const CF* cf, const float* x,
                                 const EpiArgs& A, const int* act, cudaStream_t s) {
  const int nxy = G.n[1] * G.n[2];
  const size_t smem = sizeof(float) * ((size_t)(kSTS + 2 * kSHalo) * nxy + (size_t)7 * kSTS * nxy);
  auto kern = k_schur_slab<EPI, CF>;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G.n[0] / kSTS, nvec, 1);
  cfg.blockDim = dim3(kSThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G.n[0] / kSTS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, G, cf, crep, x, A, act);
}

void launch_schur_slab(int epi, const Geo& G, int nvec, int crep, const void* cf, bool bf16,
                       const float* x, const EpiArgs& A, const int* act, cudaStream_t s) {
  ++g_launch_count;
#define SLAB_CASE(E)                                                                              \
  case E:                                                                                         \
    if (bf16)                                                                                     \
      launch_slab_t<E, __nv_bfloat16>(G, nvec, crep, static_cast<const __nv_bfloat16*>(cf), x, A, act, s); \
    else                                                                                          \
      launch_slab_t<E, float>(G, nvec, crep, static_cast<const float*>(cf), x, A, act, s);       \
    break;
  switch (epi) {
    SLAB_CASE(EPI_STORE)
    SLAB_CASE(EPI_DOT)
    SLAB_CASE(EPI_POWER)
    SLAB_CASE(EPI_RESID)
    SLAB_CASE(EPI_SMOOTH)
    SLAB_CASE(EPI_SMOOTH_LAST)
    SLAB_CASE(EPI_POST0)
  }
#undef SLAB_CASE
}

}  // namespace mpde
