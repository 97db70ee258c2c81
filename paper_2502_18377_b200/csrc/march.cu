// march.cu -- the condensed operator S applied in ONE kernel by t-marching x-strips, with the
// plane data streamed in by bulk-async (TMA) copies and the x-halo of the intermediate
// exchanged through distributed shared memory (B200 / sm_100a).
//
// Operator (schur.cu header; Eq. 9 P:193-196 condensed onto u_phi):
//   h(p)  = (1/sigma) ( sigma alpha x - sum_d u~_d . (K_d x)(p) )                 (pass 1)
//   S x   = sum_d P0_d x - sum_d K_d^T (u~_d h) + sigma alpha h + w_bnd^2 [p in B] x (pass 2)
// The two-pass kernels (schur.cu) round-trip h through HBM and read the per-point
// coefficients cf twice: x 4 + cf 32 + h 4 (pass 1) and x 4 + h 4 + cf 28 (pass 2) bytes per
// point before the epilogue.  Here one kernel reads x 4 + cf 32 (16 as bf16) per point.
//
// Decomposition (3D levels, n_y = NY in {32, 64, 128}, n_x = NX = kMTX * CL, CL <= 16):
//   * one CTA per (vector, strip of kMTX = 8 x-rows x all NY y-points); the CL strips of one
//     vector form a thread-block cluster;
//   * the CTA marches along t (dim 0, the slowest).  At step s it
//       - receives x plane s (rows X0-5 .. X0+12, clipped) and cf plane s-4 (its 8 rows) by
//         cp.async.bulk into shared-memory rings, completion on mbarriers (expect-tx); one
//         thread issues the copies 2 / 3 steps ahead of use; the thread's own column of x(s)
//         for the t queue is a plain coalesced load issued 2 steps ahead (register prefetch);
//       - phase A on plane m = s-4: h(m) and q_d = u~_d h(m) at its own points.  The t-part of
//         K_t x comes from a per-thread register queue of x(m-4 .. m+4); the x / y parts from
//         the x plane in shared memory.  q_x of the two rows next to each strip edge is also
//         stored into the neighbouring CTA's halo rows (st.shared::cluster);
//       - scatters the t-direction terms of plane m (P0_t x(m), K_t^T q_t(m)) into a register
//         queue of 11 output accumulators (planes m-5 .. m+5) -- every point's t-terms stay in
//         the thread that owns its column, no shared memory traffic;
//       - after a CTA barrier: the y-terms (P0_y x, K_y^T q_y) and P0_x x of plane m;
//       - after the cluster barrier that publishes q_x(m-1): the x-terms K_x^T q_x(m-1);
//       - plane s-9 is complete: the fused PCG / smoother epilogue (EpiArgs contract).
//   * a thread owns a pair of consecutive y points (float2).  Pairs 4 .. NY/2-5 of every row
//     run the interior stencils (coefficients in the kernel-parameter bank, no branches);
//     the 8 edge pairs of every row are packed into their own warps and use table rows.
//     Strips whose rows are all interior use the constant-bank x stencils; the two edge
//     strips use table rows staged in shared memory.
//
// Reaches (schur.cu tables): K (derivative + Taylor rows) 2 interior / 4 at the edge classes,
// K^T 2 / 4, P0 4 / 5 (rows 0 <-> 5 and n-6 <-> n-1 only).  Strip boundaries are at multiples
// of 8 >= 8 rows from the domain edge, where every reach is the interior one, so the x halo
// is 4 rows of x (+1 row of slack for the P0 edge reach inside the edge strips) and 2 rows of q_x.
#include <cuda_bf16.h>

#include "internal.h"

namespace mpde {
namespace {

constexpr int kMTX = 8;    // x rows per strip (CTA)
constexpr int kMRX = 3;    // x-plane ring slots: planes m .. m+2 (plane p issued at step p+2, used at p+4)
constexpr int kMRC = 2;    // cf ring slots: planes m, m+1 (plane p issued at step p+2, used at p+4)
constexpr int kMXR = kMTX + 10;  // rows of an x slot: X0-5 .. X0+kMTX+4
constexpr int kMQR = kMTX + 4;   // rows of a q_x slot: X0-2 .. X0+kMTX+1
constexpr int kMaxNT = 256;      // t extent the per-step coefficient tables hold

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
// global -> shared bulk copy (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// arrive (count 1) on an mbarrier of another CTA of the cluster (release at cluster scope:
// this thread's prior shared-memory reads are ordered before the peer's reuse of the slot)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t rbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// asynchronous remote store into a neighbour CTA's shared memory; completion (8 bytes) is
// counted on the neighbour's mbarrier `rbar` (no fence on the sending side)
__device__ __forceinline__ void st_async2(uint32_t addr, float a, float b, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
      "f"(a), "f"(b), "r"(rbar)
      : "memory");
}

__device__ __forceinline__ float2 ld2s(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2s(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
// packed fp32x2 FMA (FFMA2 on sm_100a): a += c * x for both points of a pair
__device__ __forceinline__ void fma2(float2& a, float c, float2 x) {
  a = __ffma2_rn(make_float2(c, c), x, a);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }
template <typename CF>
__device__ __forceinline__ float2 cf2(const CF* p);
template <>
__device__ __forceinline__ float2 cf2<float>(const float* p) {
  return *reinterpret_cast<const float2*>(p);
}
template <>
__device__ __forceinline__ float2 cf2<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}

// fused PCG / smoother epilogue for two consecutive points (same contract as schur.cu), split
// in two so that its global loads are issued one step before the plane is complete (they are
// then in flight during the step instead of exposing a full memory round trip per step).
// x of the output plane is the thread's own column, taken from the t queue (no load).
struct EpiIn {
  float2 r, d, e, p;
};
template <int EPI>
__device__ __forceinline__ EpiIn pair_epi_load(const EpiArgs& A, size_t o) {
  EpiIn in;
  in.r = in.d = in.e = in.p = make_float2(0.f, 0.f);
  if (EPI == EPI_POWER) in.d = __ldg(reinterpret_cast<const float2*>(A.dinv + o));
  if (EPI == EPI_RESID || EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) {
    in.r = *reinterpret_cast<const float2*>(A.res + o);
  }
  if (EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) {
    in.d = __ldg(reinterpret_cast<const float2*>(A.dinv + o));
    in.e = *reinterpret_cast<const float2*>(A.e + o);
    if (A.rdot) in.p = *reinterpret_cast<const float2*>(A.rdot + o);
  }
  return in;
}
template <int EPI>
__device__ __forceinline__ double pair_epi_finish(const EpiArgs& A, int pde, size_t o, const EpiIn& in,
                                                  float2 xv, float2 q) {
  double dot = 0.0;
  if (EPI == EPI_STORE) {
    *reinterpret_cast<float2*>(A.y + o) = q;
  } else if (EPI == EPI_DOT) {
    *reinterpret_cast<float2*>(A.y + o) = q;
    dot = double(xv.x) * q.x + double(xv.y) * q.y;
  } else if (EPI == EPI_POWER) {
    *reinterpret_cast<float2*>(A.y + o) = make_float2(in.d.x * q.x, in.d.y * q.y);
    dot = double(xv.x) * q.x + double(xv.y) * q.y;
  } else if (EPI == EPI_RESID) {
    *reinterpret_cast<float2*>(A.res + o) = make_float2(in.r.x - q.x, in.r.y - q.y);
  } else if (EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST) {
    const float al = A.coef[pde * A.coef_stride + 2 * A.step];
    const float be = A.coef[pde * A.coef_stride + 2 * A.step + 1];
    const float2 r = make_float2(in.r.x - q.x, in.r.y - q.y);
    const float2 dn = make_float2(al * xv.x + be * in.d.x * r.x, al * xv.y + be * in.d.y * r.y);
    const float2 e = make_float2(in.e.x + dn.x, in.e.y + dn.y);
    *reinterpret_cast<float2*>(A.e + o) = e;
    if (EPI == EPI_SMOOTH) {
      *reinterpret_cast<float2*>(A.res + o) = r;
      *reinterpret_cast<float2*>(A.d_out + o) = dn;
    }
    if (A.rdot) dot = double(in.p.x) * e.x + double(in.p.y) * e.y;
  } else if (EPI == EPI_POST0) {
    const float be = A.coef[pde * A.coef_stride + 1];
    const float2 r = make_float2(in.r.x - q.x, in.r.y - q.y);
    const float2 dn = make_float2(be * in.d.x * r.x, be * in.d.y * r.y);
    const float2 e = make_float2(in.e.x + xv.x + dn.x, in.e.y + xv.y + dn.y);
    *reinterpret_cast<float2*>(A.e + o) = e;
    *reinterpret_cast<float2*>(A.res + o) = r;
    *reinterpret_cast<float2*>(A.d_out + o) = dn;
    if (A.rdot) dot = double(in.p.x) * e.x + double(in.p.y) * e.y;
  }
  return dot;
}

template <int NY, typename CF>
struct MarchSmem {
  static constexpr int NP = NY / 2;          // pairs per row
  static constexpr int NI = NP - 8;          // interior pairs per row (4 .. NP-5)
  static constexpr int THREADS = kMTX * NP;  // one thread per pair of the strip
  static constexpr int XS = kMXR * NY;       // floats per x slot
  static constexpr int CS = 8 * kMTX * NY;   // CF elements per cf slot (8 fields)
  static constexpr int QX = 2 * kMQR * NY;   // floats per q_x slot (2 fields)
  static constexpr int QY = 2 * kMTX * NY;   // floats per q_y buffer (2 fields)
  // byte offsets (16-byte aligned)
  static constexpr size_t oX = 0;
  static constexpr size_t oC = oX + sizeof(float) * kMRX * XS;
  static constexpr size_t oQX = oC + sizeof(CF) * kMRC * CS;
  static constexpr size_t oQY = oQX + sizeof(float) * 3 * QX;  // 3 q_x slots
  static constexpr size_t oXT = oQY + sizeof(float) * 2 * QY;   // x-axis rows of the strip
  static constexpr size_t oYT = oXT + sizeof(float) * kMTX * kTabRow;  // 16 edge y rows
  static constexpr size_t oTT = oYT + sizeof(float) * 16 * kTabRow;    // per-step t rows
  static constexpr int TT = 56;  // per-step t row: Kf [0,18) | pad | scatter [20,53) | pad
  __host__ __device__ static size_t tt_floats(int n0) { return (size_t)n0 * TT; }
  static size_t bytes(int n0) {
    return oTT + sizeof(float) * tt_floats(n0) + sizeof(uint64_t) * (kMRX + kMRC + 9) + 16;
  }
};

template <int EPI, int NY, typename CF>
__global__ void __launch_bounds__(MarchSmem<NY, CF>::THREADS)
    k_schur_march(Geo G, const CF* __restrict__ cf, int crep, const float* __restrict__ x,
                  EpiArgs A, const int* act) {
  using SM = MarchSmem<NY, CF>;
  constexpr int NP = SM::NP, NI = SM::NI;
  MPDE_PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char msm[];
  const int v = blockIdx.y, P = G.P, pde = v / crep;
  if (act && !act[pde]) return;  // uniform over the cluster (same vector)
  const int n0 = G.n[0], NX = G.n[1];
  const int s0 = NX * NY;  // plane stride
  const int strip = blockIdx.x, X0 = strip * kMTX;
  const int CL = gridDim.x;  // cluster = all strips of the vector
  const int tid = threadIdx.x;

  float* xs = reinterpret_cast<float*>(msm + SM::oX);
  CF* cs = reinterpret_cast<CF*>(msm + SM::oC);
  float* qxs = reinterpret_cast<float*>(msm + SM::oQX);
  float* qys = reinterpret_cast<float*>(msm + SM::oQY);
  float* xtab = reinterpret_cast<float*>(msm + SM::oXT);
  float* ytab = reinterpret_cast<float*>(msm + SM::oYT);
  float* ttab = reinterpret_cast<float*>(msm + SM::oTT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(msm + SM::oTT + sizeof(float) * SM::tt_floats(n0));

  // ---- thread -> pair: interior pairs first (whole warps), then the 8 edge pairs per row --
  const bool ipair = tid < kMTX * NI;
  int r, q;
  if (ipair) {
    r = tid / NI;
    q = 4 + (tid - r * NI);
  } else {
    const int e = tid - kMTX * NI;
    r = e >> 3;
    const int k = e & 7;
    q = k < 4 ? k : NP - 8 + k;
  }
  const int y0 = 2 * q, xo = X0 + r;
  // strip whose rows are all interior for K (2..n-3), K^T and P0 (7..n-8)
  const bool istrip = X0 >= 7 && X0 + kMTX - 1 <= NX - 8;

  // ---- set-up: zero the rings (out-of-domain halo rows stay zero), tables, barriers -------
  for (int i = tid; i < (int)(SM::oXT / 4); i += SM::THREADS) reinterpret_cast<float*>(msm)[i] = 0.f;
  for (int i = tid; i < kMTX * kTabRow; i += SM::THREADS) {
    const int rr = i / kTabRow, c = i - rr * kTabRow;
    xtab[i] = X0 + rr < NX ? __ldg(G.tab + G.tab_off[1] + (X0 + rr) * kTabRow + c) : 0.f;
  }
  for (int i = tid; i < 16 * kTabRow; i += SM::THREADS) {
    const int rr = i / kTabRow, c = i - rr * kTabRow;
    const int yy = rr < 8 ? rr : NY - 16 + rr;
    ytab[i] = __ldg(G.tab + G.tab_off[2] + yy * kTabRow + c);
  }
  // per-step t rows (16-byte aligned, read as float4 broadcasts): [0,18) Kf of row m
  // (coefficient of x(m+o), o=-4..4, k), [20,53) the scatter of plane m into the outputs
  // j = m-5+i: (P0(j, m-j), KT(j, m-j, 0), KT(j, m-j, 1))
  for (int i = tid; i < n0 * SM::TT; i += SM::THREADS) {
    const int m = i / SM::TT, c = i - m * SM::TT;
    float val = 0.f;
    if (c < 18) {
      const int o = c / 2 - 4;
      if (m + o >= 0 && m + o < n0) val = __ldg(G.tab + G.tab_off[0] + m * kTabRow + kTabKf + c);
    } else if (c >= 20 && c < 53) {
      const int ii = (c - 20) / 3, k = (c - 20) % 3, j = m - 5 + ii, o = m - j;
      if (j >= 0 && j < n0) {
        const float* row = G.tab + G.tab_off[0] + j * kTabRow;
        if (k == 0) val = __ldg(row + kTabP0 + o + 5);
        else if (o >= -4 && o <= 4) val = __ldg(row + kTabKT + (o + 4) * 2 + (k - 1));
      }
    }
    ttab[i] = val;
  }
  uint64_t* hbar = bar + kMRX + kMRC;  // [3] q_x halo rows of plane p received (slot p % 3)
  // [2][3] the left (0) / right (1) neighbour has finished reading its halo slot p % 3, so
  // this CTA may store plane p+3's rows there (flow control instead of a cluster barrier)
  uint64_t* fbar = hbar + 3;
  const bool has_left = strip > 0, has_right = strip < CL - 1;
  const uint32_t halo_bytes = (uint32_t)((int(has_left) + int(has_right)) * 2 * 2 * NY * sizeof(float));
  if (tid == 0) {
    for (int i = 0; i < kMRX + kMRC + 9; ++i) mbar_init(bar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int p = 0; p < 3 && p < n0; ++p) mbar_expect_tx(hbar + p, halo_bytes);  // planes 0..2
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  const float* xb = x + (size_t)v * P;
  const CF* cb = cf + (size_t)pde * 8 * P;
  const int xr0 = max(X0 - 5, 0), xr1 = min(X0 + kMTX + 5, NX);  // x rows copied per plane
  auto issue_x = [&](int p) {
    if (p >= n0) return;
    uint64_t* b = bar + (p % kMRX);
    const uint32_t bytes = (uint32_t)((xr1 - xr0) * NY * sizeof(float));
    mbar_expect_tx(b, bytes);
    bulk_g2s(xs + (p % kMRX) * SM::XS + (xr0 - (X0 - 5)) * NY, xb + (size_t)p * s0 + (size_t)xr0 * NY,
             bytes, b);
  };
  auto issue_c = [&](int p) {
    if (p >= n0) return;
    uint64_t* b = bar + kMRX + (p % kMRC);
    const uint32_t fb = (uint32_t)(kMTX * NY * sizeof(CF));
    mbar_expect_tx(b, 8 * fb);
    CF* dst = cs + (p % kMRC) * SM::CS;
    const CF* src = cb + (size_t)p * s0 + (size_t)X0 * NY;
#pragma unroll 1
    for (int f = 0; f < 8; ++f) bulk_g2s(dst + f * kMTX * NY, src + (size_t)f * P, fb, b);
  };
  // every CTA of the cluster is running before any remote store (DSMEM)
  cluster_arrive();
  cluster_wait();

  const uint32_t crank = cluster_rank();
  // remote halo slots: my rows 0,1 -> left neighbour's rows kMTX+2, kMTX+3; my rows
  // kMTX-2, kMTX-1 -> right neighbour's rows 0, 1
  uint32_t rq_remote = 0, rq_bar = 0;
  bool rq_send = false;
  const uint64_t* rq_free = nullptr;  // my fbar row for the neighbour I send to
  if (r < 2 && has_left) {
    rq_remote = map_rank(qxs + (kMTX + 2 + r) * NY + y0, crank - 1);
    rq_bar = map_rank(hbar, crank - 1);
    rq_free = fbar;
    rq_send = true;
  } else if (r >= kMTX - 2 && has_right) {
    rq_remote = map_rank(qxs + (r - (kMTX - 2)) * NY + y0, crank + 1);
    rq_bar = map_rank(hbar, crank + 1);
    rq_free = fbar + 3;
    rq_send = true;
  }
  // slot-free signals to the CTAs that send into my halo rows: the left neighbour tracks my
  // slots in its fbar[1][.], the right neighbour in its fbar[0][.]
  const uint32_t free_left = has_left ? map_rank(fbar + 3, crank - 1) : 0u;
  const uint32_t free_right = has_right ? map_rank(fbar, crank + 1) : 0u;

  const float wb2 = G.wb * G.wb;
  const bool xface = dir_face(G, 1, xo);  // Dirichlet rows (Eq. 4) on the x / y faces
  const bool yface0 = dir_face(G, 2, y0), yface1 = dir_face(G, 2, y0 + 1);
  const float* yt0 = ytab + (q < 4 ? y0 : y0 - (NY - 16)) * kTabRow;  // edge pairs: rows y0, y0+1
  const float* xt = xtab + r * kTabRow;

  const float* xown = xb + (size_t)xo * NY + y0;  // this thread's column
  float2 xpre0 = __ldg(reinterpret_cast<const float2*>(xown));  // x(0), x(1): prefetched
  float2 xpre1 = n0 > 1 ? __ldg(reinterpret_cast<const float2*>(xown + s0)) : make_float2(0.f, 0.f);
  float2 xq[9];   // x(m-4 .. m+4) of this column, m = s-4
  float2 acc[11]; // outputs of planes s-9 .. s+1
#pragma unroll
  for (int i = 0; i < 9; ++i) xq[i] = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 11; ++i) acc[i] = make_float2(0.f, 0.f);
  double dot = 0.0;
  const int nsteps = n0 + 9;

#pragma unroll 1
  for (int s = 0; s < nsteps; ++s) {
    const int m = s - 4;
    // epilogue inputs of plane j = s-9 (completed at the end of this step): loads issued now
    const int j = s - 9;
    const size_t oj = (size_t)v * P + (size_t)max(j, 0) * s0 + (size_t)xo * NY + y0;
    EpiIn ein;
    if (j >= 0) ein = pair_epi_load<EPI>(A, oj);
    const float2 xj = xq[0];  // x(s-9), leaving the queue
    // ---- own x(s) into the t queue (loaded 2 steps ago) -----------------------------------
#pragma unroll
    for (int i = 0; i < 8; ++i) xq[i] = xq[i + 1];
    xq[8] = xpre0;
    xpre0 = xpre1;
    xpre1 = s + 2 < n0 ? __ldg(reinterpret_cast<const float2*>(xown + (size_t)(s + 2) * s0))
                       : make_float2(0.f, 0.f);
    // ---- phase A on plane m: h, q; scatter of the t-terms ----------------------------------
    const bool mval = m >= 0 && m < n0;
    const float* xm = xs + ((m + kMRX) % kMRX) * SM::XS + (r + 5) * NY + y0;  // own point, plane m
    if (mval) {
      mbar_wait(bar + (m % kMRX), (uint32_t)((m / kMRX) & 1));
      mbar_wait(bar + kMRX + (m % kMRC), (uint32_t)((m / kMRC) & 1));
      const CF* cm = cs + (m % kMRC) * SM::CS + r * NY + y0;
      const float2 csa = cf2(cm), cis = cf2(cm + kMTX * NY);
      const float2 ut1 = cf2(cm + 2 * kMTX * NY), ut2 = cf2(cm + 3 * kMTX * NY);
      const float2 ux1 = cf2(cm + 4 * kMTX * NY), ux2 = cf2(cm + 5 * kMTX * NY);
      const float2 uy1 = cf2(cm + 6 * kMTX * NY), uy2 = cf2(cm + 7 * kMTX * NY);
      const float* tt = ttab + m * SM::TT;
      const float2 x0 = xq[4];
      float2 g = mul2(csa, x0);
      {  // t: K_t x from the register queue (row m of the t table, zero outside the domain)
        float2 k1 = make_float2(0.f, 0.f), k2 = k1;
        if (m >= 2 && m <= n0 - 3) {  // central rows: constant-bank coefficients, 5 taps
#pragma unroll
          for (int o = -2; o <= 2; ++o) {
            fma2(k1, G.irow[0][(o + 2) * 2], xq[4 + o]);
            fma2(k2, G.irow[0][(o + 2) * 2 + 1], xq[4 + o]);
          }
        } else {
          float kf[20];
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const float4 t4 = *reinterpret_cast<const float4*>(tt + 4 * k);
            kf[4 * k] = t4.x;
            kf[4 * k + 1] = t4.y;
            kf[4 * k + 2] = t4.z;
            kf[4 * k + 3] = t4.w;
          }
#pragma unroll
          for (int o = 0; o < 9; ++o) {
            fma2(k1, kf[2 * o], xq[o]);
            fma2(k2, kf[2 * o + 1], xq[o]);
          }
        }
        g.x -= ut1.x * k1.x + ut2.x * k2.x;
        g.y -= ut1.y * k1.y + ut2.y * k2.y;
      }
      {  // x: K_x x from the x plane (rows r+5+o of the slot)
        float2 k1 = make_float2(0.f, 0.f), k2 = k1;
        if (istrip) {
#pragma unroll
          for (int o = -2; o <= 2; ++o) {
            const float2 xv = ld2s(xm + o * NY);
            fma2(k1, G.irow[1][(o + 2) * 2], xv);
            fma2(k2, G.irow[1][(o + 2) * 2 + 1], xv);
          }
        } else {
#pragma unroll
          for (int o = -4; o <= 4; ++o) {
            const float2 xv = ld2s(xm + o * NY);
            fma2(k1, xt[kTabKf + (o + 4) * 2], xv);
            fma2(k2, xt[kTabKf + (o + 4) * 2 + 1], xv);
          }
        }
        g.x -= ux1.x * k1.x + ux2.x * k2.x;
        g.y -= ux1.y * k1.y + ux2.y * k2.y;
      }
      {  // y: K_y x along the row
        float k1a = 0.f, k2a = 0.f, k1b = 0.f, k2b = 0.f;
        if (ipair) {  // window y0-2 .. y0+3, interior coefficients
          const float2 wa = ld2s(xm - 2), wb = ld2s(xm + 2);
          const float w[6] = {wa.x, wa.y, x0.x, x0.y, wb.x, wb.y};
#pragma unroll
          for (int o = -2; o <= 2; ++o) {
            k1a = fmaf(G.irow[2][(o + 2) * 2], w[2 + o], k1a);
            k2a = fmaf(G.irow[2][(o + 2) * 2 + 1], w[2 + o], k2a);
            k1b = fmaf(G.irow[2][(o + 2) * 2], w[3 + o], k1b);
            k2b = fmaf(G.irow[2][(o + 2) * 2 + 1], w[3 + o], k2b);
          }
        } else {  // edge pairs: table rows, offsets -4..4, clipped to the row
          const float* ta = yt0;
          const float* tb = yt0 + kTabRow;
          const float* row = xm - y0;
#pragma unroll
          for (int o = -4; o <= 5; ++o) {
            const int yy = y0 + o;
            const float xv = (yy >= 0 && yy < NY) ? row[yy] : 0.f;
            if (o <= 4) {
              k1a = fmaf(ta[kTabKf + (o + 4) * 2], xv, k1a);
              k2a = fmaf(ta[kTabKf + (o + 4) * 2 + 1], xv, k2a);
            }
            if (o >= -3) {
              k1b = fmaf(tb[kTabKf + (o + 3) * 2], xv, k1b);
              k2b = fmaf(tb[kTabKf + (o + 3) * 2 + 1], xv, k2b);
            }
          }
        }
        g.x -= uy1.x * k1a + uy2.x * k2a;
        g.y -= uy1.y * k1b + uy2.y * k2b;
      }
      const float2 h = make_float2(cis.x * g.x, cis.y * g.y);
      // q_x (own rows + the neighbour's halo), q_y
      float* qx = qxs + (m % 3) * SM::QX + (r + 2) * NY + y0;
      const float2 qx1 = make_float2(ux1.x * h.x, ux1.y * h.y), qx2 = make_float2(ux2.x * h.x, ux2.y * h.y);
      st2s(qx, qx1);
      st2s(qx + kMQR * NY, qx2);
      if (rq_send) {
        // the neighbour has consumed plane m-3 from this slot (flow control)
        if (m >= 3) mbar_wait(const_cast<uint64_t*>(rq_free) + m % 3, (uint32_t)(((m / 3) - 1) & 1));
        const uint32_t ra = rq_remote + (uint32_t)((m % 3) * SM::QX * sizeof(float));
        const uint32_t rb = rq_bar + (uint32_t)((m % 3) * sizeof(uint64_t));
        st_async2(ra, qx1.x, qx1.y, rb);
        st_async2(ra + (uint32_t)(kMQR * NY * sizeof(float)), qx2.x, qx2.y, rb);
      }
      float* qy = qys + (m & 1) * SM::QY + r * NY + y0;
      st2s(qy, make_float2(uy1.x * h.x, uy1.y * h.y));
      st2s(qy + kMTX * NY, make_float2(uy2.x * h.x, uy2.y * h.y));
      // t-terms of plane m scattered into the outputs of planes m-5 .. m+5
      const float2 qt1 = mul2(ut1, h), qt2 = mul2(ut2, h);
      const float2 nq1 = make_float2(-qt1.x, -qt1.y), nq2 = make_float2(-qt2.x, -qt2.y);
      float sc[36];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const float4 t4 = *reinterpret_cast<const float4*>(tt + 20 + 4 * k);
        sc[4 * k] = t4.x;
        sc[4 * k + 1] = t4.y;
        sc[4 * k + 2] = t4.z;
        sc[4 * k + 3] = t4.w;
      }
#pragma unroll
      for (int i = 0; i < 11; ++i) {
        fma2(acc[i], sc[3 * i], x0);
        fma2(acc[i], sc[3 * i + 1], nq1);
        fma2(acc[i], sc[3 * i + 2], nq2);
      }
      // sigma alpha h + w_bnd^2 [p in B] x
      const bool tface = dir_face(G, 0, m) | xface;
      acc[5].x += csa.x * h.x + ((tface | yface0) ? wb2 * x0.x : 0.f);
      acc[5].y += csa.y * h.y + ((tface | yface1) ? wb2 * x0.y : 0.f);
    }
    __syncthreads();  // q_y(m) visible; every thread is done with step s-1's slots
    if (tid == 0) {
      // every thread finished the x-terms of plane s-6 (step s-1): its halo slot is free again
      if (s >= 6 && s - 6 < n0 - 3) {
        const uint32_t off = (uint32_t)(((s - 6) % 3) * sizeof(uint64_t));
        if (has_left) mbar_arrive_remote(free_left + off);
        if (has_right) mbar_arrive_remote(free_right + off);
      }
      if (s >= 2) issue_x(s - 2);  // into the slot of plane m-1 (last read at step s-1)
      if (s >= 2) issue_c(s - 2);  // into the slot of cf(m) (read in phase A above)
    }
    // ---- y-terms and P0_x of plane m ---------------------------------------------------------
    if (mval) {
      float2 a = make_float2(0.f, 0.f);
      const float* q1 = qys + (m & 1) * SM::QY + r * NY + y0;
      const float* q2 = q1 + kMTX * NY;
      if (ipair) {
        // P0_y: window y0-4 .. y0+5; K_y^T q_y: windows y0-2 .. y0+3
        float w[10];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const float2 t = ld2s(xm - 4 + 2 * k);
          w[2 * k] = t.x;
          w[2 * k + 1] = t.y;
        }
#pragma unroll
        for (int o = -4; o <= 4; ++o) {
          a.x = fmaf(G.irow[2][20 + o + 4], w[4 + o], a.x);
          a.y = fmaf(G.irow[2][20 + o + 4], w[5 + o], a.y);
        }
        float u1[6], u2[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float2 t1 = ld2s(q1 - 2 + 2 * k), t2 = ld2s(q2 - 2 + 2 * k);
          u1[2 * k] = t1.x;
          u1[2 * k + 1] = t1.y;
          u2[2 * k] = t2.x;
          u2[2 * k + 1] = t2.y;
        }
#pragma unroll
        for (int o = -2; o <= 2; ++o) {
          const float c1 = G.irow[2][10 + (o + 2) * 2], c2 = G.irow[2][10 + (o + 2) * 2 + 1];
          a.x -= c1 * u1[2 + o] + c2 * u2[2 + o];
          a.y -= c1 * u1[3 + o] + c2 * u2[3 + o];
        }
      } else {
        const float* ta = yt0;
        const float* tb = yt0 + kTabRow;
        const float* row = xm - y0;
        const float* r1 = q1 - y0;
        const float* r2 = q2 - y0;
#pragma unroll
        for (int o = -5; o <= 6; ++o) {
          const int yy = y0 + o;
          const bool in = yy >= 0 && yy < NY;
          const float xv = in ? row[yy] : 0.f;
          if (o <= 5) a.x = fmaf(ta[kTabP0 + o + 5], xv, a.x);
          if (o >= -4) a.y = fmaf(tb[kTabP0 + o + 4], xv, a.y);
          if (o >= -4 && o <= 5) {
            const float v1 = in ? r1[yy] : 0.f, v2 = in ? r2[yy] : 0.f;
            if (o <= 4) a.x -= ta[kTabKT + (o + 4) * 2] * v1 + ta[kTabKT + (o + 4) * 2 + 1] * v2;
            if (o >= -3) a.y -= tb[kTabKT + (o + 3) * 2] * v1 + tb[kTabKT + (o + 3) * 2 + 1] * v2;
          }
        }
      }
      if (istrip) {
#pragma unroll
        for (int o = -4; o <= 4; ++o) fma2(a, G.irow[1][20 + o + 4], ld2s(xm + o * NY));
      } else {
#pragma unroll
        for (int o = -5; o <= 5; ++o) fma2(a, xt[kTabP0 + o + 5], ld2s(xm + o * NY));
      }
      acc[5].x += a.x;
      acc[5].y += a.y;
    }
    // ---- x-terms of plane s-5: K_x^T q_x (q_x halo rows published by the cluster barrier) ----
    if (s >= 5 && s - 5 < n0) {
      // halo rows of q_x(s-5) from the neighbours (own rows: CTA barrier above)
      mbar_wait(hbar + (s - 5) % 3, (uint32_t)(((s - 5) / 3) & 1));
      const float* q1 = qxs + ((s - 5) % 3) * SM::QX + (r + 2) * NY + y0;
      const float* q2 = q1 + kMQR * NY;
      float2 a = make_float2(0.f, 0.f);
      if (istrip) {
#pragma unroll
        for (int o = -2; o <= 2; ++o) {
          fma2(a, G.irow[1][10 + (o + 2) * 2], ld2s(q1 + o * NY));
          fma2(a, G.irow[1][10 + (o + 2) * 2 + 1], ld2s(q2 + o * NY));
        }
      } else {
#pragma unroll
        for (int o = -2; o <= 2; ++o) {  // reach 2 inside the q_x slot (edge reach 4 is clipped
          // below: rows beyond the slot belong to rows whose K^T offset is zero)
          fma2(a, xt[kTabKT + (o + 4) * 2], ld2s(q1 + o * NY));
          fma2(a, xt[kTabKT + (o + 4) * 2 + 1], ld2s(q2 + o * NY));
        }
#pragma unroll
        for (int o = -4; o <= 4; ++o) {
          if (o >= -2 && o <= 2) continue;
          const int rq = r + 2 + o;  // row in the q_x slot
          if (rq < 0 || rq >= kMQR) continue;
          fma2(a, xt[kTabKT + (o + 4) * 2], ld2s(q1 + o * NY));
          fma2(a, xt[kTabKT + (o + 4) * 2 + 1], ld2s(q2 + o * NY));
        }
      }
      acc[4].x -= a.x;
      acc[4].y -= a.y;
      __syncwarp();
      // re-arm the slot for plane s-2 (its senders write it at their step s+2, after the cluster
      // barrier that follows every thread of this CTA finishing this step)
      if (tid == 0 && s - 2 < n0) mbar_expect_tx(hbar + (s - 5) % 3, halo_bytes);
    }

    // ---- plane s-9 complete: epilogue -----------------------------------------------------------
    if (j >= 0) dot += pair_epi_finish<EPI>(A, pde, oj, ein, xj, acc[0]);
#pragma unroll
    for (int i = 0; i < 10; ++i) acc[i] = acc[i + 1];
    acc[10] = make_float2(0.f, 0.f);
  }
  // no CTA leaves while a neighbour may still signal it (DSMEM targets must stay resident)
  cluster_arrive();
  cluster_wait();
  if (A.pts && tid == 0) atomicAdd(A.pts + EPI, (unsigned long long)kMTX * NY * n0);
  if (EPI == EPI_DOT || EPI == EPI_POWER ||
      ((EPI == EPI_SMOOTH || EPI == EPI_SMOOTH_LAST || EPI == EPI_POST0) && A.rdot)) {
    dot = block_sum(dot);
    if (tid == 0) A.part[(size_t)v * gridDim.x + blockIdx.x] = dot;
  }
}

int g_march = -1;  // env MPDE_MARCH: 0 (default) two-pass kernels, 1 the march on launches with
                   // >= 148 CTAs, 2 the march on every eligible level (tests)
}  // namespace

// 3D levels the t-marching kernel handles: NY in {32, 64, 128}, NX a multiple of 8 with
// 2..8 strips (one portable cluster per vector), n_t in [6, kMaxNT], fp32 arithmetic; the vectors must be 16-byte aligned
// (checked by the caller through march_aligned).
bool use_march(const Geo& G, bool f64, int nvec) {
  if (g_march < 0) {
    const char* e = getenv("MPDE_MARCH");
    g_march = e ? atoi(e) : 0;  // opt-in: at C4 it ties the two-pass kernels
  }
  if (!g_march || f64 || G.D != 3) return false;
  const int ny = G.n[2], nx = G.n[1];
  if (ny != 32 && ny != 64 && ny != 128) return false;
  if (nx % kMTX || nx / kMTX < 2 || nx / kMTX > 8) return false;  // portable cluster sizes
  // at least one CTA per SM: the march is serial along t, so a small grid stays latency bound
  // (those launches keep the two-pass kernels)
  // (MPDE_MARCH=2 forces the march for every eligible level: tests)
  return G.n[0] >= 6 && G.n[0] <= kMaxNT && (g_march == 2 || nvec * (nx / kMTX) >= 148);
}

int march_ctas(const Geo& G) { return G.n[1] / kMTX; }

template <int EPI, int NY, typename CF>
static cudaError_t launch_march_t(const Geo& G, int nvec, int crep, const CF* cf, const float* x,
                                  const EpiArgs& A, const int* act, cudaStream_t s) {
  using SM = MarchSmem<NY, CF>;
  const size_t smem = SM::bytes(G.n[0]);
  auto kern = k_schur_march<EPI, NY, CF>;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G.n[1] / kMTX, nvec, 1);
  cfg.blockDim = dim3(SM::THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G.n[1] / kMTX;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, G, cf, crep, x, A, act);
}

template <typename CF>
static cudaError_t launch_march_cf(int epi, const Geo& G, int nvec, int crep, const CF* cf,
                                   const float* x, const EpiArgs& A, const int* act, cudaStream_t s) {
#define MARCH_NY(E)                                                                         \
  case E:                                                                                   \
    if (G.n[2] == 64) return launch_march_t<E, 64, CF>(G, nvec, crep, cf, x, A, act, s);    \
    if (G.n[2] == 32) return launch_march_t<E, 32, CF>(G, nvec, crep, cf, x, A, act, s);    \
    return launch_march_t<E, 128, CF>(G, nvec, crep, cf, x, A, act, s);
  switch (epi) {
    MARCH_NY(EPI_STORE)
    MARCH_NY(EPI_DOT)
    MARCH_NY(EPI_POWER)
    MARCH_NY(EPI_RESID)
    MARCH_NY(EPI_SMOOTH)
    MARCH_NY(EPI_SMOOTH_LAST)
    MARCH_NY(EPI_POST0)
  }
#undef MARCH_NY
  return cudaErrorInvalidValue;
}

void launch_schur_march(int epi, const Geo& G, int nvec, int crep, const void* cf, bool bf16,
                        const float* x, const EpiArgs& A, const int* act, cudaStream_t s) {
  ++g_launch_count;
  cudaError_t e = bf16 ? launch_march_cf<__nv_bfloat16>(epi, G, nvec, crep,
                                                        static_cast<const __nv_bfloat16*>(cf), x, A, act, s)
                       : launch_march_cf<float>(epi, G, nvec, crep, static_cast<const float*>(cf), x,
                                                A, act, s);
  (void)e;  // launch errors surface through the caller's cudaGetLastError check (CKL)
}

}  // namespace mpde
