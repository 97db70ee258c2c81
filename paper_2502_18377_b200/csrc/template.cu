// template.cu -- polynomial PDE-expression template.
//
// The paper builds the coefficient fields and the right-hand side of the PDE from
// learned polynomials of transformed data fields u~ ("p_1(u~) = theta_0 +
// theta_1 u~ + theta_2 u~^2", "third degree polynomial functions built from
// ... u~, v~ ... coefficients of the u term, ... u_xx and u_yy terms, and ... the right
// hand side b", "degree 1 polynomials"):
//   c_m(p) = sum_k theta[m][k] Phi_k(u~(p)),   b(p) = sum_k theta[M][k] Phi_k(u~(p)),
// Phi_k = prod_f u~_f^e_f over all exponent tuples of total degree <= G, ordered by degree,
// then by tuple in descending lexicographic order (include/mpde.h).  theta is shared by
// the batch.  Backward (chain rule through the template):
//   grad_theta[r][k] = sum_b sum_p g_r(b, p) Phi_k(u~_b(p))       (g_r = dl/dc_r, r = M: dl/db)
//   grad_feat_f(p)   = sum_r g_r(p) sum_k theta[r][k] dPhi_k/du~_f(p)
// Both kernels are HBM-bound pointwise passes: coeff reads F and writes M+1 floats per
// point; grad reads M+1+F and writes F floats per point, and reduces grad_theta with warp
// shuffles into per-CTA fp64 partials (fixed order: deterministic), summed by a second
// kernel.
#include "internal.h"

namespace mpde {

namespace {

// theta rows and exponent tuples in the kernel-parameter bank
struct TmplArgs {
  int R;                   // rows of theta: M + 1
  int M;                   // coefficient fields
  int P;                   // points per PDE
  unsigned char e[kTmplMaxK][3];
};

template <int F, int K>
__device__ __forceinline__ void monomials(const TmplArgs& t, const float (&u)[F], float (&phi)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float v = 1.f;
#pragma unroll
    for (int f = 0; f < F; ++f)
      for (int j = 0; j < t.e[k][f]; ++j) v *= u[f];
    phi[k] = v;
  }
}

constexpr int kTmplPts = 4;  // point groups of kThreads per CTA in the gradient kernel

template <int F, int K>
__global__ void __launch_bounds__(kThreads) k_template_coeff(TmplArgs t, const float* __restrict__ theta,
                                                             const float* __restrict__ feat,
                                                             float* __restrict__ coeff,
                                                             float* __restrict__ rhs) {
  MPDE_PDL_ENTRY();
  __shared__ float th[kTmplMaxR * kTmplMaxK];
  for (int i = threadIdx.x; i < t.R * K; i += blockDim.x) th[i] = theta[i];
  __syncthreads();
  const int b = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= t.P) return;
  float u[F];
#pragma unroll
  for (int f = 0; f < F; ++f) u[f] = feat[((size_t)b * F + f) * t.P + p];
  float phi[K];
  monomials<F, K>(t, u, phi);
  for (int r = 0; r < t.R; ++r) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) acc = fmaf(th[r * K + k], phi[k], acc);
    if (r < t.M)
      coeff[((size_t)b * t.M + r) * t.P + p] = acc;
    else
      rhs[(size_t)b * t.P + p] = acc;
  }
}

// One CTA: kTmplPts * kThreads consecutive points of one PDE.  Partials
// part[(b * gridDim.x + blockIdx.x) * R * K + r * K + k] (fp64).
template <int F, int K>
__global__ void __launch_bounds__(kThreads) k_template_grad(TmplArgs t, const float* __restrict__ theta,
                                                            const float* __restrict__ feat,
                                                            const float* __restrict__ gc,
                                                            const float* __restrict__ gb,
                                                            float* __restrict__ gfeat,
                                                            double* __restrict__ part) {
  MPDE_PDL_ENTRY();
  __shared__ float th[kTmplMaxR * kTmplMaxK];
  __shared__ double acc[kThreads / 32][kTmplMaxR * kTmplMaxK];
  const int NP = t.R * K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < NP; i += blockDim.x) th[i] = theta[i];
  for (int i = lane; i < NP; i += 32) acc[warp][i] = 0.0;
  __syncthreads();
  const int b = blockIdx.y;
  const int p0 = blockIdx.x * (kTmplPts * kThreads);
  for (int it = 0; it < kTmplPts; ++it) {
    const int p = p0 + it * kThreads + threadIdx.x;
    if (p0 + it * kThreads >= t.P) break;  // CTA-uniform
    const bool in = p < t.P;
    float u[F], phi[K];
#pragma unroll
    for (int f = 0; f < F; ++f) u[f] = in ? feat[((size_t)b * F + f) * t.P + p] : 0.f;
    monomials<F, K>(t, u, phi);
    // w_k = sum_r g_r theta[r][k];  grad_theta partial += g_r phi_k (warp sums)
    float w[K];
#pragma unroll
    for (int k = 0; k < K; ++k) w[k] = 0.f;
    for (int r = 0; r < t.R; ++r) {
      float g = 0.f;
      if (in) g = r < t.M ? gc[((size_t)b * t.M + r) * t.P + p] : gb[(size_t)b * t.P + p];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        w[k] = fmaf(g, th[r * K + k], w[k]);
        float s = g * phi[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) acc[warp][r * K + k] += (double)s;
      }
    }
    if (gfeat && in) {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        float gf = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int ef = t.e[k][f];
          if (ef == 0) continue;
          float d = (float)ef;
#pragma unroll
          for (int f2 = 0; f2 < F; ++f2) {
            const int n = t.e[k][f2] - (f2 == f ? 1 : 0);
            for (int j = 0; j < n; ++j) d *= u[f2];
          }
          gf = fmaf(w[k], d, gf);
        }
        gfeat[((size_t)b * F + f) * t.P + p] = gf;
      }
    }
  }
  __syncthreads();
  double* out = part + ((size_t)b * gridDim.x + blockIdx.x) * NP;
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < kThreads / 32; ++w8) s += acc[w8][i];
    out[i] = s;
  }
}

// grad_theta[j] = sum over nparts partials (one CTA per j, fixed-order tree)
__global__ void __launch_bounds__(kThreads) k_template_reduce(const double* __restrict__ part, int nparts,
                                                              int NP, float* __restrict__ gtheta) {
  MPDE_PDL_ENTRY();
  __shared__ double s[kThreads];
  const int j = blockIdx.x;
  double a = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) a += part[(size_t)i * NP + j];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) gtheta[j] = float(s[0]);
}

// monomial exponent tuples: degree ascending, then descending lexicographic order
int fill_exponents(int F, int G, TmplArgs& t) {
  int K = 0;
  for (int deg = 0; deg <= G; ++deg) {
    // descending lexicographic over (e0, e1, e2) with e0 + ... + e_{F-1} = deg
    for (int e0 = deg; e0 >= 0; --e0) {
      if (F == 1) {
        if (e0 != deg) continue;
        t.e[K][0] = e0; t.e[K][1] = 0; t.e[K][2] = 0; ++K;
        continue;
      }
      for (int e1 = deg - e0; e1 >= 0; --e1) {
        const int e2 = deg - e0 - e1;
        if (F == 2 && e2 != 0) continue;
        t.e[K][0] = e0; t.e[K][1] = e1; t.e[K][2] = F == 3 ? e2 : 0; ++K;
      }
    }
  }
  return K;
}

template <int F, int K>
cudaError_t run_coeff(const TmplArgs& t, int B, const float* theta, const float* feat, float* coeff,
                      float* rhs, cudaStream_t s) {
  ++g_launch_count;
  k_template_coeff<F, K><<<dim3((t.P + kThreads - 1) / kThreads, B), kThreads, 0, s>>>(t, theta, feat,
                                                                                       coeff, rhs);
  return cudaGetLastError();
}

template <int F, int K>
cudaError_t run_grad(const TmplArgs& t, int B, const float* theta, const float* feat, const float* gc,
                     const float* gb, float* gtheta, float* gfeat, double* part, cudaStream_t s) {
  const int nx = (t.P + kTmplPts * kThreads - 1) / (kTmplPts * kThreads);
  g_launch_count += 2;
  k_template_grad<F, K><<<dim3(nx, B), kThreads, 0, s>>>(t, theta, feat, gc, gb, gfeat, part);
  k_template_reduce<<<t.R * K, kThreads, 0, s>>>(part, nx * B, t.R * K, gtheta);
  return cudaGetLastError();
}

// (F, K) dispatch over every admissible (n_feat, degree): K = C(F+G, G)
#define MPDE_TMPL_DISPATCH(FN, ...)                                    \
  switch (F * 100 + K) {                                               \
    case 101: return FN<1, 1>(__VA_ARGS__);                            \
    case 102: return FN<1, 2>(__VA_ARGS__);                            \
    case 103: return FN<1, 3>(__VA_ARGS__);                            \
    case 104: return FN<1, 4>(__VA_ARGS__);                            \
    case 105: return FN<1, 5>(__VA_ARGS__);                            \
    case 201: return FN<2, 1>(__VA_ARGS__);                            \
    case 203: return FN<2, 3>(__VA_ARGS__);                            \
    case 206: return FN<2, 6>(__VA_ARGS__);                            \
    case 210: return FN<2, 10>(__VA_ARGS__);                           \
    case 215: return FN<2, 15>(__VA_ARGS__);                           \
    case 301: return FN<3, 1>(__VA_ARGS__);                            \
    case 304: return FN<3, 4>(__VA_ARGS__);                            \
    case 310: return FN<3, 10>(__VA_ARGS__);                           \
    case 320: return FN<3, 20>(__VA_ARGS__);                           \
    case 335: return FN<3, 35>(__VA_ARGS__);                           \
    default: return cudaErrorInvalidValue;                             \
  }

}  // namespace

int template_terms(int F, int G) {
  if (F < 1 || F > 3 || G < 0 || G > 4) return -1;
  TmplArgs t;
  return fill_exponents(F, G, t);
}

size_t template_partials(int P, int B, int F, int G, int M) {
  const int K = template_terms(F, G);
  if (K < 0) return 0;
  const size_t nx = (P + kTmplPts * kThreads - 1) / (kTmplPts * kThreads);
  return nx * B * (size_t)(M + 1) * K;
}

cudaError_t launch_template_coeff(int P, int B, int M, int F, int G, const float* theta,
                                  const float* feat, float* coeff, float* rhs, cudaStream_t s) {
  TmplArgs t{};
  const int K = fill_exponents(F, G, t);
  t.R = M + 1;
  t.M = M;
  t.P = P;
  MPDE_TMPL_DISPATCH(run_coeff, t, B, theta, feat, coeff, rhs, s)
}

cudaError_t launch_template_grad(int P, int B, int M, int F, int G, const float* theta,
                                 const float* feat, const float* gc, const float* gb, float* gtheta,
                                 float* gfeat, double* part, cudaStream_t s) {
  TmplArgs t{};
  const int K = fill_exponents(F, G, t);
  t.R = M + 1;
  t.M = M;
  t.P = P;
  MPDE_TMPL_DISPATCH(run_grad, t, B, theta, feat, gc, gb, gtheta, gfeat, part, s)
}

}  // namespace mpde
