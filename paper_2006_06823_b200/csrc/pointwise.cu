// Grid-pointwise kernels (fp32 fields, fp64 reductions) (sm_100a).
//
// Residual/energy (variants.hpp:272-274,428), the adjoint terminal sources
// r1 / dr1 (variants.hpp:326-336,431), the truncated-product integrands
// star / star_dot / band_jac(T)_mul evaluated on the small product grid
// (spectral.hpp:460-510), and det(I - Du) (metrics.hpp:40-65).  All
// HBM-bound; each field is touched once.
#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

__global__ void f64_to_f32_kernel(long long n, const double* __restrict__ in, float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) out[i] = (float)in[i];
}
__global__ void f32_to_f64_kernel(long long n, const float* __restrict__ in, double* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) out[i] = (double)in[i];
}
void launch_f64_to_f32(long long n, const double* in, float* out, cudaStream_t s) {
  pdl_launch(f64_to_f32_kernel, grid_for(n, 256), 256, 0, s, n, in, out);
  LDDMM_LAUNCH_CHECK();
}
void launch_f32_to_f64(long long n, const float* in, double* out, cudaStream_t s) {
  pdl_launch(f32_to_f64_kernel, grid_for(n, 256), 256, 0, s, n, in, out);
  LDDMM_LAUNCH_CHECK();
}

static int red_grid(long long n) {
  long long g = (n + 255) / 256;
  if (g > kReduceBlocks) g = kReduceBlocks;
  return (int)(g < 1 ? 1 : g);
}

__global__ __launch_bounds__(256) void residual_kernel(long long n, const float* __restrict__ m1,
                                                       const float* __restrict__ I1, float* __restrict__ res,
                                                       double* part) {
  pdl_prologue();
  double s = 0.0;
  GRID_STRIDE(i, n) {
    const float r = m1[i] - I1[i];
    res[i] = r;
    s += (double)r * (double)r;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
int launch_residual(long long n, const float* m1, const float* I1, float* res, double* part, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(residual_kernel, g, 256, 0, s, n, m1, I1, res, part);
  LDDMM_LAUNCH_CHECK();
  return g;
}

__global__ __launch_bounds__(256) void sumsq_kernel(long long n, const float* __restrict__ x, double* part) {
  pdl_prologue();
  double s = 0.0;
  GRID_STRIDE(i, n) s += (double)x[i] * (double)x[i];
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
int launch_sumsq_partial(long long n, const float* x, double* part, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(sumsq_kernel, g, 256, 0, s, n, x, part);
  LDDMM_LAUNCH_CHECK();
  return g;
}

__global__ __launch_bounds__(256) void absmax_kernel(long long n, const float* __restrict__ x, double* part) {
  pdl_prologue();
  double m = 0.0;
  GRID_STRIDE(i, n) m = fmax(m, (double)fabsf(x[i]));
  m = block_max(m);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}
int launch_absmax_partial(long long n, const float* x, double* part, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(absmax_kernel, g, 256, 0, s, n, x, part);
  LDDMM_LAUNCH_CHECK();
  return g;
}

__global__ void scale_vec_kernel(long long n, const float* __restrict__ res, float c, const float* __restrict__ g,
                                 float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) {
    const float r = res[i] * c;
    out[i] = r * g[i];
    out[n + i] = r * g[n + i];
    out[2 * n + i] = r * g[2 * n + i];
  }
}
void launch_scale_vec(long long n, const float* res, double c, const float* g, float* out, cudaStream_t s) {
  pdl_launch(scale_vec_kernel, grid_for(n, 256), 256, 0, s, n, res, (float)c, g, out);
  LDDMM_LAUNCH_CHECK();
}

__global__ void dr1_kernel(long long n, const float* __restrict__ g, const float* __restrict__ du, float c,
                           float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) {
    const float g0 = g[i], g1 = g[n + i], g2 = g[2 * n + i];
    float dm = 0.f;
    dm += g0 * du[i];
    dm += g1 * du[n + i];
    dm += g2 * du[2 * n + i];
    const float dl = (-dm) * c;
    out[i] = dl * g0;
    out[n + i] = dl * g1;
    out[2 * n + i] = dl * g2;
  }
}
void launch_dr1(long long n, const float* g, const float* du, double c, float* out, cudaStream_t s) {
  pdl_launch(dr1_kernel, grid_for(n, 256), 256, 0, s, n, g, du, (float)c, out);
  LDDMM_LAUNCH_CHECK();
}

// dlam1 = ((-1 * sum_b g_b du_b) * c)   (variants.hpp:326-327, state branch)
__global__ void dlam1_kernel(long long n, const float* __restrict__ g, const float* __restrict__ du, float c,
                             float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) {
    float dm = 0.f;
    dm += g[i] * du[i];
    dm += g[n + i] * du[n + i];
    dm += g[2 * n + i] * du[2 * n + i];
    out[i] = (-dm) * c;
  }
}
void launch_dlam1(long long n, const float* g, const float* du, double c, float* out, cudaStream_t s) {
  pdl_launch(dlam1_kernel, grid_for(n, 256), 256, 0, s, n, g, du, (float)c, out);
  LDDMM_LAUNCH_CHECK();
}

// a: derivative fields / scalars, b: factors; layouts:
//  op 0 jac : a = D[a][b][n] (d_b u_a), b = w[b][n] -> acc[a] += sum_b D[a][b] w[b]
//  op 1 jacT: a = D[a][b][n],           b = w[a][n] -> acc[b] += sum_a D[a][b] w[a]
//  op 2 s*v : a = s[n], b = x[c][n]                 -> acc[c] += s x[c]
//  op 3 dot : a = x[c][n], b = y[c][n]              -> acc    += sum_c x[c] y[c]
//  op 4 s*s : a = s[n], b = t[n]                    -> acc    += s t
__global__ void products_kernel(int op, long long n, const float* __restrict__ A, const float* __restrict__ B,
                                float* __restrict__ acc, float w, int init) {
  pdl_prologue();
  GRID_STRIDE(i, n) {
    if (op == 0 || op == 1) {
      float o[3] = {0.f, 0.f, 0.f};
      if (op == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) o[a] += A[(a * 3 + b) * n + i] * B[b * n + i];
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) o[b] += A[(a * 3 + b) * n + i] * B[a * n + i];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c * n + i] = (init ? 0.f : acc[c * n + i]) + w * o[c];
    } else if (op == 2) {
      const float s = A[i];
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c * n + i] = (init ? 0.f : acc[c * n + i]) + w * (s * B[c * n + i]);
    } else if (op == 3) {
      float d = 0.f;
#pragma unroll
      for (int c = 0; c < 3; ++c) d += A[c * n + i] * B[c * n + i];
      acc[i] = (init ? 0.f : acc[i]) + w * d;
    } else {
      acc[i] = (init ? 0.f : acc[i]) + w * (A[i] * B[i]);
    }
  }
}
void launch_products(int op, long long n, const float* a, const float* b, float* acc, float w, bool init,
                     cudaStream_t s) {
  pdl_launch(products_kernel, grid_for(n, 256), 256, 0, s, op, n, a, b, acc, w, init ? 1 : 0);
  LDDMM_LAUNCH_CHECK();
}

__global__ void jac_batch_kernel(int transpose, int nn, long long M, const float* __restrict__ D,
                                 const float* __restrict__ W, long long wstride, float* __restrict__ out,
                                 long long ostride, NodeWeights wts, int init) {
  pdl_prologue();
  GRID_STRIDE(i, M) {
    float acc[3] = {0.f, 0.f, 0.f};
    if (ostride == 0 && !init) {
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] = out[c * M + i];
    }
    for (int n = 0; n < nn; ++n) {
      const float* d = D + (long long)n * 9 * M;
      const float* w = W + (long long)n * wstride;
      float o[3] = {0.f, 0.f, 0.f};
      if (!transpose) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) o[a] += d[(a * 3 + b) * M + i] * w[b * M + i];
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) o[b] += d[(a * 3 + b) * M + i] * w[a * M + i];
      }
      if (ostride == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += wts.w[n] * o[c];
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) out[n * ostride + c * M + i] = o[c];
      }
    }
    if (ostride == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c * M + i] = acc[c];
    }
  }
}
void launch_jac_batch(bool transpose, int nn, long long M, const float* derivs, const float* w,
                      long long w_node_stride, float* out, long long out_stride, NodeWeights wts, bool init,
                      cudaStream_t s) {
  pdl_launch(jac_batch_kernel, grid_for(M, 256), 256, 0, s, transpose ? 1 : 0, nn, M, derivs, w, w_node_stride, out,
                                                    out_stride, wts, init ? 1 : 0);
  LDDMM_LAUNCH_CHECK();
}

__device__ __forceinline__ double det3(const float* du, long long n, long long i) {
  double m[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) m[a][b] = (a == b ? 1.0 : 0.0) - (double)du[(a * 3 + b) * n + i];
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

__global__ __launch_bounds__(256) void jacdet_minmax_kernel(long long n, const float* __restrict__ du,
                                                            double* pmin, double* pmax) {
  pdl_prologue();
  double lo = 1e300, hi = -1e300;
  GRID_STRIDE(i, n) {
    const double d = det3(du, n, i);
    lo = fmin(lo, d);
    hi = fmax(hi, d);
  }
  hi = block_max(hi);
  lo = -block_max(-lo);
  if (threadIdx.x == 0) {
    pmin[blockIdx.x] = -lo;  // stored negated so both reduce with max
    pmax[blockIdx.x] = hi;
  }
}
int launch_jacdet_minmax(long long n, const float* du, double* part_min, double* part_max, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(jacdet_minmax_kernel, g, 256, 0, s, n, du, part_min, part_max);
  LDDMM_LAUNCH_CHECK();
  return g;
}
__global__ void jacdet_kernel(long long n, const float* __restrict__ du, float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) out[i] = (float)det3(du, n, i);
}
void launch_jacdet(long long n, const float* du, float* out, cudaStream_t s) {
  pdl_launch(jacdet_kernel, grid_for(n, 256), 256, 0, s, n, du, out);
  LDDMM_LAUNCH_CHECK();
}

// Dice counts (metrics.hpp:100-118): per-block shared counters, one atomic per
// counter per block.  Exact integer counts, so the host-side Dice ratio is
// bitwise the reference's.
constexpr int DICE_MAXL = 64;
__global__ __launch_bounds__(256) void dice_counts_kernel(long long n, const float* __restrict__ a,
                                                          const float* __restrict__ b,
                                                          const float* __restrict__ labels, int nl,
                                                          unsigned long long* counts) {
  pdl_prologue();
  __shared__ unsigned int sc[3 * DICE_MAXL];
  __shared__ float sl[DICE_MAXL];
  for (int t = threadIdx.x; t < 3 * DICE_MAXL; t += blockDim.x) sc[t] = 0u;
  for (int t = threadIdx.x; t < nl; t += blockDim.x) sl[t] = labels[t];
  __syncthreads();
  GRID_STRIDE(i, n) {
    const float x = a[i], y = b[i];
    for (int l = 0; l < nl; ++l) {
      const bool ia = x == sl[l], ib = y == sl[l];
      if (ia) atomicAdd(&sc[3 * l], 1u);
      if (ib) atomicAdd(&sc[3 * l + 1], 1u);
      if (ia && ib) atomicAdd(&sc[3 * l + 2], 1u);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 3 * nl; t += blockDim.x)
    if (sc[t]) atomicAdd(counts + t, (unsigned long long)sc[t]);
}

void launch_dice_counts(long long n, const float* a, const float* b, const float* labels, int nl,
                        unsigned long long* counts, cudaStream_t s) {
  LDDMM_CUDA(cudaMemsetAsync(counts, 0, 3 * (size_t)nl * sizeof(unsigned long long), s));
  for (int l0 = 0; l0 < nl; l0 += DICE_MAXL) {
    const int m = nl - l0 < DICE_MAXL ? nl - l0 : DICE_MAXL;
    pdl_launch(dice_counts_kernel, grid_for(n, 256), 256, 0, s, n, a, b, labels + l0, m, counts + 3 * l0);
    LDDMM_LAUNCH_CHECK();
  }
}

__global__ void affine_kernel(long long n, const float* __restrict__ x, float a, float b, float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) out[i] = a * x[i] + b;
}
void launch_affine_f32(long long n, const float* x, float a, float b, float* out, cudaStream_t s) {
  pdl_launch(affine_kernel, grid_for(n, 256), 256, 0, s, n, x, a, b, out);
  LDDMM_LAUNCH_CHECK();
}
__global__ void mul_kernel(long long n, const float* __restrict__ x, const float* __restrict__ y,
                           float* __restrict__ out) {
  pdl_prologue();
  GRID_STRIDE(i, n) out[i] = x[i] * y[i];
}
void launch_mul_f32(long long n, const float* x, const float* y, float* out, cudaStream_t s) {
  pdl_launch(mul_kernel, grid_for(n, 256), 256, 0, s, n, x, y, out);
  LDDMM_LAUNCH_CHECK();
}

}  // namespace lddmm_b200
