// fp64 band-field algebra and deterministic reductions (sm_100a).
//
// Replaces spectral.hpp:112-185 (axpy, scaled, linf_norm, all_finite,
// band_inner), spectral.hpp:440-451 (band_divergence) and
// spectral.hpp:518-544 (SobolevOperator::apply on band fields).  Band vectors
// are tiny (K^3 complex per component), so these are latency-bound grid-stride
// loops; reductions are two-pass (per-block partials, then one block in fixed
// order) with warp-shuffle trees and fp64 accumulation, so results are
// bit-reproducible run to run.
#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

__global__ void axpby_kernel(long long n, double a, const double2* __restrict__ x, double b,
                             const double2* __restrict__ y, double2* __restrict__ out) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 xv = x[i];
    double2 r;
    if (y) {
      const double2 yv = y[i];
      if (b == 1.0) {
        // axpy: a*x + y evaluated like the reference (core.hpp:188-202)
        r = make_double2(a * xv.x + yv.x, a * xv.y + yv.y);
      } else {
        r = make_double2(a * xv.x + b * yv.x, a * xv.y + b * yv.y);
      }
    } else {
      r = make_double2(a * xv.x, a * xv.y);
    }
    out[i] = r;
  }
}

// out = sum_j w_j x_j over count vectors x_j = x + j stride, accumulated in order j = 0, 1,
// ... exactly as launch_scale(w_0) followed by launch_axpy(w_j, x_j, out, out) would (one
// launch instead of count)
struct WSum {
  double w[64];
};
__global__ void weighted_sum_kernel(long long n, int count, const __grid_constant__ WSum ws,
                                    const double2* __restrict__ x, long long stride, double2* __restrict__ out) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 x0 = x[i];
    double2 r = make_double2(ws.w[0] * x0.x, ws.w[0] * x0.y);
    for (int j = 1; j < count; ++j) {
      const double2 xv = x[j * stride + i];
      r = make_double2(ws.w[j] * xv.x + r.x, ws.w[j] * xv.y + r.y);
    }
    out[i] = r;
  }
}

void launch_weighted_sum(long long n, int count, const double* w, const double2* x, long long stride, double2* out,
                         cudaStream_t s) {
  if (count > 64) {
    launch_scale(n, w[0], x, out, s);
    for (int j = 1; j < count; ++j) launch_axpy(n, w[j], x + j * stride, out, out, s);
    return;
  }
  WSum ws;
  for (int j = 0; j < count; ++j) ws.w[j] = w[j];
  pdl_launch(weighted_sum_kernel, grid_for(n, 256, 4), 256, 0, s, n, count, ws, x, stride, out);
  LDDMM_LAUNCH_CHECK();
}

void launch_axpy(long long n, double a, const double2* x, const double2* y, double2* out, cudaStream_t s) {
  pdl_launch(axpby_kernel, grid_for(n, 256, 4), 256, 0, s, n, a, x, 1.0, y, out);
  LDDMM_LAUNCH_CHECK();
}
void launch_axpby(long long n, double a, const double2* x, double b, const double2* y, double2* out,
                  cudaStream_t s) {
  pdl_launch(axpby_kernel, grid_for(n, 256, 4), 256, 0, s, n, a, x, b, y, out);
  LDDMM_LAUNCH_CHECK();
}
void launch_scale(long long n, double a, const double2* x, double2* out, cudaStream_t s) {
  pdl_launch(axpby_kernel, grid_for(n, 256, 4), 256, 0, s, n, a, x, 0.0, nullptr, out);
  LDDMM_LAUNCH_CHECK();
}

__device__ __forceinline__ int signed_freq(int f, int K) { return f < K / 2 ? f : f - K; }

__global__ void sobolev_kernel(const double2* __restrict__ in, double2* __restrict__ out, int ncomp, int Kx,
                               int Ky, int Kz, double wx, double wy, double wz, double alpha, double s,
                               int inverse) {
  pdl_prologue();
  const long long per = (long long)Kx * Ky * Kz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per; i += (long long)gridDim.x * blockDim.x) {
    const int fz = (int)(i % Kz);
    const int fy = (int)((i / Kz) % Ky);
    const int fx = (int)(i / ((long long)Kz * Ky));
    const double ox = wx * signed_freq(fx, Kx), oy = wy * signed_freq(fy, Ky), oz = wz * signed_freq(fz, Kz);
    double w2 = 0.0;
    w2 += ox * ox;
    w2 += oy * oy;
    w2 += oz * oz;
    double m = pow(1.0 + alpha * w2, s);
    if (inverse) m = 1.0 / m;
    for (int c = 0; c < ncomp; ++c) {
      const double2 v = in[c * per + i];
      out[c * per + i] = make_double2(v.x * m, v.y * m);
    }
  }
}

void launch_sobolev(const double2* in, double2* out, int ncomp, const int* K, const double* wunit, double alpha,
                    int s, bool inverse, cudaStream_t st) {
  const long long per = (long long)K[0] * K[1] * K[2];
  pdl_launch(sobolev_kernel, grid_for(per, 256, 4), 256, 0, st, in, out, ncomp, K[0], K[1], K[2], wunit[0], wunit[1],
                                                         wunit[2], alpha, (double)s, inverse ? 1 : 0);
  LDDMM_LAUNCH_CHECK();
}

__global__ void divergence_kernel(const double2* __restrict__ v, double2* __restrict__ out, int Kx, int Ky, int Kz,
                                  double wx, double wy, double wz) {
  pdl_prologue();
  const long long per = (long long)Kx * Ky * Kz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per; i += (long long)gridDim.x * blockDim.x) {
    const int fz = (int)(i % Kz);
    const int fy = (int)((i / Kz) % Ky);
    const int fx = (int)(i / ((long long)Kz * Ky));
    const double om[3] = {wx * signed_freq(fx, Kx), wy * signed_freq(fy, Ky), wz * signed_freq(fz, Kz)};
    double sx = 0.0, sy = 0.0;
    for (int a = 0; a < 3; ++a) {
      const double2 c = v[a * per + i];
      // c * (0 + i om) = (-c.y om) + i (c.x om)
      sx += -c.y * om[a];
      sy += c.x * om[a];
    }
    out[i] = make_double2(sx, sy);
  }
}

void launch_band_divergence(const double2* v, double2* out, const int* K, const double* wunit, cudaStream_t s) {
  const long long per = (long long)K[0] * K[1] * K[2];
  pdl_launch(divergence_kernel, grid_for(per, 256, 4), 256, 0, s, v, out, K[0], K[1], K[2], wunit[0], wunit[1], wunit[2]);
  LDDMM_LAUNCH_CHECK();
}

// ---- reductions -----------------------------------------------------------------

__global__ __launch_bounds__(256) void inner_partial_kernel(long long n, const double2* __restrict__ x,
                                                            const double2* __restrict__ y, double* part) {
  pdl_prologue();
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i], b = y[i];
    s += a.x * b.x + a.y * b.y;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ __launch_bounds__(256) void linf_partial_kernel(long long n, const double2* __restrict__ x, double* part) {
  pdl_prologue();
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i];
    m = fmax(m, hypot(a.x, a.y));
  }
  m = block_max(m);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ __launch_bounds__(256) void nonfinite_partial_kernel(long long n, const double2* __restrict__ x,
                                                                double* part) {
  pdl_prologue();
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i];
    if (!isfinite(a.x) || !isfinite(a.y)) m = 1.0;
  }
  m = block_max(m);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ __launch_bounds__(1024) void reduce_final_kernel(const double* __restrict__ part, int n, int op,
                                                            double* slot) {
  pdl_prologue();
  double v = op == 0 ? 0.0 : -INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v = op == 0 ? v + part[i] : fmax(v, part[i]);
  v = op == 0 ? block_sum(v) : block_max(v);
  if (threadIdx.x == 0) *slot = v;
}

static int red_grid(long long n) {
  long long g = (n + 255) / 256;
  if (g > kReduceBlocks) g = kReduceBlocks;
  return (int)(g < 1 ? 1 : g);
}

int launch_inner_partial(long long n, const double2* x, const double2* y, double* part, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(inner_partial_kernel, g, 256, 0, s, n, x, y, part);
  LDDMM_LAUNCH_CHECK();
  return g;
}
int launch_linf_partial(long long n, const double2* x, double* part, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(linf_partial_kernel, g, 256, 0, s, n, x, part);
  LDDMM_LAUNCH_CHECK();
  return g;
}
// Non-finite flag in one launch: block maxima into part[0..g), and the last block to
// finish (counter in part[kReduceBlocks], reset by that block) reduces them into slot —
// the same max of 0/1 flags as nonfinite_partial + reduce_final.
__global__ __launch_bounds__(256) void nonfinite_flag_kernel(long long n, const double2* __restrict__ x, double* part,
                                                             double* slot) {
  pdl_prologue();
  unsigned* counter = reinterpret_cast<unsigned*>(part + kReduceBlocks);
  __shared__ bool last;
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i];
    if (!isfinite(a.x) || !isfinite(a.y)) m = 1.0;
  }
  m = block_max(m);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = m;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double v = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v = fmax(v, reinterpret_cast<volatile double*>(part)[b]);
    v = block_max(v);
    if (threadIdx.x == 0) {
      *slot = v;
      *counter = 0u;
    }
  }
}

void launch_nonfinite_flag(long long n, const double2* x, double* part, double* slot, cudaStream_t s) {
  pdl_launch(nonfinite_flag_kernel, red_grid(n), 256, 0, s, n, x, part, slot);
  LDDMM_LAUNCH_CHECK();
}

// Non-finite flags of `count` consecutive series nodes (node j = base + j V) in one
// launch: a thread that meets a non-finite value stores 1 into its node's step slot
// (every writer stores the same value); the slots are zeroed by the caller beforehand.
// Step of node j: step0 + j, or step0 + count - 1 - j for a backward march.
__global__ __launch_bounds__(256) void nonfinite_series_kernel(const double2* __restrict__ base, long long V,
                                                               int count, int step0, int backward,
                                                               double* __restrict__ slots) {
  pdl_prologue();
  const long long n = V * count;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = base[i];
    if (!isfinite(a.x) || !isfinite(a.y)) {
      const int j = (int)(i / V);
      slots[backward ? step0 + count - 1 - j : step0 + j] = 1.0;
    }
  }
}

void launch_nonfinite_series(const double2* base, long long V, int count, int step0, bool backward, double* slots,
                             cudaStream_t s) {
  LDDMM_CUDA(cudaMemsetAsync(slots + step0, 0, count * sizeof(double), s));
  pdl_launch(nonfinite_series_kernel, grid_for(V * count, 256), 256, 0, s, base, V, count, step0, backward ? 1 : 0,
             slots);
  LDDMM_LAUNCH_CHECK();
}

int launch_nonfinite_partial(long long n, const double2* x, double* part, cudaStream_t s) {
  const int g = red_grid(n);
  pdl_launch(nonfinite_partial_kernel, g, 256, 0, s, n, x, part);
  LDDMM_LAUNCH_CHECK();
  return g;
}
void launch_reduce_final(const double* part, int nparts, int op, double* slot, cudaStream_t s) {
  pdl_launch(reduce_final_kernel, 1, 1024, 0, s, part, nparts, op, slot);
  LDDMM_LAUNCH_CHECK();
}

}  // namespace lddmm_b200

namespace lddmm_b200 {

// *mismatch = number of CTAs that saw a[i] != b[i] bitwise (0: the arrays are equal)
__global__ void equal_flag_kernel(long long n, const double* __restrict__ a, const double* __restrict__ b,
                                  unsigned long long* mismatch) {
  pdl_prologue();
  bool same = true;
  GRID_STRIDE(i, n) same = same && (__double_as_longlong(a[i]) == __double_as_longlong(b[i]));
  if (__syncthreads_or(!same) && threadIdx.x == 0) atomicAdd(mismatch, 1ULL);
}

void launch_equal_flag(long long n, const double* a, const double* b, unsigned long long* mismatch, cudaStream_t s) {
  LDDMM_CUDA(cudaMemsetAsync(mismatch, 0, sizeof(unsigned long long), s));
  pdl_launch(equal_flag_kernel, grid_for(n, 256, 4), 256, 0, s, n, a, b, mismatch);
  LDDMM_LAUNCH_CHECK();
}

}  // namespace lddmm_b200
