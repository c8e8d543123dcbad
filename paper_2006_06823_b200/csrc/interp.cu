// Periodic cubic B-spline sampling, SL departure points and the exact periodic
// prefilter (sm_100a).
//
// Replaces interp.hpp:65-210 (cubic_weights, wrap, ScalarSampler::eval_cubic /
// accumulate<4>, warp) and transport.hpp:83-102 (sl_departure).  Departure
// points are carried as DISPLACEMENTS in grid units (X = x + d*h) instead of
// the reference's absolute physical coordinates: floor(i + d) = i + floor(d)
// exactly, so the fp32 weights lose nothing to large coordinates.
#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

__device__ __forceinline__ void cubic_w(float t, float* w) {
  // interp.hpp:65-71
  const float t2 = t * t, t3 = t2 * t;
  w[0] = (1.0f - 3.0f * t + 3.0f * t2 - t3) * (1.0f / 6.0f);
  w[1] = (4.0f - 6.0f * t2 + 3.0f * t3) * (1.0f / 6.0f);
  w[2] = (1.0f + 3.0f * t + 3.0f * t2 - 3.0f * t3) * (1.0f / 6.0f);
  w[3] = t3 * (1.0f / 6.0f);
}

__device__ __forceinline__ int wrapi(int i, int n) {
  // interp.hpp:73-76 (periodic); fast path for the usual |i| < n case
  if (i < 0) i += n;
  if (i >= n) i -= n;
  if ((unsigned)i >= (unsigned)n) {
    i %= n;
    if (i < 0) i += n;
  }
  return i;
}

// Stencil for one point: node (i,j,k) plus displacement d (grid units).
struct Stencil {
  int ix[4], iy[4], iz[4];
  float wx[4], wy[4], wz[4];
};

__device__ __forceinline__ void make_stencil(int i, int j, int k, float dx, float dy, float dz, int Nx, int Ny,
                                             int Nz, Stencil& s) {
  const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
  cubic_w(dx - fx, s.wx);
  cubic_w(dy - fy, s.wy);
  cubic_w(dz - fz, s.wz);
  const int x0 = i + (int)fx - 1, y0 = j + (int)fy - 1, z0 = k + (int)fz - 1;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    s.ix[m] = wrapi(x0 + m, Nx);
    s.iy[m] = wrapi(y0 + m, Ny);
    s.iz[m] = wrapi(z0 + m, Nz);
  }
}

// accumulate<4> order of interp.hpp:145-156: sum_j0 sum_j1 (w0 w1) * sum_j2 w2 c
template <int F>
__device__ __forceinline__ void sample(const float* __restrict__ coef, long long N, int Ny, int Nz,
                                       const Stencil& s, float* out) {
#pragma unroll
  for (int c = 0; c < F; ++c) out[c] = 0.f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const long long row = ((long long)s.ix[a] * Ny + s.iy[b]) * Nz;
      const float w01 = s.wx[a] * s.wy[b];
#pragma unroll
      for (int c = 0; c < F; ++c) {
        const float* r = coef + c * N + row;
        float p = s.wz[0] * __ldg(r + s.iz[0]);
        p = fmaf(s.wz[1], __ldg(r + s.iz[1]), p);
        p = fmaf(s.wz[2], __ldg(r + s.iz[2]), p);
        p = fmaf(s.wz[3], __ldg(r + s.iz[3]), p);
        out[c] = fmaf(w01, p, out[c]);
      }
    }
  }
}

template <int F>
__global__ __launch_bounds__(256) void gather_cubic_kernel(const float* __restrict__ coef,
                                                           const float* __restrict__ disp,
                                                           float* __restrict__ out, int Nx, int Ny, int Nz) {
  const long long N = (long long)Nx * Ny * Nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N;
       p += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(p % Nz);
    const long long q = p / Nz;
    const int j = (int)(q % Ny);
    const int i = (int)(q / Ny);
    Stencil s;
    make_stencil(i, j, k, __ldg(disp + p), __ldg(disp + N + p), __ldg(disp + 2 * N + p), Nx, Ny, Nz, s);
    float v[F];
    sample<F>(coef, N, Ny, Nz, s, v);
#pragma unroll
    for (int c = 0; c < F; ++c) out[c * N + p] = v[c];
  }
}

void launch_gather_cubic(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                         cudaStream_t s) {
  const long long n = (long long)N[0] * N[1] * N[2];
  const int grid = grid_for(n, 256, 16);
  int done = 0;
  while (done < ncomp) {
    const int left = ncomp - done;
    const float* c = coef + (long long)done * n;
    float* o = out + (long long)done * n;
    if (left >= 6) {
      gather_cubic_kernel<6><<<grid, 256, 0, s>>>(c, disp, o, N[0], N[1], N[2]);
      done += 6;
    } else if (left >= 3) {
      gather_cubic_kernel<3><<<grid, 256, 0, s>>>(c, disp, o, N[0], N[1], N[2]);
      done += 3;
    } else {
      gather_cubic_kernel<1><<<grid, 256, 0, s>>>(c, disp, o, N[0], N[1], N[2]);
      done += 1;
    }
    LDDMM_LAUNCH_CHECK();
  }
}

// ---------------------------------------------------------------------------
// departure points (transport.hpp:83-102), both directions at once; stationary
// velocity: v_grid and v_traced are the same node.

__global__ __launch_bounds__(256) void departure_kernel(const float* __restrict__ vg, const float* __restrict__ vc,
                                                        float dtx, float dty, float dtz, float* __restrict__ df,
                                                        float* __restrict__ db, int Nx, int Ny, int Nz) {
  const long long N = (long long)Nx * Ny * Nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N;
       p += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(p % Nz);
    const long long q = p / Nz;
    const int j = (int)(q % Ny);
    const int i = (int)(q / Ny);
    // velocity in grid units per unit time scaled by dt: dt * v / h
    const float ux = __ldg(vg + p) * dtx, uy = __ldg(vg + N + p) * dty, uz = __ldg(vg + 2 * N + p) * dtz;
#pragma unroll
    for (int dir = 0; dir < (db ? 2 : 1); ++dir) {
      const float sg = dir == 0 ? -1.f : 1.f;
      Stencil s;
      make_stencil(i, j, k, sg * ux, sg * uy, sg * uz, Nx, Ny, Nz, s);
      float vm[3];
      sample<3>(vc, N, Ny, Nz, s, vm);
      float* o = dir == 0 ? df : db;
      o[p] = sg * 0.5f * (vm[0] * dtx + ux);
      o[N + p] = sg * 0.5f * (vm[1] * dty + uy);
      o[2 * N + p] = sg * 0.5f * (vm[2] * dtz + uz);
    }
  }
}

void launch_departure(const float* vgrid, const float* vcoef, double dt, const double* h, float* dep_fwd,
                      float* dep_bwd, const int* N, cudaStream_t s) {
  const long long n = (long long)N[0] * N[1] * N[2];
  departure_kernel<<<grid_for(n, 256, 16), 256, 0, s>>>(vgrid, vcoef, (float)(dt / h[0]), (float)(dt / h[1]),
                                                        (float)(dt / h[2]), dep_fwd, dep_bwd, N[0], N[1], N[2]);
  LDDMM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// pull-back through points x - disp (disp physical), used for m1 = I0 o phi1 etc.

template <int F>
__global__ __launch_bounds__(256) void warp_disp_kernel(const float* __restrict__ coef,
                                                        const float* __restrict__ disp, float ihx, float ihy,
                                                        float ihz, float* __restrict__ out, int Nx, int Ny,
                                                        int Nz) {
  const long long N = (long long)Nx * Ny * Nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N;
       p += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(p % Nz);
    const long long q = p / Nz;
    const int j = (int)(q % Ny);
    const int i = (int)(q / Ny);
    Stencil s;
    make_stencil(i, j, k, -__ldg(disp + p) * ihx, -__ldg(disp + N + p) * ihy, -__ldg(disp + 2 * N + p) * ihz, Nx,
                 Ny, Nz, s);
    float v[F];
    sample<F>(coef, N, Ny, Nz, s, v);
#pragma unroll
    for (int c = 0; c < F; ++c) out[c * N + p] = v[c];
  }
}

void launch_warp_by_displacement(const float* coef, int ncomp, const float* disp_phys, const double* h,
                                 float* out, const int* N, cudaStream_t s) {
  const long long n = (long long)N[0] * N[1] * N[2];
  const int grid = grid_for(n, 256, 16);
  const float ix = (float)(1.0 / h[0]), iy = (float)(1.0 / h[1]), iz = (float)(1.0 / h[2]);
  if (ncomp == 1)
    warp_disp_kernel<1><<<grid, 256, 0, s>>>(coef, disp_phys, ix, iy, iz, out, N[0], N[1], N[2]);
  else if (ncomp == 3)
    warp_disp_kernel<3><<<grid, 256, 0, s>>>(coef, disp_phys, ix, iy, iz, out, N[0], N[1], N[2]);
  else if (ncomp == 4)
    warp_disp_kernel<4><<<grid, 256, 0, s>>>(coef, disp_phys, ix, iy, iz, out, N[0], N[1], N[2]);
  else
    throw EngineError(3, "warp_by_displacement: unsupported component count");
  LDDMM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// exact periodic cubic B-spline prefilter along one axis (interp.hpp:23-63),
// one thread per line, in place (the causal pass overwrites the line with c+,
// the anticausal pass overwrites c+ with 6 c-).

template <typename T>
__global__ void prefilter_axis_kernel(T* __restrict__ v, int n, long long stride, long long lines,
                                      long long outer_stride) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < lines;
       l += (long long)gridDim.x * blockDim.x) {
    const long long o = l / stride, s = l % stride;
    T* base = v + o * outer_stride + s;
    const double z = -0.26794919243112270647;  // sqrt(3) - 2 (interp.hpp:18)
    double zn = 1.0;
    for (int m = 0; m < n; ++m) zn *= z;  // std::pow(z, n) to rounding
    const double denom = 1.0 - zn;
    double init = 0.0, zp = 1.0;
    for (int m = 0; m < n; ++m) {
      init += zp * (double)base[(long long)((n - m) % n) * stride];
      zp *= z;
    }
    double cp = init / denom;
    base[0] = (T)cp;
    for (int k = 1; k < n; ++k) {
      cp = (double)base[(long long)k * stride] + z * cp;
      base[(long long)k * stride] = (T)cp;
    }
    double tail = 0.0;
    zp = 1.0;
    for (int m = 0; m < n; ++m) {
      tail += zp * (double)base[(long long)((n - 1 + m) % n) * stride];
      zp *= z;
    }
    double cm = -z * tail / denom;
    base[(long long)(n - 1) * stride] = (T)(6.0 * cm);
    for (int k = n - 2; k >= 0; --k) {
      cm = z * (cm - (double)base[(long long)k * stride]);
      base[(long long)k * stride] = (T)(6.0 * cm);
    }
  }
}

template <typename T>
static void prefilter3d(T* f, const int* N, cudaStream_t s) {
  const long long total = (long long)N[0] * N[1] * N[2];
  for (int a = 0; a < 3; ++a) {
    const int n = N[a];
    if (n <= 1) continue;
    long long stride = 1;
    for (int b = a + 1; b < 3; ++b) stride *= N[b];
    const long long lines = total / n;
    prefilter_axis_kernel<T><<<grid_for(lines, 128, 32), 128, 0, s>>>(f, n, stride, lines, stride * n);
    LDDMM_LAUNCH_CHECK();
  }
}

// ---------------------------------------------------------------------------
// Full-grid spectral derivative along one axis (spectral.hpp:326-354): the symbol
// depends on k_a only, so the 3-D FFT / multiply / inverse FFT collapses to a
// real circulant convolution along that axis, out[i] = sum_j D[(i - j) mod n] in[j],
// with D the inverse DFT of i*omega (grid Nyquist zeroed), built in fp64 on the host.
__global__ void circulant_axis_kernel(const double* __restrict__ in, double* __restrict__ out,
                                      const double* __restrict__ D, int n, long long stride, long long total) {
  extern __shared__ double sD[];
  for (int t = threadIdx.x; t < n; t += blockDim.x) sD[t] = D[t];
  __syncthreads();
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    const long long inner = p % stride;
    const long long outer = p / stride;
    const int i = (int)(outer % n);
    const long long base = (outer / n) * n * stride + inner;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      int d = i - j;
      if (d < 0) d += n;
      acc = fma(sD[d], in[base + (long long)j * stride], acc);
    }
    out[p] = acc;
  }
}

void launch_circulant_axis_f64(const double* in, double* out, const double* D, int axis, const int* N,
                               cudaStream_t s) {
  long long stride = 1;
  for (int b = axis + 1; b < 3; ++b) stride *= N[b];
  const long long total = (long long)N[0] * N[1] * N[2];
  circulant_axis_kernel<<<grid_for(total, 256, 16), 256, N[axis] * sizeof(double), s>>>(in, out, D, N[axis],
                                                                                        stride, total);
  LDDMM_LAUNCH_CHECK();
}

void launch_prefilter3d(double* f, const int* N, cudaStream_t s) { prefilter3d<double>(f, N, s); }
void launch_prefilter3d_f32(float* f, const int* N, cudaStream_t s) { prefilter3d<float>(f, N, s); }

}  // namespace lddmm_b200
