// Device helpers shared by the SL cubic gathers (interp.cu, gather_pipe.cu):
// cubic B-spline weights (interp.hpp:65-71), periodic wrap (interp.hpp:73-76), the
// 5-tap window weights of the sub-voxel regime and the global-memory per-point path.
#pragma once

#include "common.cuh"

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

// one cubic weight (same expressions as cubic_w)
__device__ __forceinline__ float cubic_w1(float t, int a) {
  const float t2 = t * t, t3 = t2 * t;
  if (a == 0) return (1.0f - 3.0f * t + 3.0f * t2 - t3) * (1.0f / 6.0f);
  if (a == 1) return (4.0f - 6.0f * t2 + 3.0f * t3) * (1.0f / 6.0f);
  if (a == 2) return (1.0f + 3.0f * t + 3.0f * t2 - 3.0f * t3) * (1.0f / 6.0f);
  return t3 * (1.0f / 6.0f);
}

// Out-of-tile point (|floor(d)| > 1 on some axis): taps straight from global memory,
// compact loops (rare path; keeps the register budget of the tiled kernel).
template <int FG>
__device__ __forceinline__ void gather_point_global(const float* __restrict__ coef, const float* __restrict__ disp,
                                                    int i, int j, int k, int Nx, int Ny, int Nz, int nc, float* v,
                                                    float3 sc) {
  const long long N = (long long)Nx * Ny * Nz;
  const long long p = ((long long)i * Ny + j) * Nz + k;
  const float dx = sc.x * __ldg(disp + p), dy = sc.y * __ldg(disp + N + p), dz = sc.z * __ldg(disp + 2 * N + p);
  const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
  const float tx = dx - fx, ty = dy - fy, tz = dz - fz;
  const int xb = i + (int)fx - 1, yb = j + (int)fy - 1, zb = k + (int)fz - 1;
  for (int c = 0; c < FG; ++c) v[c] = 0.f;
#pragma unroll 1
  for (int a = 0; a < 4; ++a) {
    const float wa = cubic_w1(tx, a);
    const int ix = wrapi(xb + a, Nx);
#pragma unroll 1
    for (int b = 0; b < 4; ++b) {
      const float w01 = wa * cubic_w1(ty, b);
      const long long row = ((long long)ix * Ny + wrapi(yb + b, Ny)) * Nz;
      const int z0 = wrapi(zb, Nz), z1 = wrapi(zb + 1, Nz), z2 = wrapi(zb + 2, Nz), z3 = wrapi(zb + 3, Nz);
      for (int c = 0; c < nc; ++c) {
        const float* r = coef + c * N + row;
        float pp = cubic_w1(tz, 0) * __ldg(r + z0);
        pp = fmaf(cubic_w1(tz, 1), __ldg(r + z1), pp);
        pp = fmaf(cubic_w1(tz, 2), __ldg(r + z2), pp);
        pp = fmaf(cubic_w1(tz, 3), __ldg(r + z3), pp);
        v[c] = fmaf(w01, pp, v[c]);
      }
    }
  }
}

// 5-tap window weights for |floor(d)| <= 1: taps -2..2 with the zero weight first
// (d >= 0) or last (d < 0), so the sum is bitwise the reference's 4-tap accumulate<4>.
__device__ __forceinline__ void w5(float d, float f, float* w) {
  float w4[4];
  cubic_w(d - f, w4);
  const bool lo = f < 0.f;  // taps -2..1, else -1..2
  w[0] = lo ? w4[0] : 0.f;
  w[1] = lo ? w4[1] : w4[0];
  w[2] = lo ? w4[2] : w4[1];
  w[3] = lo ? w4[3] : w4[2];
  w[4] = lo ? 0.f : w4[3];
}

}  // namespace lddmm_b200
