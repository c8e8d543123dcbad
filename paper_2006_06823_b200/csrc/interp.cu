// Periodic cubic B-spline sampling, SL departure points and the exact periodic
// prefilter (sm_100a).
//
// Replaces interp.hpp:65-210 (cubic_weights, wrap, ScalarSampler::eval_cubic /
// accumulate<4>, warp) and transport.hpp:83-102 (sl_departure).  Departure
// points are carried as DISPLACEMENTS in grid units (X = x + d*h) instead of
// the reference's absolute physical coordinates: floor(i + d) = i + floor(d)
// exactly, so the fp32 weights lose nothing to large coordinates.
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "kernels.cuh"
#include "gather_common.cuh"

namespace lddmm_b200 {


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
                                                           float* __restrict__ out, int Nx, int Ny, int Nz,
                                                           float3 sc) {
  pdl_prologue();
  const long long N = (long long)Nx * Ny * Nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N;
       p += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(p % Nz);
    const long long q = p / Nz;
    const int j = (int)(q % Ny);
    const int i = (int)(q / Ny);
    Stencil s;
    make_stencil(i, j, k, sc.x * __ldg(disp + p), sc.y * __ldg(disp + N + p), sc.z * __ldg(disp + 2 * N + p), Nx,
                 Ny, Nz, s);
    float v[F];
    sample<F>(coef, N, Ny, Nz, s, v);
#pragma unroll
    for (int c = 0; c < F; ++c) out[c * N + p] = v[c];
  }
}

// ---------------------------------------------------------------------------
// Shared-memory tiled gather.  A CTA owns an 8 x 8 x 32 block of output nodes
// and stages the periodic 12 x 12 x 36 source box (halo 2) of up to 3
// components at a time.  With |floor(d)| <= 1 per axis (departure CFL < 1,
// the regime SL runs in) every 64-tap stencil lies in the box: each tap is one
// conflict-free LDS (a warp covers 32 consecutive z of one row) instead of an
// L1 global load whose lanes straddle rows.  Points outside that regime read
// their taps from global memory (same arithmetic, same order).
constexpr int GT_X = 8, GT_Y = 8, GT_Z = 32, GT_H = 2;
constexpr int GS_X = GT_X + 2 * GT_H, GS_Y = GT_Y + 2 * GT_H;
// z pitch of a staged row is 64 words (36 used): rows differ by multiples of 32
// banks, so a warp whose lanes straddle two rows (floor(d) changes along z) stays
// bank-conflict free.
constexpr int GS_ZUSED = GT_Z + 2 * GT_H, GS_Z = 64;
constexpr int GS_VOL = GS_X * GS_Y * GS_Z;
constexpr int GT_THREADS = 512;
constexpr int GT_PTS = GT_X * GT_Y * GT_Z / GT_THREADS;  // 4 points per thread

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(float* smem, const float* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(float* smem, const float* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }


template <int FG>
__global__ __launch_bounds__(GT_THREADS, 2) void gather_tiled_kernel(const float* __restrict__ coef, int F,
                                                                  const float* __restrict__ disp,
                                                                  float* __restrict__ out, int Nx, int Ny, int Nz,
                                                                  float3 sc) {
  pdl_prologue();
  extern __shared__ float sm[];
  const long long N = (long long)Nx * Ny * Nz;
  const int x0 = blockIdx.x * GT_X, y0 = blockIdx.y * GT_Y, z0 = blockIdx.z * GT_Z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this thread's points: rows warp*4 .. warp*4+3 of the 64 (x, y) rows, z = z0 + lane;
  // the (cheap) per-point stencil set-up is redone per component group so that no
  // per-point state is carried in registers across the staging barriers.
  for (int c0 = 0; c0 < F; c0 += FG) {
    const int nc = min(FG, F - c0);
    __syncthreads();
    {
      // one warp per staged row: lanes copy z = z0-2 .. z0+33 (wrapped) with
      // cp.async (LDGSTS), all rows in flight before one wait
      const int gz0 = wrapi(z0 - GT_H + lane, Nz);
      const int gz1 = wrapi(z0 - GT_H + 32 + (lane & 3), Nz);
      for (int row = warp; row < nc * GS_X * GS_Y; row += GT_THREADS / 32) {
        const int c = row / (GS_X * GS_Y);
        const int rr = row - c * (GS_X * GS_Y);
        const int ix = rr / GS_Y, jy = rr % GS_Y;
        const float* src = coef + (c0 + c) * N +
                           ((long long)wrapi(x0 - GT_H + ix, Nx) * Ny + wrapi(y0 - GT_H + jy, Ny)) * Nz;
        float* dst = sm + c * GS_VOL + rr * GS_Z;
        cp_async4(dst + lane, src + gz0);
        if (lane < GS_ZUSED - 32) cp_async4(dst + 32 + lane, src + gz1);
      }
      cp_async_wait_all();
    }
    __syncthreads();
#pragma unroll 1
    for (int q = 0; q < GT_PTS; ++q) {
      const int r = warp * GT_PTS + q;
      const int rx = r / GT_Y, ry = r % GT_Y;
      const int i = x0 + rx, j = y0 + ry, k = z0 + lane;
      if (i >= Nx || j >= Ny || k >= Nz) continue;
      const long long p = ((long long)i * Ny + j) * Nz + k;
      const float dx = sc.x * __ldg(disp + p), dy = sc.y * __ldg(disp + N + p), dz = sc.z * __ldg(disp + 2 * N + p);
      const float fx = floorf(dx), fy = floorf(dy), fz = floorf(dz);
      float v[FG];
      if (fx >= -1.f && fx <= 0.f && fy >= -1.f && fy <= 0.f && fz >= -1.f && fz <= 0.f) {
        // x, y: the 4 rows selected by floor(d); z: a fixed 5-tap window z-2..z+2
        // (one weight exactly zero), so a warp's 32 lanes always read 32
        // consecutive words -> conflict-free whatever floor(dz) does along z.  The
        // zero-weight tap comes first or last, so the sum is bitwise the 4-tap one.
        const int lb = ((rx + GT_H + (int)fx - 1) * GS_Y + (ry + GT_H + (int)fy - 1)) * GS_Z + lane;
        float wx[4], wy[4], w4[4], wz[5];
        cubic_w(dx - fx, wx);
        cubic_w(dy - fy, wy);
        cubic_w(dz - fz, w4);
        const bool lo = fz < 0.f;  // taps z-2..z+1
        wz[0] = lo ? w4[0] : 0.f;
        wz[1] = lo ? w4[1] : w4[0];
        wz[2] = lo ? w4[2] : w4[1];
        wz[3] = lo ? w4[3] : w4[2];
        wz[4] = lo ? 0.f : w4[3];
#pragma unroll
        for (int c = 0; c < FG; ++c) v[c] = 0.f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int row = lb + (a * GS_Y + b) * GS_Z;
            const float w01 = wx[a] * wy[b];
#pragma unroll
            for (int c = 0; c < FG; ++c) {
              const float* rr = sm + c * GS_VOL + row;
              float pp = wz[0] * rr[0];
              pp = fmaf(wz[1], rr[1], pp);
              pp = fmaf(wz[2], rr[2], pp);
              pp = fmaf(wz[3], rr[3], pp);
              pp = fmaf(wz[4], rr[4], pp);
              v[c] = fmaf(w01, pp, v[c]);
            }
          }
        }
      } else {
        gather_point_global<FG>(coef + c0 * N, disp, i, j, k, Nx, Ny, Nz, nc, v, sc);
      }
#pragma unroll
      for (int c = 0; c < FG; ++c)
        if (c < nc) out[(c0 + c) * N + p] = v[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Register-window gather (the production path).  A CTA owns TX x TY full
// z-rows of output nodes and stages the periodic (TX+4) x (TY+4) source rows of
// up to FG components in shared memory (row pitch P >= Nz + 4, a compile-time
// constant so every row address below is an immediate offset, z halo 2).  A
// thread evaluates FOUR consecutive z nodes of one row: for every source row of
// the 5 x 5 (x, y) neighbourhood it loads one aligned 8-float window (two
// LDS.128) covering the 5-tap z stencils of the four nodes.  Every axis uses
// the fixed 5-tap window [-2, 2] with the zero weight first or last
// (|floor(d)| <= 1, the SL regime): the sum is bitwise the reference's 4-tap
// accumulate<4> (interp.hpp:145-156), same x-outer / y-inner order.  Nodes
// outside that regime fall back to the global-memory path.
//
// The component count of a group (NC) is a template parameter, so the 25-row
// loop is branch-free straight-line code the scheduler can interleave across
// components.  Node pairs (0,1) and (2,3) share FFMA2 instructions where their
// taps form an aligned register pair (even taps); odd taps use scalar FFMA
// (a packed operand there would cost two MOVs).
constexpr int GW_H = 2;


__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

// Staged row layout.  SHIFT = false (any even Nz): smem index i holds z = i - 2,
// 8-byte cp.async.  SHIFT = true (Nz % 4 == 0): index i holds z = i - 4 and the
// node groups are shifted by -2 (group g = nodes 4g-2 .. 4g+1, group 0 wrapping
// to Nz-2, Nz-1, 0, 1), so both the staging copies (16-byte cp.async.cg) and the
// per-group windows (indices 4g .. 4g+7) are 16-byte aligned.
template <int TX, int TY, int NTH, bool SHIFT>
__device__ __forceinline__ void gw_stage(float* dst_base, const float* __restrict__ coef, long long N, int c0, int nc,
                                         int x0, int y0, int Nx, int Ny, int Nz, int RL) {
  constexpr int SX = TX + 2 * GW_H, SY = TY + 2 * GW_H;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cvol = SX * SY * RL;
  const int zlen = SHIFT ? Nz + 8 : ((Nz + 3) & ~3) + 2 * GW_H;
  for (int row = warp; row < nc * SX * SY; row += NTH / 32) {
    const int c = row / (SX * SY);
    const int rr = row - c * (SX * SY);
    const int ix = rr / SY, jy = rr - (rr / SY) * SY;
    const float* src =
        coef + (c0 + c) * N + ((long long)wrapi(x0 - GW_H + ix, Nx) * Ny + wrapi(y0 - GW_H + jy, Ny)) * Nz;
    float* dst = dst_base + c * cvol + rr * RL;
    if (SHIFT) {
      // 16-byte copies: z = zz - 4 is a multiple of 4, the periodic wrap falls on
      // 4-float boundaries
      for (int zz = 4 * lane; zz < zlen; zz += 128) {
        int gz = zz - 4;
        gz += gz < 0 ? Nz : 0;
        gz -= gz >= Nz ? Nz : 0;
        cp_async16_cg(dst + zz, src + gz);
      }
    } else {
      // 8-byte copies: Nz is even, so every pair (z, z+1), z = zz - 2 even, is
      // contiguous in global memory even across the periodic wrap
      for (int zz = 2 * lane; zz < zlen; zz += 64) {
        int gz = zz - GW_H;
        gz += gz < 0 ? Nz : 0;
        gz -= gz >= Nz ? Nz : 0;
        cp_async8(dst + zz, src + gz);
      }
    }
  }
}

// One 4-node z group of output row (i, j): departure displacements, the SL-regime
// check (else the global-memory path), weights, the 5 x 5 source rows pl[a] + b P
// (pl[a] = the staged x-plane a of the neighbourhood, offset to the group's first
// y row and z window; components CVOL apart) and the stores.
template <int NC, int P, int CVOL, bool SHIFT>
__device__ __forceinline__ void gw_item(const float* const (&pl)[5], const float* __restrict__ coef,
                                        const float* __restrict__ disp, float* __restrict__ out, long long N, int c0,
                                        int i, int j, int g, int Nx, int Ny, int Nz, float3 sc) {
  const bool vec = (Nz & 3) == 0;
  const long long rowp0 = ((long long)i * Ny + j) * Nz;
  // z of nodes (0,1) and (2,3) of the group
  const int zA = SHIFT ? (g == 0 ? Nz - 2 : 4 * g - 2) : 4 * g;
  const int zB = SHIFT ? 4 * g : 4 * g + 2;
  const int npt = SHIFT ? 4 : min(4, Nz - 4 * g);
  float dx[4], dy[4], dz[4];
  if (SHIFT) {
    const float2 ax = *reinterpret_cast<const float2*>(disp + rowp0 + zA);
    const float2 bx = *reinterpret_cast<const float2*>(disp + rowp0 + zB);
    const float2 ay = *reinterpret_cast<const float2*>(disp + N + rowp0 + zA);
    const float2 by = *reinterpret_cast<const float2*>(disp + N + rowp0 + zB);
    const float2 az = *reinterpret_cast<const float2*>(disp + 2 * N + rowp0 + zA);
    const float2 bz = *reinterpret_cast<const float2*>(disp + 2 * N + rowp0 + zB);
    dx[0] = ax.x; dx[1] = ax.y; dx[2] = bx.x; dx[3] = bx.y;
    dy[0] = ay.x; dy[1] = ay.y; dy[2] = by.x; dy[3] = by.y;
    dz[0] = az.x; dz[1] = az.y; dz[2] = bz.x; dz[3] = bz.y;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      dx[m] *= sc.x;
      dy[m] *= sc.y;
      dz[m] *= sc.z;
    }
  } else if (vec) {
    const long long p0 = rowp0 + 4 * g;
    const float4 a = *reinterpret_cast<const float4*>(disp + p0);
    const float4 b = *reinterpret_cast<const float4*>(disp + N + p0);
    const float4 cc = *reinterpret_cast<const float4*>(disp + 2 * N + p0);
    dx[0] = a.x; dx[1] = a.y; dx[2] = a.z; dx[3] = a.w;
    dy[0] = b.x; dy[1] = b.y; dy[2] = b.z; dy[3] = b.w;
    dz[0] = cc.x; dz[1] = cc.y; dz[2] = cc.z; dz[3] = cc.w;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      dx[m] *= sc.x;
      dy[m] *= sc.y;
      dz[m] *= sc.z;
    }
  } else {
    const long long p0 = rowp0 + 4 * g;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const bool in = m < npt;
      dx[m] = in ? sc.x * __ldg(disp + p0 + m) : 0.f;
      dy[m] = in ? sc.y * __ldg(disp + N + p0 + m) : 0.f;
      dz[m] = in ? sc.z * __ldg(disp + 2 * N + p0 + m) : 0.f;
    }
  }
  float fx[4], fy[4], fz[4];
  bool ok = true;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    fx[m] = floorf(dx[m]);
    fy[m] = floorf(dy[m]);
    fz[m] = floorf(dz[m]);
    ok = ok && fx[m] >= -1.f && fx[m] <= 0.f && fy[m] >= -1.f && fy[m] <= 0.f && fz[m] >= -1.f && fz[m] <= 0.f;
  }
  if (!ok) {
    for (int m = 0; m < npt; ++m) {
      const int zm = (m < 2 ? zA : zB) + (m & 1);
      float v[NC];
      gather_point_global<NC>(coef + c0 * N, disp, i, j, zm, Nx, Ny, Nz, NC, v, sc);
      for (int c = 0; c < NC; ++c) out[(c0 + c) * N + rowp0 + zm] = v[c];
    }
    return;
  }
  // weights of node pairs (0,1) and (2,3) packed as float2 for the sm_100 packed
  // FFMA2 pipe: each __ffma2_rn is two independent, correctly rounded fmaf.
  float2 wx[2][5], wy[2][5], wz[2][5];
#pragma unroll
  for (int hp = 0; hp < 2; ++hp) {
    float t0[5], t1[5];
    w5(dx[2 * hp], fx[2 * hp], t0);
    w5(dx[2 * hp + 1], fx[2 * hp + 1], t1);
#pragma unroll
    for (int k = 0; k < 5; ++k) wx[hp][k] = make_float2(t0[k], t1[k]);
    w5(dy[2 * hp], fy[2 * hp], t0);
    w5(dy[2 * hp + 1], fy[2 * hp + 1], t1);
#pragma unroll
    for (int k = 0; k < 5; ++k) wy[hp][k] = make_float2(t0[k], t1[k]);
    w5(dz[2 * hp], fz[2 * hp], t0);
    w5(dz[2 * hp + 1], fz[2 * hp + 1], t1);
#pragma unroll
    for (int k = 0; k < 5; ++k) wz[hp][k] = make_float2(t0[k], t1[k]);
  }
  float2 acc[NC][2];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c][0] = acc[c][1] = make_float2(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < 5; ++a) {
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      const float* rowp = pl[a] + b * P;
      const float2 w01a = __fmul2_rn(wx[0][a], wy[0][b]);
      const float2 w01b = __fmul2_rn(wx[1][a], wy[1][b]);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const float4 A = *reinterpret_cast<const float4*>(rowp + c * CVOL);
        const float4 B = *reinterpret_cast<const float4*>(rowp + c * CVOL + 4);
        const float win[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
        // nodes (0,1): taps win[k], win[k+1]; nodes (2,3): win[k+2], win[k+3]
        float2 pa = __fmul2_rn(wz[0][0], make_float2(win[0], win[1]));
        float2 pb = __fmul2_rn(wz[1][0], make_float2(win[2], win[3]));
#pragma unroll
        for (int k = 1; k < 5; ++k) {
          if (k & 1) {
            pa.x = fmaf(wz[0][k].x, win[k], pa.x);
            pa.y = fmaf(wz[0][k].y, win[k + 1], pa.y);
            pb.x = fmaf(wz[1][k].x, win[k + 2], pb.x);
            pb.y = fmaf(wz[1][k].y, win[k + 3], pb.y);
          } else {
            pa = __ffma2_rn(wz[0][k], make_float2(win[k], win[k + 1]), pa);
            pb = __ffma2_rn(wz[1][k], make_float2(win[k + 2], win[k + 3]), pb);
          }
        }
        acc[c][0] = __ffma2_rn(w01a, pa, acc[c][0]);
        acc[c][1] = __ffma2_rn(w01b, pb, acc[c][1]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float* o = out + (c0 + c) * N + rowp0;
    if (SHIFT) {
      *reinterpret_cast<float2*>(o + zA) = acc[c][0];
      *reinterpret_cast<float2*>(o + zB) = acc[c][1];
    } else if (vec) {
      *reinterpret_cast<float4*>(o + 4 * g) = make_float4(acc[c][0].x, acc[c][0].y, acc[c][1].x, acc[c][1].y);
    } else {
      const float v4[4] = {acc[c][0].x, acc[c][0].y, acc[c][1].x, acc[c][1].y};
      for (int m = 0; m < npt; ++m) o[4 * g + m] = v4[m];
    }
  }
}

template <int NC, int TX, int TY, int NTH, int P, bool SHIFT>
__device__ __forceinline__ void gw_compute(const float* sbuf, const float* __restrict__ coef,
                                           const float* __restrict__ disp, float* __restrict__ out, long long N,
                                           int c0, int x0, int y0, int Nx, int Ny, int Nz, float3 sc) {
  constexpr int SY = TY + 2 * GW_H, SX = TX + 2 * GW_H;
  constexpr int cvol = SX * SY * P;
  const int G = (Nz + 3) >> 2;
  const int items = TX * TY * G;
  for (int it = threadIdx.x; it < items; it += NTH) {
    const int r = it / G, g = it - r * G;
    const int rx = r / TY, ry = r - (r / TY) * TY;
    const int i = x0 + rx, j = y0 + ry;
    if (i >= Nx || j >= Ny) continue;
    const float* base = sbuf + (rx * SY + ry) * P + 4 * g;
    const float* const pl[5] = {base, base + SY * P, base + 2 * SY * P, base + 3 * SY * P, base + 4 * SY * P};
    gw_item<NC, P, cvol, SHIFT>(pl, coef, disp, out, N, c0, i, j, g, Nx, Ny, Nz, sc);
  }
}

// Components in groups of FG (single-buffered: stage, compute, repeat); the tail
// group dispatches to the matching NC instantiation outside the row loop.
template <int FG, int TX, int TY, int NTH, int P, bool SHIFT>
__global__ __launch_bounds__(NTH, 1) void gather_win_kernel(const float* __restrict__ coef, int F,
                                                            const float* __restrict__ disp, float* __restrict__ out,
                                                            int Nx, int Ny, int Nz, float3 sc) {
  pdl_prologue();
  extern __shared__ __align__(16) float smw[];
  const long long N = (long long)Nx * Ny * Nz;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  for (int c0 = 0; c0 < F; c0 += FG) {
    const int nc = min(FG, F - c0);
    __syncthreads();
    gw_stage<TX, TY, NTH, SHIFT>(smw, coef, N, c0, nc, x0, y0, Nx, Ny, Nz, P);
    cp_async_commit();
    cp_async_wait_group<0>();
    __syncthreads();
    if (FG >= 3 && nc == 3)
      gw_compute<3, TX, TY, NTH, P, SHIFT>(smw, coef, disp, out, N, c0, x0, y0, Nx, Ny, Nz, sc);
    else if (FG >= 2 && nc == 2)
      gw_compute<2, TX, TY, NTH, P, SHIFT>(smw, coef, disp, out, N, c0, x0, y0, Nx, Ny, Nz, sc);
    else
      gw_compute<1, TX, TY, NTH, P, SHIFT>(smw, coef, disp, out, N, c0, x0, y0, Nx, Ny, Nz, sc);
  }
}

constexpr int GW_TX = 8, GW_TY = 4, GW_NTH = 512;
constexpr size_t GW_SMEM_MAX = 227 * 1024;

// ---------------------------------------------------------------------------
// Marching window gather.  A CTA owns TY output y rows and a segment of x rows and
// walks x: shared memory holds a ring of GM_RING staged x planes, each the
// (TY+4) periodic y rows x (P-pitched z row) of FG components.  Output row x needs
// planes x-2 .. x+2; while it is computed, plane x+3 streams in (cp.async) into the
// slot plane x-3 vacated, so staging overlaps the FMAs instead of alternating with
// them, and every source plane is staged once per (y tile, x segment) rather than
// once per 8 x 4 tile (halo amplification (TY+4)/TY instead of 3).  The per-group
// arithmetic is gw_item, bitwise the same as the tiled kernel.
constexpr int GM_RING = 6;
constexpr int GM_NTH = 512;

template <int FG, int P>
constexpr int gm_tymax() {
  constexpr int t = (int)(GW_SMEM_MAX / sizeof(float) / (GM_RING * FG * P)) - 2 * GW_H;
  return t > 16 ? 16 : t;
}

template <int NTH, bool SHIFT>
__device__ __forceinline__ void gm_stage_plane(float* dst_slot, int cvol, const float* __restrict__ coef, long long N,
                                               int c0, int nc, int x, int y0, int TY, int Nx, int Ny, int Nz,
                                               int P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int SYr = TY + 2 * GW_H;
  const int zlen = SHIFT ? Nz + 8 : ((Nz + 3) & ~3) + 2 * GW_H;
  const long long xoff = (long long)wrapi(x, Nx) * Ny;
  for (int row = warp; row < nc * SYr; row += NTH / 32) {
    const int c = row / SYr, jy = row - c * SYr;
    const float* src = coef + (c0 + c) * N + (xoff + wrapi(y0 - GW_H + jy, Ny)) * Nz;
    float* dst = dst_slot + c * cvol + jy * P;
    if (SHIFT) {
      for (int zz = 4 * lane; zz < zlen; zz += 128) {
        int gz = zz - 4;
        gz += gz < 0 ? Nz : 0;
        gz -= gz >= Nz ? Nz : 0;
        cp_async16_cg(dst + zz, src + gz);
      }
    } else {
      for (int zz = 2 * lane; zz < zlen; zz += 64) {
        int gz = zz - GW_H;
        gz += gz < 0 ? Nz : 0;
        gz -= gz >= Nz ? Nz : 0;
        cp_async8(dst + zz, src + gz);
      }
    }
  }
}

template <int NC, int NTH, int P, int CVOL, int SLOT, bool SHIFT>
__device__ __forceinline__ void gm_row(const float* smw, int xr, const float* __restrict__ coef,
                                       const float* __restrict__ disp, float* __restrict__ out, long long N, int c0,
                                       int i, int y0, int TY, int Nx, int Ny, int Nz, float3 sc) {
  const int G = (Nz + 3) >> 2;
  const int items = TY * G;
  int sl[5];
#pragma unroll
  for (int a = 0; a < 5; ++a) sl[a] = ((xr + a) % GM_RING) * SLOT;
  for (int it = threadIdx.x; it < items; it += NTH) {
    const int ry = it / G, g = it - ry * G;
    const int j = y0 + ry;
    if (j >= Ny) continue;
    const float* base = smw + ry * P + 4 * g;
    const float* const pl[5] = {base + sl[0], base + sl[1], base + sl[2], base + sl[3], base + sl[4]};
    gw_item<NC, P, CVOL, SHIFT>(pl, coef, disp, out, N, c0, i, j, g, Nx, Ny, Nz, sc);
  }
}

template <int FG, int NTH, int P, bool SHIFT>
__global__ __launch_bounds__(NTH, 1) void gather_march_kernel(const float* __restrict__ coef, int F,
                                                              const float* __restrict__ disp, float* __restrict__ out,
                                                              int Nx, int Ny, int Nz, float3 sc, int TY, int seg) {
  pdl_prologue();
  constexpr int TYM = gm_tymax<FG, P>();
  constexpr int CVOL = (TYM + 2 * GW_H) * P;
  constexpr int SLOT = FG * CVOL;
  extern __shared__ __align__(16) float smw[];
  const long long N = (long long)Nx * Ny * Nz;
  const int x0 = blockIdx.x * seg, nx = min(seg, Nx - x0);
  const int y0 = blockIdx.y * TY;
  if (nx <= 0) return;
  for (int c0 = 0; c0 < F; c0 += FG) {
    const int nc = min(FG, F - c0);
    __syncthreads();
    // prologue: planes x0-2 .. x0+2 in slots 0..4
    for (int q = 0; q < 5; ++q)
      gm_stage_plane<NTH, SHIFT>(smw + q * SLOT, CVOL, coef, N, c0, nc, x0 - GW_H + q, y0, TY, Nx, Ny, Nz, P);
    cp_async_commit();
    cp_async_wait_group<0>();
    __syncthreads();
    for (int xr = 0; xr < nx; ++xr) {
      // plane x0+xr+3 (needed by row xr+1) into the slot of plane x0+xr-3 (last read by row xr-1)
      if (xr + 1 < nx)
        gm_stage_plane<NTH, SHIFT>(smw + ((xr + 5) % GM_RING) * SLOT, CVOL, coef, N, c0, nc, x0 + xr + 3, y0, TY,
                                   Nx, Ny, Nz, P);
      cp_async_commit();
      if (FG >= 3 && nc == 3)
        gm_row<3, NTH, P, CVOL, SLOT, SHIFT>(smw, xr, coef, disp, out, N, c0, x0 + xr, y0, TY, Nx, Ny, Nz, sc);
      else if (FG >= 2 && nc == 2)
        gm_row<2, NTH, P, CVOL, SLOT, SHIFT>(smw, xr, coef, disp, out, N, c0, x0 + xr, y0, TY, Nx, Ny, Nz, sc);
      else
        gm_row<1, NTH, P, CVOL, SLOT, SHIFT>(smw, xr, coef, disp, out, N, c0, x0 + xr, y0, TY, Nx, Ny, Nz, sc);
      cp_async_wait_group<0>();
      __syncthreads();
    }
  }
}

static bool use_pipe() {
  static const bool on = [] {
    const char* e = std::getenv("LDDMM_GATHER_PIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool use_march() {
  static const bool on = [] {
    const char* e = std::getenv("LDDMM_GATHER_MARCH");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int P, bool SHIFT>
static bool launch_gm_pitch(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                            cudaStream_t s) {
  const int need = SHIFT ? N[2] + 8 : ((N[2] + 3) & ~3) + 2 * GW_H;
  if (need > P) return false;
  const int G = (N[2] + 3) / 4;
  if (G > GM_NTH) return false;
  const int FG = std::min(3, ncomp);
  const int tym = FG == 3 ? gm_tymax<3, P>() : FG == 2 ? gm_tymax<2, P>() : gm_tymax<1, P>();
  if (tym < 1) return false;
  const int TY = std::max(1, std::min(tym, GM_NTH / G));
  const int tiles_y = ceil_div(N[1], TY);
  int nseg = std::max(1, kSMs / tiles_y);
  const int seg = ceil_div(N[0], nseg);
  nseg = ceil_div(N[0], seg);
  const size_t smem = (size_t)GM_RING * FG * (tym + 2 * GW_H) * P * sizeof(float);
  static bool attr_set[64][3] = {};
  int dev = 0;
  LDDMM_CUDA(cudaGetDevice(&dev));
  dim3 grid(nseg, tiles_y, 1);
  auto go = [&](auto kern, int k) {
    if (!attr_set[dev & 63][k]) {
      LDDMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GW_SMEM_MAX));
      attr_set[dev & 63][k] = true;
    }
    pdl_launch(kern, grid, GM_NTH, smem, s, coef, ncomp, disp, out, N[0], N[1], N[2], sc, TY, seg);
  };
  if (FG == 3)
    go(gather_march_kernel<3, GM_NTH, P, SHIFT>, 2);
  else if (FG == 2)
    go(gather_march_kernel<2, GM_NTH, P, SHIFT>, 1);
  else
    go(gather_march_kernel<1, GM_NTH, P, SHIFT>, 0);
  LDDMM_LAUNCH_CHECK();
  return true;
}

template <bool SHIFT>
static bool launch_gm_any(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                          cudaStream_t s) {
  return launch_gm_pitch<64, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gm_pitch<128, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gm_pitch<192, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gm_pitch<264, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gm_pitch<392, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gm_pitch<520, SHIFT>(coef, ncomp, disp, out, N, sc, s);
}


template <int P, bool SHIFT>
static bool launch_gw_pitch(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                            cudaStream_t s) {
  const int need = SHIFT ? N[2] + 8 : ((N[2] + 3) & ~3) + 2 * GW_H;
  if (need > P) return false;
  const size_t per_comp = (size_t)(GW_TX + 4) * (GW_TY + 4) * P * sizeof(float);
  const int fg = (int)std::min<size_t>(3, GW_SMEM_MAX / per_comp);
  if (fg < 1) return false;
  static bool attr_set[64][3] = {};
  int dev = 0;
  LDDMM_CUDA(cudaGetDevice(&dev));
  dim3 grid(ceil_div(N[0], GW_TX), ceil_div(N[1], GW_TY), 1);
  const int FG = std::min(fg, ncomp);
  const size_t smem = (size_t)FG * per_comp;
  auto go = [&](auto kern, int k) {
    if (!attr_set[dev & 63][k]) {
      LDDMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GW_SMEM_MAX));
      attr_set[dev & 63][k] = true;
    }
    pdl_launch(kern, grid, GW_NTH, smem, s, coef, ncomp, disp, out, N[0], N[1], N[2], sc);
  };
  if (FG == 3)
    go(gather_win_kernel<3, GW_TX, GW_TY, GW_NTH, P, SHIFT>, 2);
  else if (FG == 2)
    go(gather_win_kernel<2, GW_TX, GW_TY, GW_NTH, P, SHIFT>, 1);
  else
    go(gather_win_kernel<1, GW_TX, GW_TY, GW_NTH, P, SHIFT>, 0);
  LDDMM_LAUNCH_CHECK();
  return true;
}

template <bool SHIFT>
static bool launch_gw_any(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                          cudaStream_t s) {
  return launch_gw_pitch<64, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gw_pitch<128, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gw_pitch<192, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gw_pitch<264, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gw_pitch<392, SHIFT>(coef, ncomp, disp, out, N, sc, s) ||
         launch_gw_pitch<520, SHIFT>(coef, ncomp, disp, out, N, sc, s);
}

void launch_gather_cubic(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                         cudaStream_t s) {
  launch_gather_scaled(coef, ncomp, disp, 1.f, 1.f, 1.f, out, N, s);
}

// Row pitch: the smallest compiled pitch holding the staged row (Nz + 8 with the
// shifted groups when Nz % 4 == 0, else Nz + 4 rounded to 4); longer z rows go to
// the tiled kernel (unit scale only).  `march`: the SL-step gathers (sub-voxel
// departures) take the marching kernel; pull-backs through whole deformation maps
// (many nodes outside the window regime, served by the global-memory path) keep the
// tiled kernel, whose 16 waves of small CTAs balance those slow nodes.
void launch_gather_scaled(const float* coef, int ncomp, const float* disp, float sx, float sy, float sz, float* out,
                          const int* N, cudaStream_t s, bool march) {
  const float3 sc = make_float3(sx, sy, sz);
  if (march && use_pipe() && launch_gather_pipe(coef, ncomp, disp, out, N, sc, s)) return;
  if (march && use_march() && (N[2] % 4 == 0 ? launch_gm_any<true>(coef, ncomp, disp, out, N, sc, s)
                                    : launch_gm_any<false>(coef, ncomp, disp, out, N, sc, s)))
    return;
  if (N[2] % 4 == 0 ? launch_gw_any<true>(coef, ncomp, disp, out, N, sc, s)
                    : launch_gw_any<false>(coef, ncomp, disp, out, N, sc, s))
    return;
  shape_require(sx == 1.f && sy == 1.f && sz == 1.f, "gather: z rows longer than 516 need unit scale");
  launch_gather_cubic_tiled(coef, ncomp, disp, out, N, s);
}

void launch_gather_cubic_tiled(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                               cudaStream_t s) {
  {
    const int FG = ncomp >= 3 ? 3 : ncomp;
    dim3 grid(ceil_div(N[0], GT_X), ceil_div(N[1], GT_Y), ceil_div(N[2], GT_Z));
    const size_t smem = (size_t)FG * GS_VOL * sizeof(float);
    static bool attr_set[64] = {false};
    int dev = 0;
    LDDMM_CUDA(cudaGetDevice(&dev));
    if (!attr_set[dev & 63]) {
      LDDMM_CUDA(cudaFuncSetAttribute(gather_tiled_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      3 * GS_VOL * (int)sizeof(float)));
      LDDMM_CUDA(cudaFuncSetAttribute(gather_tiled_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      2 * GS_VOL * (int)sizeof(float)));
      LDDMM_CUDA(cudaFuncSetAttribute(gather_tiled_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      1 * GS_VOL * (int)sizeof(float)));
      attr_set[dev & 63] = true;
    }
    if (FG == 3)
      pdl_launch(gather_tiled_kernel<3>, grid, GT_THREADS, smem, s, coef, ncomp, disp, out, N[0], N[1], N[2], make_float3(1.f, 1.f, 1.f));
    else if (FG == 2)
      pdl_launch(gather_tiled_kernel<2>, grid, GT_THREADS, smem, s, coef, ncomp, disp, out, N[0], N[1], N[2], make_float3(1.f, 1.f, 1.f));
    else
      pdl_launch(gather_tiled_kernel<1>, grid, GT_THREADS, smem, s, coef, ncomp, disp, out, N[0], N[1], N[2], make_float3(1.f, 1.f, 1.f));
    LDDMM_LAUNCH_CHECK();
    return;
  }
}

static void launch_gather_global_scaled(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                                       float3 sc, cudaStream_t s) {
  const long long n = (long long)N[0] * N[1] * N[2];
  const int grid = grid_for(n, 256, 16);
  int done = 0;
  while (done < ncomp) {
    const int left = ncomp - done;
    const float* c = coef + (long long)done * n;
    float* o = out + (long long)done * n;
    if (left >= 6) {
      pdl_launch(gather_cubic_kernel<6>, grid, 256, 0, s, c, disp, o, N[0], N[1], N[2], sc);
      done += 6;
    } else if (left >= 4) {
      pdl_launch(gather_cubic_kernel<4>, grid, 256, 0, s, c, disp, o, N[0], N[1], N[2], sc);
      done += 4;
    } else if (left >= 3) {
      pdl_launch(gather_cubic_kernel<3>, grid, 256, 0, s, c, disp, o, N[0], N[1], N[2], sc);
      done += 3;
    } else {
      pdl_launch(gather_cubic_kernel<1>, grid, 256, 0, s, c, disp, o, N[0], N[1], N[2], sc);
      done += 1;
    }
    LDDMM_LAUNCH_CHECK();
  }
}

void launch_gather_cubic_global(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                                cudaStream_t s) {
  launch_gather_global_scaled(coef, ncomp, disp, out, N, make_float3(1.f, 1.f, 1.f), s);
}

// ---------------------------------------------------------------------------
// departure points (transport.hpp:83-102), both directions at once; stationary
// velocity: v_grid and v_traced are the same node.

__global__ __launch_bounds__(256) void departure_kernel(const float* __restrict__ vg, const float* __restrict__ vc,
                                                        float dtx, float dty, float dtz, float* __restrict__ df,
                                                        float* __restrict__ db, int Nx, int Ny, int Nz) {
  pdl_prologue();
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

// D = sg * dt/2 * (v_traced(X*) + v_grid) in grid units, vm = v_traced(X*) gathered
__global__ void departure_combine_kernel(long long n, const float* __restrict__ vg, const float* __restrict__ vm,
                                         float dtx, float dty, float dtz, float sg, float* __restrict__ o) {
  pdl_prologue();
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const float ux = vg[p] * dtx, uy = vg[n + p] * dty, uz = vg[2 * n + p] * dtz;
    o[p] = sg * 0.5f * (vm[p] * dtx + ux);
    o[n + p] = sg * 0.5f * (vm[n + p] * dty + uy);
    o[2 * n + p] = sg * 0.5f * (vm[2 * n + p] * dtz + uz);
  }
}

// sl_departure (transport.hpp:83-102) for a stationary velocity: X* = x + sg dt v(x),
// v_traced(X*) through the production gather (displacement scale sg dt / h), then the
// trapezoid combination; scratch holds [3][N] floats per direction.
void launch_departure_dir(const float* vgrid, const float* vcoef, double dt, const double* h, float sg, float* out,
                          float* vm, const int* N, cudaStream_t s) {
  const long long n = (long long)N[0] * N[1] * N[2];
  const float dtx = (float)(dt / h[0]), dty = (float)(dt / h[1]), dtz = (float)(dt / h[2]);
  launch_gather_scaled(vcoef, 3, vgrid, sg * dtx, sg * dty, sg * dtz, vm, N, s);
  pdl_launch(departure_combine_kernel, grid_for(n, 256), 256, 0, s, n, vgrid, vm, dtx, dty, dtz, sg, out);
  LDDMM_LAUNCH_CHECK();
}

void launch_departure(const float* vgrid, const float* vcoef, double dt, const double* h, float* dep_fwd,
                      float* dep_bwd, float* scratch, const int* N, cudaStream_t s) {
  launch_departure_dir(vgrid, vcoef, dt, h, -1.f, dep_fwd, scratch, N, s);
  if (dep_bwd) launch_departure_dir(vgrid, vcoef, dt, h, 1.f, dep_bwd, scratch, N, s);
}

// pull-back through points x - disp (disp physical): the production gather with
// displacement scale -1/h (m1 = I0 o phi1, grad_src_warped, warp of grid fields).
// `large`: the caller expects multi-voxel displacements (a whole deformation map, e.g.
// u(1) with max |v| T / h > 1): most nodes leave the window regime, and the plain
// per-node gather (L1 / L2 taps, weights shared by the components) beats the staged
// window kernel with its per-node fallback (2.3x at 1.5 voxels, 3.6x at 4,
// tools/lab/gather_lab.py); both are bitwise the same samples.
void launch_warp_by_displacement(const float* coef, int ncomp, const float* disp_phys, const double* h,
                                 float* out, const int* N, cudaStream_t s, bool large) {
  const float3 sc = make_float3(-(float)(1.0 / h[0]), -(float)(1.0 / h[1]), -(float)(1.0 / h[2]));
  if (large) {
    launch_gather_global_scaled(coef, ncomp, disp_phys, out, N, sc, s);
    return;
  }
  launch_gather_scaled(coef, ncomp, disp_phys, sc.x, sc.y, sc.z, out, N, s, false);
}

// ---------------------------------------------------------------------------
// warp_nearest (interp.hpp:213-225): the point x - d is divided by h and rounded
// half away from zero (std::llround), then wrapped periodically; label values are
// copied, never mixed.
__global__ void warp_nearest_kernel(const float* __restrict__ f, int ncomp, const float* __restrict__ disp,
                                    double hx, double hy, double hz, float* __restrict__ out, int Nx, int Ny,
                                    int Nz) {
  pdl_prologue();
  const long long N = (long long)Nx * Ny * Nz;
  GRID_STRIDE(p, N) {
    const int k = (int)(p % Nz);
    const long long q = p / Nz;
    const int j = (int)(q % Ny), i = (int)(q / Ny);
    const double ux = ((double)i * hx - (double)disp[p]) / hx;
    const double uy = ((double)j * hy - (double)disp[N + p]) / hy;
    const double uz = ((double)k * hz - (double)disp[2 * N + p]) / hz;
    long long ix = llround(ux) % Nx, iy = llround(uy) % Ny, iz = llround(uz) % Nz;
    ix += ix < 0 ? Nx : 0;
    iy += iy < 0 ? Ny : 0;
    iz += iz < 0 ? Nz : 0;
    const long long src = (ix * Ny + iy) * Nz + iz;
    for (int c = 0; c < ncomp; ++c) out[c * N + p] = f[c * N + src];
  }
}

void launch_warp_nearest(const float* f, int ncomp, const float* disp_phys, const double* h, float* out,
                         const int* N, cudaStream_t s) {
  const long long n = (long long)N[0] * N[1] * N[2];
  pdl_launch(warp_nearest_kernel, grid_for(n, 256), 256, 0, s, f, ncomp, disp_phys, h[0], h[1], h[2], out, N[0], N[1],
                                                       N[2]);
  LDDMM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// exact periodic cubic B-spline prefilter along one axis (interp.hpp:23-63),
// one thread per line, in place (the causal pass overwrites the line with c+,
// the anticausal pass overwrites c+ with 6 c-).

template <typename T>
__global__ void prefilter_axis_kernel(T* __restrict__ v, int n, long long stride, long long lines,
                                      long long outer_stride) {
  pdl_prologue();
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
    pdl_launch(prefilter_axis_kernel<T>, grid_for(lines, 128, 32), 128, 0, s, f, n, stride, lines, stride * n);
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
  pdl_prologue();
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

// Register-blocked circulant: each thread produces CR consecutive outputs i0 ..
// i0+CR-1 of its line, so every loaded input feeds CR accumulators, and the circulant
// taps are read through a sliding window (CR + 7 shared-memory loads per 8 inputs).
// Each accumulator still sums j = 0 .. n-1 in order with fma: bitwise the same as
// circulant_axis_kernel (kept for lines shorter than 8).
constexpr int CR = 8;
__global__ void circulant_axis_blocked_kernel(const double* __restrict__ in, double* __restrict__ out,
                                              const double* __restrict__ D, int n, long long stride,
                                              long long work) {
  pdl_prologue();
  extern __shared__ double sD[];
  for (int t = threadIdx.x; t < n; t += blockDim.x) sD[t] = D[t];
  __syncthreads();
  const int nb = (n + CR - 1) / CR;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < work;
       q += (long long)gridDim.x * blockDim.x) {
    const long long inner = q % stride;
    const long long t = q / stride;
    const int ib = (int)(t % nb);
    const long long oh = t / nb;
    const int i0 = ib * CR;
    const long long base = oh * n * stride + inner;
    double acc[CR];
#pragma unroll
    for (int r = 0; r < CR; ++r) acc[r] = 0.0;
    auto dmod = [n](int d) {
      d %= n;
      return d < 0 ? d + n : d;
    };
    int j0 = 0;
    for (; j0 + 8 <= n; j0 += 8) {
      // window m = 0 .. CR+6 holds D[(i0 - j0 - 7 + m) mod n]; tap (r, jj) is m = r - jj + 7
      double w[CR + 7];
      int d = dmod(i0 - j0 - 7);
#pragma unroll
      for (int m = 0; m < CR + 7; ++m) {
        w[m] = sD[d];
        d = d + 1 == n ? 0 : d + 1;
      }
      double x[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) x[jj] = in[base + (long long)(j0 + jj) * stride];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
#pragma unroll
        for (int r = 0; r < CR; ++r) acc[r] = fma(w[r - jj + 7], x[jj], acc[r]);
    }
    for (; j0 < n; ++j0) {
      const double x = in[base + (long long)j0 * stride];
      int d = dmod(i0 - j0);
#pragma unroll
      for (int r = 0; r < CR; ++r) {
        acc[r] = fma(sD[d], x, acc[r]);
        d = d + 1 == n ? 0 : d + 1;
      }
    }
#pragma unroll
    for (int r = 0; r < CR; ++r)
      if (i0 + r < n) out[base + (long long)(i0 + r) * stride] = acc[r];
  }
}

void launch_circulant_axis_f64(const double* in, double* out, const double* D, int axis, const int* N,
                               cudaStream_t s) {
  long long stride = 1;
  for (int b = axis + 1; b < 3; ++b) stride *= N[b];
  const long long total = (long long)N[0] * N[1] * N[2];
  if (N[axis] >= 8) {
    const long long work = total / N[axis] * ((N[axis] + CR - 1) / CR);
    pdl_launch(circulant_axis_blocked_kernel, grid_for(work, 256, 8), 256, N[axis] * sizeof(double), s, in, out, D, N[axis],
                                                                                               stride, work);
    LDDMM_LAUNCH_CHECK();
    return;
  }
  pdl_launch(circulant_axis_kernel, grid_for(total, 256, 16), 256, N[axis] * sizeof(double), s, in, out, D, N[axis],
                                                                                        stride, total);
  LDDMM_LAUNCH_CHECK();
}

void launch_prefilter3d(double* f, const int* N, cudaStream_t s) { prefilter3d<double>(f, N, s); }
void launch_prefilter3d_f32(float* f, const int* N, cudaStream_t s) { prefilter3d<float>(f, N, s); }

}  // namespace lddmm_b200
