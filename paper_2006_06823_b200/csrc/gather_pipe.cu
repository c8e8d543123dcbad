// Pipelined marching SL gather (sm_100a): the production kernel for the SL-step
// cubic gathers (ScalarSampler::eval_cubic / accumulate<4> at the departure points,
// interp.hpp:119-159, inside advect_state, transport.hpp:67-73).
//
// Layout of the work.  A CTA owns TY output y rows and a segment of x rows
// and walks x.  Shared memory is a ring of GP_RING staged x planes; a plane holds, for
// each of the FG components of the pass, the TY+4 periodic y rows x..x (halo 2) as
// dense rows of P >= Nz floats (P a multiple of 32, so every row starts on a 128-byte
// boundary).  Output row x reads planes x-2 .. x+2.
//
// Roles.  Every warp computes.  Planes stream into the ring with TMA tensor copies
// (cp.async.bulk.tensor, completion counted on a per-slot `full` mbarrier; the z tail
// P - Nz of each row is zero-filled by the TMA unit and never read).  Warps take the
// (row, item) sequence of the segment in order, wait on `full` for the planes an item
// needs and release a plane once they are past it; the warp whose release completes a
// slot's count (a shared-memory atomic) issues the refill with the plane RING ahead.
// No CTA-wide barrier and no dedicated producer warp are on the path, so warps drift
// across x rows instead of stepping in lockstep, and every warp slot computes.
//
// Item (GP_ROWS = 1, production) = one output row x one 4-node z group: 5 x 5 source
// rows, each one aligned 8-float window (two LDS.128) serving the 5-tap z stencils of
// the four nodes (SHIFT layout: group g = nodes 4g-2 .. 4g+1, window z = 4g-4 .. 4g+3;
// the first chunk of group 0 wraps to Nz-4 .. Nz-1 of the same row, so the rows need
// no staged halo).  Per node the arithmetic is gw_item's (interp.cu): x-outer /
// y-inner, w01 = wx * wy, z taps in order, the zero-weight tap first or last —
// bitwise the marching / window kernels (tests/test_gpu_ops.py) and the reference's
// accumulation order (interp.hpp:145-156).  Nodes outside the sub-voxel regime
// (|floor(d)| > 1) take the global-memory path (same arithmetic).
//
// GP_ROWS = 2 (y-pair items: rows j, j+1 share the 5 x 6 source rows, 0.6x the
// shared-memory wavefronts) is kept as a measured alternative: it needs ~250
// registers, so only 2 warps per SM sub-partition fit, and on B200 it is 12% slower
// than the one-row item (tools/lab/gather_lab.py).
//
// Requirements (else the caller uses the older kernels): Nz % 4 == 0, Nz <= 256
// (TMA box extent), Ny even.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "gather_common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

namespace {

#ifndef GP_ROWS
#define GP_ROWS 1  // output y rows per item (1: 4-node items, 2: y-pair items; see the header)
#endif
#ifndef GP_SCALAR
#define GP_SCALAR 0
#endif
#ifndef GP_PREFETCH
#define GP_PREFETCH 1
#endif
#ifndef GP_RING_N
#define GP_RING_N 6
#endif
constexpr int GP_RING = GP_RING_N;  // staged planes (lab: -DGP_RING_N=7 with TY = 10)
#ifndef GP_THREADS
#define GP_THREADS 384
#endif
constexpr int GP_NTH = GP_THREADS;         // 384: 12 warps (3 per SM sub-partition), <= 168 registers
constexpr int GP_CW = GP_NTH / 32;         // every warp computes; lane 0 of warp 0 also produces
constexpr size_t GP_SMEM_MAX = 226 * 1024;

__device__ __forceinline__ uint32_t gp_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void gp_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n GP_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra GP_WAIT;\n}\n" ::"r"(gp_su32(bar)),
      "r"(parity)
      : "memory");
}

// one row box (P floats of row (y, x') of the [F*Nx][Ny][Nz] view) or a box of R rows
__device__ __forceinline__ void gp_tma(const CUtensorMap* tm, float* dst, unsigned long long* bar, int z, int y,
                                       int xc) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
          "r"(gp_su32(dst)),
      "l"(tm), "r"(z), "r"(y), "r"(xc), "r"(gp_su32(bar))
      : "memory");
}

// Per-node displacement -> floors -> the regime check (|floor(d)| <= 1 on every axis)
struct NodeD {
  float dx[4], dy[4], dz[4];
};

__device__ __forceinline__ void gp_load_disp(const float* __restrict__ disp, long long N, long long rowp, int zA,
                                             int zB, NodeD& d) {
  const float2 ax = __ldg(reinterpret_cast<const float2*>(disp + rowp + zA));
  const float2 bx = __ldg(reinterpret_cast<const float2*>(disp + rowp + zB));
  const float2 ay = __ldg(reinterpret_cast<const float2*>(disp + N + rowp + zA));
  const float2 by = __ldg(reinterpret_cast<const float2*>(disp + N + rowp + zB));
  const float2 az = __ldg(reinterpret_cast<const float2*>(disp + 2 * N + rowp + zA));
  const float2 bz = __ldg(reinterpret_cast<const float2*>(disp + 2 * N + rowp + zB));
  d.dx[0] = ax.x; d.dx[1] = ax.y; d.dx[2] = bx.x; d.dx[3] = bx.y;
  d.dy[0] = ay.x; d.dy[1] = ay.y; d.dy[2] = by.x; d.dy[3] = by.y;
  d.dz[0] = az.x; d.dz[1] = az.y; d.dz[2] = bz.x; d.dz[3] = bz.y;
}

// displacement scale (grid units per stored unit), applied when the item starts so the
// prefetched loads are not consumed right after issue
__device__ __forceinline__ NodeD gp_scaled(const NodeD& r, float3 sc) {
  NodeD d;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    d.dx[m] = r.dx[m] * sc.x;
    d.dy[m] = r.dy[m] * sc.y;
    d.dz[m] = r.dz[m] * sc.z;
  }
  return d;
}

__device__ __forceinline__ bool gp_regime(const NodeD& d) {
  bool ok = true;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float fx = floorf(d.dx[m]), fy = floorf(d.dy[m]), fz = floorf(d.dz[m]);
    ok = ok && fx >= -1.f && fx <= 0.f && fy >= -1.f && fy <= 0.f && fz >= -1.f && fz <= 0.f;
  }
  return ok;
}

// packed (node 0,1) / (node 2,3) 5-tap weights of one axis
__device__ __forceinline__ void gp_w5pair(const float* dv, float2 (&w)[2][5]) {
#pragma unroll
  for (int hp = 0; hp < 2; ++hp) {
    float t0[5], t1[5];
    w5(dv[2 * hp], floorf(dv[2 * hp]), t0);
    w5(dv[2 * hp + 1], floorf(dv[2 * hp + 1]), t1);
#pragma unroll
    for (int k = 0; k < 5; ++k) w[hp][k] = make_float2(t0[k], t1[k]);
  }
}

// z-dots of one 8-float window for the four nodes (gw_item's exact instruction order)
__device__ __forceinline__ void gp_zdot(const float (&win)[8], const float2 (&wz)[2][5], float2& pa, float2& pb) {
#if GP_SCALAR
  // scalar FFMA chains: the same correctly rounded products and sums as the packed form
  // (each FFMA2 lane is one fmaf), but they keep the FMA pipe full where the packed /
  // scalar mix does not (tools/lab/zdot_mix.cu: 128 vs 100 FMA/clk/SM on B200)
  pa.x = wz[0][0].x * win[0];
  pa.y = wz[0][0].y * win[1];
  pb.x = wz[1][0].x * win[2];
  pb.y = wz[1][0].y * win[3];
#pragma unroll
  for (int k = 1; k < 5; ++k) {
    pa.x = fmaf(wz[0][k].x, win[k], pa.x);
    pa.y = fmaf(wz[0][k].y, win[k + 1], pa.y);
    pb.x = fmaf(wz[1][k].x, win[k + 2], pb.x);
    pb.y = fmaf(wz[1][k].y, win[k + 3], pb.y);
  }
  return;
#endif
  pa = __fmul2_rn(wz[0][0], make_float2(win[0], win[1]));
  pb = __fmul2_rn(wz[1][0], make_float2(win[2], win[3]));
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
}

// One item: rows (j, j+1) x group g of output row i.  pl[a] = staged plane x-2+a of
// component 0 at the pair's first source row (y = j-2); components CV floats apart,
// rows P apart; offA / offB = the two window chunks within a row.
template <int NC, int P>
__device__ __forceinline__ void gp_item(const NodeD& r0, const NodeD& r1, const float* const (&pl)[5], int CV,
                                        int offA, int offB,
                                        const float* __restrict__ coef, const float* __restrict__ disp,
                                        float* __restrict__ out, long long N, int c0, int i, int j, int g, int Nx,
                                        int Ny, int Nz, float3 sc) {
  const long long rowp0 = ((long long)i * Ny + j) * Nz, rowp1 = rowp0 + Nz;
  const int zA = g == 0 ? Nz - 2 : 4 * g - 2, zB = 4 * g;
  const NodeD d0 = gp_scaled(r0, sc), d1 = gp_scaled(r1, sc);
  if (!(gp_regime(d0) && gp_regime(d1))) {
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
      const long long rp = r ? rowp1 : rowp0;
#pragma unroll 1
      for (int m = 0; m < 4; ++m) {
        const int zm = (m < 2 ? zA : zB) + (m & 1);
        float v[NC];
        gather_point_global<NC>(coef + c0 * N, disp, i, j + r, zm, Nx, Ny, Nz, NC, v, sc);
        for (int c = 0; c < NC; ++c) out[(c0 + c) * N + rp + zm] = v[c];
      }
    }
    return;
  }
  float2 wx0[2][5], wy0[2][5], wz0[2][5], wx1[2][5], wy1[2][5], wz1[2][5];
  gp_w5pair(d0.dx, wx0);
  gp_w5pair(d0.dy, wy0);
  gp_w5pair(d0.dz, wz0);
  gp_w5pair(d1.dx, wx1);
  gp_w5pair(d1.dy, wy1);
  gp_w5pair(d1.dz, wz1);
  float2 acc0[NC][2], acc1[NC][2];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc0[c][0] = acc0[c][1] = acc1[c][0] = acc1[c][1] = make_float2(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < 5; ++a) {
#pragma unroll
    for (int yb = 0; yb < 6; ++yb) {
      const float* rowp = pl[a] + yb * P;
      float2 w0a, w0b, w1a, w1b;
      if (yb < 5) {
        w0a = __fmul2_rn(wx0[0][a], wy0[0][yb]);
        w0b = __fmul2_rn(wx0[1][a], wy0[1][yb]);
      }
      if (yb > 0) {
        w1a = __fmul2_rn(wx1[0][a], wy1[0][yb - 1]);
        w1b = __fmul2_rn(wx1[1][a], wy1[1][yb - 1]);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const float4 A = *reinterpret_cast<const float4*>(rowp + c * CV + offA);
        const float4 B = *reinterpret_cast<const float4*>(rowp + c * CV + offB);
        const float win[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
        float2 pa, pb;
        if (yb < 5) {
          gp_zdot(win, wz0, pa, pb);
          acc0[c][0] = __ffma2_rn(w0a, pa, acc0[c][0]);
          acc0[c][1] = __ffma2_rn(w0b, pb, acc0[c][1]);
        }
        if (yb > 0) {
          gp_zdot(win, wz1, pa, pb);
          acc1[c][0] = __ffma2_rn(w1a, pa, acc1[c][0]);
          acc1[c][1] = __ffma2_rn(w1b, pb, acc1[c][1]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float* o = out + (c0 + c) * N;
    *reinterpret_cast<float2*>(o + rowp0 + zA) = acc0[c][0];
    *reinterpret_cast<float2*>(o + rowp0 + zB) = acc0[c][1];
    *reinterpret_cast<float2*>(o + rowp1 + zA) = acc1[c][0];
    *reinterpret_cast<float2*>(o + rowp1 + zB) = acc1[c][1];
  }
}

// One-row item: row j x group g (5 x 5 source rows; gw_item's arithmetic).
template <int NC, int P, bool UNIT>
__device__ __forceinline__ void gp_item1(const NodeD& r0, const float* const (&pl)[5], int CV, int offA, int offB,
                                         const float* __restrict__ coef, const float* __restrict__ disp,
                                         float* __restrict__ out, long long N, int c0, int i, int j, int g, int Nx,
                                         int Ny, int Nz, float3 sc) {
  const long long rowp0 = ((long long)i * Ny + j) * Nz;
  const int zA = g == 0 ? Nz - 2 : 4 * g - 2, zB = 4 * g;
  const NodeD d0 = UNIT ? r0 : gp_scaled(r0, sc);  // unit scale (SL steps): x * 1 is exact
  if (!gp_regime(d0)) {
#pragma unroll 1
    for (int m = 0; m < 4; ++m) {
      const int zm = (m < 2 ? zA : zB) + (m & 1);
      float v[NC];
      gather_point_global<NC>(coef + c0 * N, disp, i, j, zm, Nx, Ny, Nz, NC, v, sc);
      for (int c = 0; c < NC; ++c) out[(c0 + c) * N + rowp0 + zm] = v[c];
    }
    return;
  }
  float2 wx0[2][5], wy0[2][5], wz0[2][5];
  gp_w5pair(d0.dx, wx0);
  gp_w5pair(d0.dy, wy0);
  gp_w5pair(d0.dz, wz0);
  float2 acc0[NC][2];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc0[c][0] = acc0[c][1] = make_float2(0.f, 0.f);
#pragma unroll
  for (int a = 0; a < 5; ++a) {
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      const float* rowp = pl[a] + b * P;
      const float2 w0a = __fmul2_rn(wx0[0][a], wy0[0][b]);
      const float2 w0b = __fmul2_rn(wx0[1][a], wy0[1][b]);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const float4 A = *reinterpret_cast<const float4*>(rowp + c * CV + offA);
        const float4 B = *reinterpret_cast<const float4*>(rowp + c * CV + offB);
        const float win[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
        float2 pa, pb;
        gp_zdot(win, wz0, pa, pb);
        acc0[c][0] = __ffma2_rn(w0a, pa, acc0[c][0]);
        acc0[c][1] = __ffma2_rn(w0b, pb, acc0[c][1]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float* o = out + (c0 + c) * N;
    *reinterpret_cast<float2*>(o + rowp0 + zA) = acc0[c][0];
    *reinterpret_cast<float2*>(o + rowp0 + zB) = acc0[c][1];
  }
}

// tm_box: box {P, R, 1} (tiles whose staged y rows do not wrap); tm_row: box {P, 2, 1}.
template <int FG, int P, bool UNIT>
__global__ __launch_bounds__(GP_NTH, 1) void gather_pipe_kernel(const __grid_constant__ CUtensorMap tm_box,
                                                                const __grid_constant__ CUtensorMap tm_row,
                                                                const float* __restrict__ coef, int F,
                                                                const float* __restrict__ disp,
                                                                float* __restrict__ out, int Nx, int Ny, int Nz,
                                                                float3 sc, int TY, int seg) {
  pdl_prologue();
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) unsigned long long full[GP_RING];
  __shared__ int relcnt[GP_RING];
  const long long N = (long long)Nx * Ny * Nz;
  const int R = TY + 4;
  const int x0 = blockIdx.x * seg, nx = min(seg, Nx - x0);
  const int y0 = blockIdx.y * TY;
  if (nx <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int planes = nx + 4;
  const int npass = F / FG;
  const int slot_floats = FG * R * P;
  const bool wrap_y = y0 - 2 < 0 || y0 - 2 + R > Ny;
  const int total_seq = npass * planes;

  // TMA of plane `seq` (pass seq / planes, plane p = x0 - 2 + seq % planes) into its slot
  auto fill = [&](int seq) {
    const int s = seq % GP_RING;
    const int pass = seq / planes, p = seq - pass * planes;
    const int c0 = pass * FG;
    const int x = wrapi(x0 - 2 + p, Nx);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(gp_su32(&full[s])),
                 "r"((unsigned)(FG * R * P * 4))
                 : "memory");
    float* slot = sm + (size_t)s * slot_floats;
    for (int c = 0; c < FG; ++c) {
      const int xc = (c0 + c) * Nx + x;
      float* dst = slot + c * R * P;
      if (!wrap_y) {
        gp_tma(&tm_box, dst, &full[s], 0, y0 - 2, xc);
      } else {
        // two-row boxes: y0 and Ny are even, so a pair never straddles the periodic wrap
        for (int r = 0; r < R; r += 2) gp_tma(&tm_row, dst + r * P, &full[s], 0, wrapi(y0 - 2 + r, Ny), xc);
      }
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < GP_RING; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(gp_su32(&full[s])));
      relcnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int seq = 0; seq < min(GP_RING, total_seq); ++seq) fill(seq);
  }
  __syncthreads();

  const int cw = warp;
  const int G = Nz >> 2;
  const int IPR = (TY / GP_ROWS) * G;
  const int total = nx * IPR;
  for (int pass = 0; pass < npass; ++pass) {
    const int c0 = pass * FG;
    const int base = pass * planes;
    int waited = -1, released = 0;
    auto wait_to = [&](int p) {
      while (waited < p) {
        ++waited;
        const int seq = base + waited;
        gp_wait(&full[seq % GP_RING], (seq / GP_RING) & 1);
      }
    };
    // A warp releases plane p once it is past it; the warp whose release completes the
    // count refills the slot with plane p + GP_RING (no dedicated producer warp).
    auto release_below = [&](int p) {
      while (released < p) {
        wait_to(released);
        __syncwarp();
        if (lane == 0) {
          const int seq = base + released, s = seq % GP_RING;
          __threadfence_block();
          if (atomicAdd(&relcnt[s], 1) == GP_CW - 1) {
            relcnt[s] = 0;
            __threadfence_block();
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            if (seq + GP_RING < total_seq) fill(seq + GP_RING);
          }
        }
        ++released;
      }
    };
    // item q -> (row r, y row ry2, group g), carried incrementally (no integer divisions
    // on the path): a lane's items advance by STEP = GP_CW * 32 per iteration.  The
    // displacements of the warp's next item are loaded while the current one computes
    // (the weights need them first thing).
    constexpr int STEP = GP_CW * 32;
    struct Pos {
      int r, ry, g, slot;  // slot = ring slot of plane base + r (the item's first source plane)
    };
    const int TYI = TY / GP_ROWS;  // item rows per tile row
    const int step_ry = STEP / G, step_g = STEP - step_ry * G;
    auto advance = [&](Pos& p) {
      p.g += step_g;
      p.ry += step_ry;
      if (p.g >= G) {
        p.g -= G;
        ++p.ry;
      }
      while (p.ry >= TYI) {
        p.ry -= TYI;
        ++p.r;
        p.slot = p.slot + 1 == GP_RING ? 0 : p.slot + 1;
      }
    };
    auto load = [&](int q, const Pos& p, NodeD& d0, NodeD& d1) {
      if (q < total) {
        const int j = min(y0 + GP_ROWS * p.ry, Ny - GP_ROWS);
        const long long rowp0 = ((long long)(x0 + p.r) * Ny + j) * Nz;
        const int zA = p.g == 0 ? Nz - 2 : 4 * p.g - 2, zB = 4 * p.g;
        gp_load_disp(disp, N, rowp0, zA, zB, d0);
        if (GP_ROWS == 2) gp_load_disp(disp, N, rowp0 + Nz, zA, zB, d1);
      }
    };
    Pos cur;
    {
      const int q = cw * 32 + lane;  // the one division per lane and pass
      cur.r = q / IPR;
      const int loc = q - cur.r * IPR;
      cur.ry = loc / G;
      cur.g = loc - cur.ry * G;
      cur.slot = (base + cur.r) % GP_RING;
    }
    Pos nxt = cur;
    advance(nxt);
    NodeD n0, n1;
#if GP_PREFETCH
    load(cw * 32 + lane, cur, n0, n1);
#endif
    for (int q0 = cw * 32; q0 < total; q0 += GP_CW * 32) {
      const int r_lo = __shfl_sync(0xffffffffu, cur.r, 0);
      const int r_hi = q0 + 31 < total ? __shfl_sync(0xffffffffu, cur.r, 31) : nx - 1;
      release_below(r_lo);
      wait_to(r_hi + 4);
      const int q = q0 + lane;
#if GP_PREFETCH
      const NodeD c0d = n0, c1d = n1;
      load(q + GP_CW * 32, nxt, n0, n1);
#else
      NodeD c0d, c1d;
      load(q, cur, c0d, c1d);
#endif
      const Pos at = cur;
      cur = nxt;
      advance(nxt);
      if (q < total) {
        const int r = at.r, ry2 = at.ry, g = at.g;
        const int i = x0 + r, j = y0 + GP_ROWS * ry2;
        if (j < Ny) {
          const float* pl[5];
          const float* p0 = sm + GP_ROWS * ry2 * P;
#pragma unroll
          for (int a = 0; a < 5; ++a) {
            const int sl = at.slot + a;
            pl[a] = p0 + (sl >= GP_RING ? sl - GP_RING : sl) * slot_floats;
          }
          const int offA = g == 0 ? Nz - 4 : 4 * g - 4, offB = 4 * g;
          if (GP_ROWS == 2)
            gp_item<FG, P>(c0d, c1d, pl, R * P, offA, offB, coef, disp, out, N, c0, i, j, g, Nx, Ny, Nz, sc);
          else
            gp_item1<FG, P, UNIT>(c0d, pl, R * P, offA, offB, coef, disp, out, N, c0, i, j, g, Nx, Ny, Nz, sc);
        }
      }
    }
    release_below(planes);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 gp_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

void gp_encode(CUtensorMap* tm, const float* coef, int F, const int* N, int P, int rows) {
  const cuuint64_t dims[3] = {(cuuint64_t)N[2], (cuuint64_t)N[1], (cuuint64_t)F * N[0]};
  const cuuint64_t strides[2] = {(cuuint64_t)N[2] * 4, (cuuint64_t)N[1] * N[2] * 4};
  const cuuint32_t box[3] = {(cuuint32_t)P, (cuuint32_t)rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = gp_encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(coef), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(3, "gather_pipe: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

template <int FG, int P>
void gp_launch(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc, int TY,
               cudaStream_t s) {
  const int R = TY + 4;
  const int tiles_y = ceil_div(N[1], TY);
  int nseg = std::max(1, kSMs / tiles_y);
  const int seg = ceil_div(N[0], nseg);
  nseg = ceil_div(N[0], seg);
  CUtensorMap tb, tr;
  gp_encode(&tb, coef, ncomp, N, P, std::min(R, N[1]));
  gp_encode(&tr, coef, ncomp, N, P, 2);
  const size_t smem = (size_t)GP_RING * FG * R * P * sizeof(float);
  auto go = [&](auto kern, int slot) {
    static bool attr_set[64][2] = {};
    int dev = 0;
    LDDMM_CUDA(cudaGetDevice(&dev));
    if (!attr_set[dev & 63][slot]) {
      LDDMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GP_SMEM_MAX));
      attr_set[dev & 63][slot] = true;
    }
    pdl_launch(kern, dim3(nseg, tiles_y, 1), GP_NTH, smem, s, tb, tr, coef, ncomp, disp, out, N[0], N[1], N[2], sc,
               TY, seg);
  };
  if (sc.x == 1.f && sc.y == 1.f && sc.z == 1.f)
    go(gather_pipe_kernel<FG, P, true>, 0);
  else
    go(gather_pipe_kernel<FG, P, false>, 1);
  LDDMM_LAUNCH_CHECK();
}

template <int P>
bool gp_launch_p(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                 cudaStream_t s) {
  if (N[2] > P) return false;
  // components per pass: FG divides F, so every pass runs the same item code
  const int FG = ncomp % 3 == 0 ? 3 : ncomp % 2 == 0 ? 2 : 1;
  // largest even TY whose ring fits, at most the grid's y extent
  const size_t per_row = (size_t)GP_RING * FG * P * sizeof(float);
  int TY = (int)(GP_SMEM_MAX / per_row) - 4;
  TY = std::min(TY, 32);
  if (const char* e = std::getenv("LDDMM_GP_TY")) TY = std::min(TY, std::atoi(e));  // lab override
  TY = std::min(TY, N[1]);
  TY &= ~1;
  // a warp's 32 consecutive items must span at most two output rows (ring depth 6)
  if (TY < 2 || (TY / GP_ROWS) * (N[2] / 4) < 32) return false;
  // a box of R rows must lie inside the tensor when the tile does not wrap
  if (FG == 3)
    gp_launch<3, P>(coef, ncomp, disp, out, N, sc, TY, s);
  else if (FG == 2)
    gp_launch<2, P>(coef, ncomp, disp, out, N, sc, TY, s);
  else
    gp_launch<1, P>(coef, ncomp, disp, out, N, sc, TY, s);
  return true;
}

}  // namespace

bool gather_pipe_supported(const int* N) {
  return N[2] % 4 == 0 && N[2] >= 8 && N[2] <= 256 && N[1] % 2 == 0 && N[1] >= 4 && gp_encoder() != nullptr;
}

bool launch_gather_pipe(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                        cudaStream_t s) {
  if (!gather_pipe_supported(N)) return false;
  return gp_launch_p<64>(coef, ncomp, disp, out, N, sc, s) || gp_launch_p<128>(coef, ncomp, disp, out, N, sc, s) ||
         gp_launch_p<192>(coef, ncomp, disp, out, N, sc, s) || gp_launch_p<256>(coef, ncomp, disp, out, N, sc, s);
}

}  // namespace lddmm_b200
