// Band-limited projection / embedding as separable truncated DFTs (sm_100a).
//
// Replaces spectral.hpp:242-285 (project/embed through a full-grid C2C FFT,
// fft.hpp:69-101).  A band field holds the centred truncation of the unscaled
// forward DFT (K_a modes per axis, DFT order, band-Nyquist planes zero,
// spectral.hpp:8-12).  Because every embedded field is real, only the half
// band kz in [0, Kz/2) along the fastest axis is carried:
//
//   embed   C[kx,ky,kz] --prep--> D[kx,ky,kz<H]           (fold + symbol, fp64->fp32)
//           --Y--> E1[kx,y,kz] --X--> E2[x,y,kz] --Z--> f[x,y,z]   (real output, /N)
//   project f[x,y,z] --Z--> G1[x,y,kz] --X--> G2[kx,y,kz] --Y--> G3[kx,ky,kz]
//           --finalize--> C[kx,ky,kz]  (Hermitian completion kz<0, Nyquist zero, fp64)
//
// The fold D = C(k) + conj(C(-k)) for kz > 0 makes Re(sum over the half band)
// identical to the reference's Re(full complex inverse DFT) for ANY coefficient
// set, including ones that are only Hermitian to round-off.  Symbols that are
// Hermitian (i*omega derivatives, the B-spline prefilter 1/B(k), real scales)
// commute with the fold and are applied in the prep step.
//
// X/Y stages are batched complex GEMMs against fp32 twiddle tables generated in
// fp64; the Z stages are real GEMMs (K = Kz for embed, K = Nz for project).
// All products accumulate in fp32.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

// ---------------------------------------------------------------------------
// prep: fp64 band -> fp32 half band with fold and symbol

// element (f, fx, fy, fz) of the fp32 half band D (fold, symbols, scale)
__device__ __forceinline__ float2 prep_value(const PrepArgs& a, int f, int fx, int fy, int fz, int Kx, int Ky, int Kz,
                                             int Nx, int Ny, int Nz, double wx, double wy, double wz,
                                             const double* __restrict__ bsym) {
  float2 out = make_float2(0.f, 0.f);
  const PrepField pf = a.f[f];
  if (fx != Kx / 2 && fy != Ky / 2 && pf.src != nullptr) {
    const double2* C = pf.src;
    double2 v = C[((long long)fx * Ky + fy) * Kz + fz];
    if (fz > 0) {
      const int mx = (Kx - fx) % Kx, my = (Ky - fy) % Ky, mz = Kz - fz;
      const double2 w = C[((long long)mx * Ky + my) * Kz + mz];
      v.x += w.x;
      v.y -= w.y;
    }
    const int kx = fx < Kx / 2 ? fx : fx - Kx;
    const int ky = fy < Ky / 2 ? fy : fy - Ky;
    const int kz = fz;
    double s = pf.scale;
    if (pf.sym & SYM_PREFILTER) {
      // 1 / B(k), B(k) = prod_a (4 + 2 cos(2 pi k_a / N_a)) / 6 (exact periodic cubic
      // B-spline prefilter of interp.hpp:23-63 in Fourier form)
      // per-axis factors from the plan's table (band_symbol_kernel: the same expressions,
      // so the same doubles as evaluating them here)
      const double bx = __ldg(bsym + fx), by = __ldg(bsym + Kx + fy), bz = __ldg(bsym + Kx + Ky + fz);
      s /= (bx * by * bz);
    }
    const int dax = pf.sym & SYM_DERIV_MASK;
    if (dax) {
      // band_derivative: multiply by i*omega_a, omega = 2 pi k / (N_a h_a) (spectral.hpp:77-79,419-427)
      const double om = dax == 1 ? wx * kx : (dax == 2 ? wy * ky : wz * kz);
      const double re = -v.y * om, im = v.x * om;
      v.x = re;
      v.y = im;
    }
    out = make_float2((float)(v.x * s), (float)(v.y * s));
  }
  return out;
}

// B(k) factors (4 + 2 cos(2 pi k_a / N_a)) / 6 per axis and band index (signed frequency),
// concatenated [Kx | Ky | Kz], for the prefilter symbol of prep_value
__global__ void band_symbol_kernel(int Kx, int Ky, int Kz, int Nx, int Ny, int Nz, double* __restrict__ out) {
  pdl_prologue();
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < Kx + Ky + Kz; t += gridDim.x * blockDim.x) {
    double v;
    if (t < Kx) {
      const int kx = t < Kx / 2 ? t : t - Kx;
      v = (4.0 + 2.0 * cospi(2.0 * kx / Nx)) / 6.0;
    } else if (t < Kx + Ky) {
      const int f = t - Kx, ky = f < Ky / 2 ? f : f - Ky;
      v = (4.0 + 2.0 * cospi(2.0 * ky / Ny)) / 6.0;
    } else {
      const int kz = t - Kx - Ky;
      v = (4.0 + 2.0 * cospi(2.0 * kz / Nz)) / 6.0;
    }
    out[t] = v;
  }
}

void launch_band_symbols(const int* K, const int* N, double* out, cudaStream_t s) {
  pdl_launch(band_symbol_kernel, 1, 256, 0, s, K[0], K[1], K[2], N[0], N[1], N[2], out);
  LDDMM_LAUNCH_CHECK();
}

__global__ void band_prep_kernel(PrepArgs a, int Kx, int Ky, int Kz, int Nx, int Ny, int Nz, double wx,
                                 double wy, double wz, const double* __restrict__ bsym, float2* __restrict__ D) {
  pdl_prologue();
  const int H = Kz / 2;
  const long long per = (long long)Kx * Ky * H;
  const long long total = per * a.nf;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(t / per);
    long long r = t - (long long)f * per;
    const int fz = (int)(r % H);
    r /= H;
    const int fy = (int)(r % Ky);
    const int fx = (int)(r / Ky);
    D[t] = prep_value(a, f, fx, fy, fz, Kx, Ky, Kz, Nx, Ny, Nz, wx, wy, wz, bsym);
  }
}

// ---------------------------------------------------------------------------
// finalize: G3 half band (fp32) -> full band fp64 with Hermitian completion

__global__ void band_finalize_kernel(FinArgs a, int Kx, int Ky, int Kz, const float2* __restrict__ G) {
  pdl_prologue();
  const int H = Kz / 2;
  const long long per = (long long)Kx * Ky * Kz;
  const long long total = per * a.nf;
  const long long gper = (long long)Kx * Ky * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(t / per);
    long long r = t - (long long)f * per;
    const int fz = (int)(r % Kz);
    r /= Kz;
    const int fy = (int)(r % Ky);
    const int fx = (int)(r / Ky);
    double gx = 0.0, gy = 0.0;
    if (fx != Kx / 2 && fy != Ky / 2 && fz != H) {
      const float2* Gf = G + (long long)f * gper;
      if (fz < H) {
        const float2 g = Gf[((long long)fx * Ky + fy) * H + fz];
        gx = g.x;
        gy = g.y;
      } else {
        const int mx = (Kx - fx) % Kx, my = (Ky - fy) % Ky, mz = Kz - fz;
        const float2 g = Gf[((long long)mx * Ky + my) * H + mz];
        gx = g.x;
        gy = -g.y;
      }
    }
    const FinField ff = a.f[f];
    const long long idx = r * Kz + fz;  // (fx*Ky+fy)*Kz+fz
    double2 o = make_double2(ff.alpha * gx, ff.alpha * gy);
    if (ff.add) {
      const double2 ad = ff.add[idx];
      o.x += ff.beta * ad.x;
      o.y += ff.beta * ad.y;
    }
    ff.dst[idx] = o;
  }
}

// ---------------------------------------------------------------------------
// batched complex GEMM: C[b][m][n] = sum_k A[m][k] * B[b][k][n]
// 32x32 tile, 256 threads, 2x2 complex outputs per thread, BK = 16.

constexpr int CG_BM = 32, CG_BN = 32, CG_BK = 16;

__device__ __forceinline__ void cp_async8_f2(float2* smem, const float2* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// k-chunks staged with 8-byte cp.async and double-buffered: the next chunk
// streams in while the current one is multiplied.
__global__ __launch_bounds__(256) void cgemm_kernel(const float2* __restrict__ A, int lda,
                                                    const float2* __restrict__ B, long long sB, int ldb,
                                                    float2* __restrict__ C, long long sC, int ldc, int M,
                                                    int N, int K) {
  pdl_prologue();
  __shared__ float2 As[2][CG_BK][CG_BM + 1];
  __shared__ float2 Bs[2][CG_BK][CG_BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * CG_BM, n0 = blockIdx.x * CG_BN;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  float2 acc[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  auto stage = [&](int buf, int k0) {
    for (int e = tid; e < CG_BM * CG_BK; e += 256) {
      const int mm = e / CG_BK, kk = e % CG_BK;
      const int gm = m0 + mm, gk = k0 + kk;
      if (gm < M && gk < K)
        cp_async8_f2(&As[buf][kk][mm], A + (long long)gm * lda + gk);
      else
        As[buf][kk][mm] = make_float2(0.f, 0.f);
    }
    for (int e = tid; e < CG_BK * CG_BN; e += 256) {
      const int kk = e / CG_BN, nn = e % CG_BN;
      const int gk = k0 + kk, gn = n0 + nn;
      if (gk < K && gn < N)
        cp_async8_f2(&Bs[buf][kk][nn], B + (long long)gk * ldb + gn);
      else
        Bs[buf][kk][nn] = make_float2(0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  stage(0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += CG_BK, buf ^= 1) {
    if (k0 + CG_BK < K) {
      stage(buf ^ 1, k0 + CG_BK);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < CG_BK; ++kk) {
      const float2 a0 = As[buf][kk][ty], a1 = As[buf][kk][ty + 16];
      const float2 b0 = Bs[buf][kk][tx], b1 = Bs[buf][kk][tx + 16];
      acc[0][0].x = fmaf(a0.x, b0.x, fmaf(-a0.y, b0.y, acc[0][0].x));
      acc[0][0].y = fmaf(a0.x, b0.y, fmaf(a0.y, b0.x, acc[0][0].y));
      acc[0][1].x = fmaf(a0.x, b1.x, fmaf(-a0.y, b1.y, acc[0][1].x));
      acc[0][1].y = fmaf(a0.x, b1.y, fmaf(a0.y, b1.x, acc[0][1].y));
      acc[1][0].x = fmaf(a1.x, b0.x, fmaf(-a1.y, b0.y, acc[1][0].x));
      acc[1][0].y = fmaf(a1.x, b0.y, fmaf(a1.y, b0.x, acc[1][0].y));
      acc[1][1].x = fmaf(a1.x, b1.x, fmaf(-a1.y, b1.y, acc[1][1].x));
      acc[1][1].y = fmaf(a1.x, b1.y, fmaf(a1.y, b1.x, acc[1][1].y));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < M && gn < N) C[(long long)gm * ldc + gn] = acc[i][j];
    }
}

// ---------------------------------------------------------------------------
// batched real GEMM for the Z stages: C[b][m][n] = sum_k A[b][m][k] * B[k][n]
// BM = 128 (or 32 for grids with few row tiles: 4x the CTAs), BK = 16, thread tile RT x 4
// (RT = 8 or 2).  BN = 64 (256 threads) or 32 (128 threads).  Every output sums its K terms
// in the same order for any BM.

template <int BN, int BM = 128>
__global__ __launch_bounds__(BN * 4) void sgemm_kernel(const float* __restrict__ A, int lda, long long sA,
                                                       const float* __restrict__ B, int ldb,
                                                       float* __restrict__ C, int ldc, long long sC, int M,
                                                       int N, int K) {
  pdl_prologue();
  constexpr int BK = 16, NT = BN * 4, TXN = BN / 4, RT = BM * TXN / NT;
  static_assert(RT == 8 || RT == 2, "thread tile rows");
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % TXN, ty = tid / TXN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  A += blockIdx.z * sA;
  C += blockIdx.z * sC;
  float acc[RT][4];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll 4
    for (int e = tid; e < BM * BK; e += NT) {
      const int mm = e / BK, kk = e % BK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? __ldg(A + (long long)gm * lda + gk) : 0.f;
    }
#pragma unroll 4
    for (int e = tid; e < BK * BN; e += NT) {
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? __ldg(B + (long long)gk * ldb + gn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[RT];
      if constexpr (RT == 8) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
        av[0] = a0.x, av[1] = a0.y, av[2] = a0.z, av[3] = a0.w, av[4] = a1.x, av[5] = a1.y, av[6] = a1.z,
        av[7] = a1.w;
      } else {
        const float2 a0 = *reinterpret_cast<const float2*>(&As[kk][ty * 2]);
        av[0] = a0.x, av[1] = a0.y;
      }
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int gn = n0 + tx * 4;
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int gm = m0 + ty * RT + i;
    if (gm >= M) break;
    float* crow = C + (long long)gm * ldc;
    if (gn + 3 < N && (ldc & 3) == 0) {
      *reinterpret_cast<float4*>(crow + gn) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (gn + j < N) crow[gn + j] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers

void launch_band_prep(const PrepArgs& a, const DftPlan& p, float2* D, cudaStream_t s) {
  const long long total = (long long)p.K[0] * p.K[1] * (p.K[2] / 2) * a.nf;
  pdl_launch(band_prep_kernel, grid_for(total, 256), 256, 0, s, a, p.K[0], p.K[1], p.K[2], p.N[0], p.N[1], p.N[2],
                                                        p.omega_unit[0], p.omega_unit[1], p.omega_unit[2], p.bsym, D);
  LDDMM_LAUNCH_CHECK();
}

void launch_band_finalize(const FinArgs& a, const DftPlan& p, const float2* G, cudaStream_t s) {
  const long long total = (long long)p.K[0] * p.K[1] * p.K[2] * a.nf;
  pdl_launch(band_finalize_kernel, grid_for(total, 256), 256, 0, s, a, p.K[0], p.K[1], p.K[2], G);
  LDDMM_LAUNCH_CHECK();
}

// Batched complex GEMM for the y stages (small M x N per batch item, K up to Ny):
// the twiddle matrix A and one whole B slab live in shared memory, so the K loop
// runs without barriers; one batch item per CTA iteration, 2 x 2 complex outputs
// per thread.  (The k-chunked cgemm_kernel spent most of its time in barriers and
// global-load latency on these shapes.)

struct PrepCtx {
  PrepArgs a;
  int Kx, Ky, Kz, Nx, Ny, Nz;
  double wx, wy, wz;
  const double* bsym;  // the plan's B(k) factor table (band_symbol_kernel)
};

struct FinCtx {
  FinArgs a;
  int Kx, Ky, Kz;
};

// one projected half-band value g of output (f, fx, fy, fz) -> the fp64 band field,
// as band_finalize_kernel computes it (zero Nyquist planes, alpha / beta combine)
__device__ __forceinline__ void fin_store(const FinCtx& fc, int f, int fx, int fy, int fz, double gx, double gy) {
  const int H = fc.Kz / 2;
  if (fx == fc.Kx / 2 || fy == fc.Ky / 2 || fz == H) gx = gy = 0.0;
  const FinField ff = fc.a.f[f];
  const long long idx = ((long long)fx * fc.Ky + fy) * fc.Kz + fz;
  double2 o = make_double2(ff.alpha * gx, ff.alpha * gy);
  if (ff.add) {
    const double2 ad = ff.add[idx];
    o.x += ff.beta * ad.x;
    o.y += ff.beta * ad.y;
  }
  ff.dst[idx] = o;
}

// y-project output (batch b = (f, fx), row fy, column h < H): its own band entry and
// the Hermitian mirror entry ((Kx-fx)%Kx, (Ky-fy)%Ky, Kz-h) for 0 < h < H — every
// band entry of the field is written by exactly one CTA
__device__ __forceinline__ void fin_pair(const FinCtx& fc, int f, int fx, int fy, int h, float2 g) {
  fin_store(fc, f, fx, fy, h, g.x, g.y);
  if (h > 0) fin_store(fc, f, (fc.Kx - fx) % fc.Kx, (fc.Ky - fy) % fc.Ky, fc.Kz - h, g.x, -(double)g.y);
}

// MODE 1 (PREP): the y-embed with the band prep fused in — B[b] (batch b = (f, fx))
// is the half-band slab D[f][fx][.][.], computed from the fp64 band while it is
// staged (bitwise the values band_prep_kernel would have written).
// MODE 2 (FIN): the y-project with the band finalize fused in — the batch's outputs
// go straight to the fp64 band fields (fin_pair) instead of G3.
//
// Work split (cgemm_split, a function of the shape only, so every MODE of a shape sums
// in the same order): a batch item spans MS CTAs (rows [ms mrows, (ms+1) mrows)), and
// with a long K (the y-project, K = Ny) each 2 x 2 output tile is summed by KS threads
// over K slices, combined through shared memory in slice order — one CTA per batch
// item with 128 busy threads left 52 SMs idle and ran K = 210 serial FMA chains.
struct CgemmSplit {
  int MS, KS, mrows;
};

static CgemmSplit cgemm_split(int M, int N, int K, int batch) {
  CgemmSplit sp;
  // 2 (or 4) CTAs per batch item when the grid is short of CTAs or one CTA's twiddle slab
  // (M (K + 1) complex) would hold an SM alone (config 4: 131 KB -> 1 CTA of 8 warps per SM)
  const size_t slab = (size_t)M * (K + 1) * sizeof(float2);
  const int msplit = std::getenv("LDDMM_Y_MS") ? std::atoi(std::getenv("LDDMM_Y_MS")) : 0;  // lab override
  sp.MS = M >= 8 && (batch < 2 * kSMs || slab > 64 * 1024) ? 2 : 1;
  if (M >= 16 && slab > 128 * 1024) sp.MS = 4;
  if (msplit > 0) sp.MS = msplit;
  sp.mrows = ((M + sp.MS - 1) / sp.MS + 1) & ~1;
  const int tiles = (sp.mrows / 2) * ((N + 1) / 2);
  sp.KS = 1;
  if (K > 64)
    while (sp.KS < 8 && tiles * sp.KS * 2 <= 256) sp.KS *= 2;
  return sp;
}

template <int MODE>
__global__ __launch_bounds__(256) void cgemm_smem_kernel(const float2* __restrict__ A, int lda,
                                                         const float2* __restrict__ B, long long sB, int ldb,
                                                         float2* __restrict__ C, long long sC, int ldc, int M, int N,
                                                         int K, int batch, int MS, int KS, int mrows,
                                                         const __grid_constant__ PrepCtx pc,
                                                         const __grid_constant__ FinCtx fc) {
  constexpr bool PREP = MODE == 1, FIN = MODE == 2;
  extern __shared__ float2 sm2[];
  const int KP = K + 1;  // padded A row (bank spread across rows)
  const int b = blockIdx.x / MS, ms = blockIdx.x - b * MS;
  const int m_lo = ms * mrows, mh = min(M, m_lo + mrows) - m_lo;  // this CTA's rows
  float2* As = sm2;
  float2* Bs = sm2 + (long long)mrows * KP;
  float4* red = reinterpret_cast<float4*>(Bs + (long long)K * N);  // KS > 1: [KS][tiles] x 2 float4
  // cp.async (8-byte) copies: every element in flight at once, no register round trip.
  // A is a twiddle table (constant): staged before the PDL wait, overlapping the
  // preceding kernel's tail.
  for (int e = threadIdx.x; e < mh * K; e += blockDim.x) {
    const int m = e / K, k = e - (e / K) * K;
    cp_async8_f2(As + m * KP + k, A + (long long)(m_lo + m) * lda + k);
  }
  pdl_wait();
  pdl_trigger();
  if (mh <= 0) return;
  const int tn = (N + 1) / 2, tiles = ((mh + 1) / 2) * tn;
  if (PREP) {
    const int f = b / pc.Kx, fx = b - f * pc.Kx;
    for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
      const int k = e / N, n = e - (e / N) * N;
      Bs[e] = prep_value(pc.a, f, fx, k, n, pc.Kx, pc.Ky, pc.Kz, pc.Nx, pc.Ny, pc.Nz, pc.wx, pc.wy, pc.wz, pc.bsym);
    }
  } else {
    const float2* Bb = B + b * sB;
    for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
      const int k = e / N, n = e - (e / N) * N;
      cp_async8_f2(Bs + e, Bb + (long long)k * ldb + n);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  float2* Cb = C + b * sC;
  auto emit = [&](int m0, int n0, float2 c00, float2 c01, float2 c10, float2 c11) {
    const int M0 = m_lo + m0;
    if (FIN) {
      const int f = b / fc.Kx, fx = b - f * fc.Kx;
      fin_pair(fc, f, fx, M0, n0, c00);
      if (n0 + 1 < N) fin_pair(fc, f, fx, M0, n0 + 1, c01);
      if (m0 + 1 < mh) {
        fin_pair(fc, f, fx, M0 + 1, n0, c10);
        if (n0 + 1 < N) fin_pair(fc, f, fx, M0 + 1, n0 + 1, c11);
      }
    } else {
      Cb[(long long)M0 * ldc + n0] = c00;
      if (n0 + 1 < N) Cb[(long long)M0 * ldc + n0 + 1] = c01;
      if (m0 + 1 < mh) {
        Cb[(long long)(M0 + 1) * ldc + n0] = c10;
        if (n0 + 1 < N) Cb[(long long)(M0 + 1) * ldc + n0 + 1] = c11;
      }
    }
  };
  const int kslice = (K + KS - 1) / KS;
  // tall shapes (the y-embed: M = Ny rows): 4 x 2 output tiles per thread, the two B
  // values of a k step shared by four rows (6 shared loads per 32 FMA instead of 4 per 16);
  // every output still sums its K terms in order
  const int tiles4 = ((mh + 3) / 4) * tn;
  if (KS == 1 && tiles4 >= 128) {
    for (int t = threadIdx.x; t < tiles4; t += blockDim.x) {
      const int m0 = (t / tn) * 4, n0 = (t - (t / tn) * tn) * 2;
      const int n1 = min(n0 + 1, N - 1);
      const float2* ap[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ap[i] = As + min(m0 + i, mh - 1) * KP;
      float2 c[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const float2 b0 = Bs[k * N + n0], b1 = Bs[k * N + n1];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 a = ap[i][k];
          c[i][0].x = fmaf(a.x, b0.x, fmaf(-a.y, b0.y, c[i][0].x));
          c[i][0].y = fmaf(a.x, b0.y, fmaf(a.y, b0.x, c[i][0].y));
          c[i][1].x = fmaf(a.x, b1.x, fmaf(-a.y, b1.y, c[i][1].x));
          c[i][1].y = fmaf(a.x, b1.y, fmaf(a.y, b1.x, c[i][1].y));
        }
      }
      emit(m0, n0, c[0][0], c[0][1], c[1][0], c[1][1]);
      if (m0 + 2 < mh) emit(m0 + 2, n0, c[2][0], c[2][1], c[3][0], c[3][1]);
    }
  } else
  for (int it = threadIdx.x; it < tiles * KS; it += blockDim.x) {
    const int t = it % tiles, ks = it / tiles;
    const int m0 = (t / tn) * 2, n0 = (t - (t / tn) * tn) * 2;
    const int m1 = min(m0 + 1, mh - 1), n1 = min(n0 + 1, N - 1);
    float2 c00 = make_float2(0.f, 0.f), c01 = c00, c10 = c00, c11 = c00;
    const float2* a0p = As + m0 * KP;
    const float2* a1p = As + m1 * KP;
    const int k_lo = ks * kslice, k_hi = min(K, k_lo + kslice);
#pragma unroll 4
    for (int k = k_lo; k < k_hi; ++k) {
      const float2 a0 = a0p[k], a1 = a1p[k];
      const float2 b0 = Bs[k * N + n0], b1 = Bs[k * N + n1];
      c00.x = fmaf(a0.x, b0.x, fmaf(-a0.y, b0.y, c00.x));
      c00.y = fmaf(a0.x, b0.y, fmaf(a0.y, b0.x, c00.y));
      c01.x = fmaf(a0.x, b1.x, fmaf(-a0.y, b1.y, c01.x));
      c01.y = fmaf(a0.x, b1.y, fmaf(a0.y, b1.x, c01.y));
      c10.x = fmaf(a1.x, b0.x, fmaf(-a1.y, b0.y, c10.x));
      c10.y = fmaf(a1.x, b0.y, fmaf(a1.y, b0.x, c10.y));
      c11.x = fmaf(a1.x, b1.x, fmaf(-a1.y, b1.y, c11.x));
      c11.y = fmaf(a1.x, b1.y, fmaf(a1.y, b1.x, c11.y));
    }
    if (KS == 1) {
      emit(m0, n0, c00, c01, c10, c11);
    } else {
      red[(ks * tiles + t) * 2] = make_float4(c00.x, c00.y, c01.x, c01.y);
      red[(ks * tiles + t) * 2 + 1] = make_float4(c10.x, c10.y, c11.x, c11.y);
    }
  }
  if (KS > 1) {
    __syncthreads();
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
      float4 p = red[t * 2], q = red[t * 2 + 1];
      for (int ks = 1; ks < KS; ++ks) {
        const float4 p2 = red[(ks * tiles + t) * 2], q2 = red[(ks * tiles + t) * 2 + 1];
        p.x += p2.x, p.y += p2.y, p.z += p2.z, p.w += p2.w;
        q.x += q2.x, q.y += q2.y, q.z += q2.z, q.w += q2.w;
      }
      const int m0 = (t / tn) * 2, n0 = (t - (t / tn) * tn) * 2;
      emit(m0, n0, make_float2(p.x, p.y), make_float2(p.z, p.w), make_float2(q.x, q.y), make_float2(q.z, q.w));
    }
  }
  if (FIN && ms == 0) {
    // the kz = Kz/2 plane (zero projection) of this batch's rows
    const int f = b / fc.Kx, fx = b - f * fc.Kx;
    for (int fy = threadIdx.x; fy < M; fy += blockDim.x) fin_store(fc, f, fx, fy, fc.Kz / 2, 0.0, 0.0);
  }
}

static size_t cgemm_smem_bytes(int M, int N, int K, int batch) {
  const CgemmSplit sp = cgemm_split(M, N, K, batch);
  const int tiles = (sp.mrows / 2) * ((N + 1) / 2);
  return ((size_t)sp.mrows * (K + 1) + (size_t)K * N) * sizeof(float2) +
         (sp.KS > 1 ? (size_t)sp.KS * tiles * 2 * sizeof(float4) : 0);
}

static bool cgemm_smem_fits(int M, int N, int K) {
  return N <= 64 && ((size_t)M * (K + 1) + (size_t)K * N) * sizeof(float2) <= 200 * 1024;
}

template <int MODE>
static void launch_cgemm_smem(const float2* A, int lda, const float2* B, long long sB, int ldb, float2* C,
                              long long sC, int ldc, int M, int N, int K, int batch, const PrepCtx& pc,
                              const FinCtx& fc, cudaStream_t s) {
  const CgemmSplit sp = cgemm_split(M, N, K, batch);
  const size_t smem = cgemm_smem_bytes(M, N, K, batch);
  static bool attr_set[64] = {false};
  int dev = 0;
  LDDMM_CUDA(cudaGetDevice(&dev));
  if (!attr_set[dev & 63]) {
    LDDMM_CUDA(
        cudaFuncSetAttribute(cgemm_smem_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set[dev & 63] = true;
  }
  pdl_launch(cgemm_smem_kernel<MODE>, batch * sp.MS, 256, smem, s, A, lda, B, sB, ldb, C, sC, ldc, M, N, K, batch,
             sp.MS, sp.KS, sp.mrows, pc, fc);
  LDDMM_LAUNCH_CHECK();
}

void launch_cgemm(const float2* A, int lda, const float2* B, long long sB, int ldb, float2* C, long long sC,
                  int ldc, int M, int N, int K, int batch, cudaStream_t s) {
  if (cgemm_smem_fits(M, N, K)) {
    static const PrepCtx none{};
    static const FinCtx nofin{};
    launch_cgemm_smem<0>(A, lda, B, sB, ldb, C, sC, ldc, M, N, K, batch, none, nofin, s);
    return;
  }
  dim3 grid(ceil_div(N, CG_BN), ceil_div(M, CG_BM), batch);
  pdl_launch(cgemm_kernel, grid, 256, 0, s, A, lda, B, sB, ldb, C, sC, ldc, M, N, K);
  LDDMM_LAUNCH_CHECK();
}

void launch_sgemm(const float* A, int lda, long long sA, const float* B, int ldb, float* C, int ldc,
                  long long sC, int M, int N, int K, int batch, cudaStream_t s) {
  if (N <= 32 && (long long)ceil_div(M, 128) * batch < kSMs) {
    // few row tiles (the small product grid's z-project: 51 CTAs): 32-row tiles
    dim3 grid(ceil_div(N, 32), ceil_div(M, 32), batch);
    pdl_launch(sgemm_kernel<32, 32>, grid, 128, 0, s, A, lda, sA, B, ldb, C, ldc, sC, M, N, K);
  } else if (N <= 32) {
    dim3 grid(ceil_div(N, 32), ceil_div(M, 128), batch);
    pdl_launch(sgemm_kernel<32>, grid, 128, 0, s, A, lda, sA, B, ldb, C, ldc, sC, M, N, K);
  } else {
    dim3 grid(ceil_div(N, 64), ceil_div(M, 128), batch);
    pdl_launch(sgemm_kernel<64>, grid, 256, 0, s, A, lda, sA, B, ldb, C, ldc, sC, M, N, K);
  }
  LDDMM_LAUNCH_CHECK();
}

// z stages on the tensor cores (3xTF32) unless LDDMM_TC=0
static bool use_tensor_cores() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LDDMM_TC");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// z-embed on tcgen05 (umma_gemm.cu) unless LDDMM_UMMA=0
static bool use_umma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LDDMM_UMMA");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static void dft_embed_xz(const DftPlan& p, int nf, const float2* E1, float2* E2, float* out, cudaStream_t s);

// embed nf half-band fields D[nf][Kx][Ky][H] -> grid fields out[nf][N] (fp32)
void dft_embed(const DftPlan& p, const float2* D, int nf, float2* E1, float2* E2, float* out, cudaStream_t s) {
  const int Kx = p.K[0], Ky = p.K[1], H = p.K[2] / 2;
  const int Ny = p.N[1];
  // Y: for each (f,kx): E1[Ny x H] = Wy[Ny x Ky] * D[Ky x H]
  launch_cgemm(p.wy_e, Ky, D, (long long)Ky * H, H, E1, (long long)Ny * H, H, Ny, H, Ky, nf * Kx, s);
  dft_embed_xz(p, nf, E1, E2, out, s);
}

// band prep + embed with the prep fused into the y stage (no D round trip, one launch
// fewer); D is only used when the y-stage operands exceed the shared-memory kernel
void dft_embed_prep(const DftPlan& p, const PrepArgs& a, float2* D, float2* E1, float2* E2, float* out,
                    cudaStream_t s) {
  const int Kx = p.K[0], Ky = p.K[1], H = p.K[2] / 2;
  const int Ny = p.N[1];
  if (!cgemm_smem_fits(Ny, H, Ky) || std::getenv("LDDMM_NO_PREP_FUSION")) {
    launch_band_prep(a, p, D, s);
    dft_embed(p, D, a.nf, E1, E2, out, s);
    return;
  }
  PrepCtx pc;
  pc.a = a;
  pc.Kx = Kx, pc.Ky = Ky, pc.Kz = p.K[2], pc.Nx = p.N[0], pc.Ny = p.N[1], pc.Nz = p.N[2];
  pc.wx = p.omega_unit[0], pc.wy = p.omega_unit[1], pc.wz = p.omega_unit[2];
  pc.bsym = p.bsym;
  static const FinCtx nofin{};
  launch_cgemm_smem<1>(p.wy_e, Ky, nullptr, 0, H, E1, (long long)Ny * H, H, Ny, H, Ky, a.nf * Kx, pc, nofin, s);
  dft_embed_xz(p, a.nf, E1, E2, out, s);
}

static void dft_embed_xz(const DftPlan& p, int nf, const float2* E1, float2* E2, float* out, cudaStream_t s) {
  const int Kx = p.K[0], H = p.K[2] / 2;
  const int Nx = p.N[0], Ny = p.N[1], Nz = p.N[2];
  // X: for each f: E2[Nx x (Ny H)] = Wx[Nx x Kx] * E1[Kx x (Ny H)]
  if (p.ux_e)
    launch_umma_xstage(p.ux_e, E1, (long long)Kx * Ny * H, E2, (long long)Nx * Ny * H, Nx, Ny * H, Kx, nf, s);
  else
    launch_cgemm(p.wx_e, Kx, E1, (long long)Kx * Ny * H, Ny * H, E2, (long long)Nx * Ny * H, Ny * H, Nx, Ny * H,
                 Kx, nf, s);
  // Z: for each f: out[(Nx Ny) x Nz] = E2 as float[(Nx Ny) x 2H] * Tz_e[2H x Nz]
  if (use_tensor_cores() && use_umma() && p.uz_e_big)
    launch_umma_zembed(reinterpret_cast<const float*>(E2), (long long)Nx * Ny * 2 * H, p.uz_e_big, p.uz_e_small, out,
                       (long long)Nx * Ny * Nz, Nx * Ny, Nz, 2 * H, nf, s);
  else if (use_tensor_cores())
    launch_tc3_gemm(reinterpret_cast<const float*>(E2), 2 * H, (long long)Nx * Ny * 2 * H, p.tz_e_big, p.tz_e_small,
                    Nz, out, Nz, (long long)Nx * Ny * Nz, Nx * Ny, Nz, 2 * H, nf, s);
  else
    launch_sgemm(reinterpret_cast<const float*>(E2), 2 * H, (long long)Nx * Ny * 2 * H, p.tz_e, Nz, out, Nz,
                 (long long)Nx * Ny * Nz, Nx * Ny, Nz, 2 * H, nf, s);
}

// project nf grid fields f[nf][N] -> half band G3[nf][Kx][Ky][H]
static void dft_project_zx(const DftPlan& p, const float* f, int nf, float2* G1, float2* G2, cudaStream_t s) {
  const int Kx = p.K[0], H = p.K[2] / 2;
  const int Nx = p.N[0], Ny = p.N[1], Nz = p.N[2];
  // small product grid: the FFMA tiled GEMM (9 us) beats the mma.sync one (15 us) at
  // K = Nz = 46 with its unaligned rows (scalar loads in the tensor-core kernel)
  const bool small = (long long)Nx * Ny * Nz < (1LL << 20);
  if (use_tensor_cores() && use_umma() && p.uz_p_big)
    launch_umma_zproject(f, p.uz_p_big, p.uz_p_small, reinterpret_cast<float*>(G1), nf * Nx * Ny, Nz, 2 * H, s);
  else if (use_tensor_cores() && !small)
    launch_tc3_gemm(f, Nz, (long long)Nx * Ny * Nz, p.tz_p_big, p.tz_p_small, 2 * H, reinterpret_cast<float*>(G1),
                    2 * H, (long long)Nx * Ny * 2 * H, Nx * Ny, 2 * H, Nz, nf, s);
  else
    launch_sgemm(f, Nz, (long long)Nx * Ny * Nz, p.tz_p, 2 * H, reinterpret_cast<float*>(G1), 2 * H,
                 (long long)Nx * Ny * 2 * H, Nx * Ny, 2 * H, Nz, nf, s);
  if (p.ux_p)
    launch_umma_xstage(p.ux_p, G1, (long long)Nx * Ny * H, G2, (long long)Kx * Ny * H, Kx, Ny * H, Nx, nf, s);
  else
    launch_cgemm(p.wx_p, Nx, G1, (long long)Nx * Ny * H, Ny * H, G2, (long long)Kx * Ny * H, Ny * H, Kx, Ny * H,
                 Nx, nf, s);
}

void dft_project(const DftPlan& p, const float* f, int nf, float2* G1, float2* G2, float2* G3, cudaStream_t s) {
  const int Kx = p.K[0], Ky = p.K[1], H = p.K[2] / 2;
  const int Ny = p.N[1];
  dft_project_zx(p, f, nf, G1, G2, s);
  launch_cgemm(p.wy_p, Ny, G2, (long long)Ny * H, H, G3, (long long)Ky * H, H, Ky, H, Ny, nf * Kx, s);
}

// project + band finalize with the finalize fused into the y stage (no G3 round trip,
// one launch fewer)
void dft_project_fin(const DftPlan& p, const float* f, const FinArgs& a, float2* G1, float2* G2, float2* G3,
                     cudaStream_t s) {
  const int Kx = p.K[0], Ky = p.K[1], H = p.K[2] / 2;
  const int Ny = p.N[1];
  if (!cgemm_smem_fits(Ky, H, Ny) || std::getenv("LDDMM_NO_FIN_FUSION")) {
    dft_project(p, f, a.nf, G1, G2, G3, s);
    launch_band_finalize(a, p, G3, s);
    return;
  }
  dft_project_zx(p, f, a.nf, G1, G2, s);
  static const PrepCtx none{};
  FinCtx fc;
  fc.a = a;
  fc.Kx = Kx, fc.Ky = Ky, fc.Kz = p.K[2];
  launch_cgemm_smem<2>(p.wy_p, Ny, G2, (long long)Ny * H, H, nullptr, 0, H, Ky, H, Ny, a.nf * Kx, none, fc, s);
}

}  // namespace lddmm_b200
