// tcgen05 (5th-generation tensor core) 3xTF32 complex GEMM for the x stage of the
// truncated DFT (spectral.hpp:242-285 embed / project, the x pass of the separable
// transform):
//
//   C[f][m][n] = sum_k W[m][k] X[f][k][n]      (complex; n = (y, kz) columns)
//
//   embed:   W = Wx_e [Nx][Kx]  exp(+2 pi i kx x / Nx),  X = E1 [Kx][Ny H],  C = E2 [Nx][Ny H]
//   project: W = Wx_p [Kx][Nx]  exp(-2 pi i kx x / Nx),  X = G1 [Nx][Ny H],  C = G2 [Kx][Ny H]
//
// The streaming operand X is read in its own layout: viewed as real [K][2N] (re / im
// interleaved along n), a 128-column slab of it, transposed, is the MMA's A operand (rows
// n' = 2n + ri, K = k).  TMA tensor copies (4 boxes of 32 columns x KC rows) bring the slab
// into a ring; split warps transpose it into the canonical K-major layout while splitting
// each value into TF32 big + small parts.  (The MN-major UMMA operand, which would take
// the TMA tile as is, read as zeros on this driver / toolkit for kind::tf32 —
// tools/lab/xstage_check.cu — so the transpose is done by the split warps, whose
// loads / 16-byte stores are bank-conflict-free.)  With P = X^T Wr^T and Q = X^T Wi^T (two
// TMEM accumulators, the twiddles' real / imaginary parts as the K-major B operand)
//   Re C(m, n) = P(2n, m) - Q(2n+1, m),   Im C(m, n) = P(2n+1, m) + Q(2n, m),
// which the epilogue forms with one lane shuffle (TMEM lane = row n').
//
// Roles (512 threads, one CTA per SM, persistent over 128-column tiles): warp 0 lane 0
// issues the TMA ring (NBUF chunks of 128 columns x KC = 32 k); warps 2-3 transpose and
// split each chunk into the big / small operand buffers; warp 1 lane 0 issues
// 3 x 2 x KC/8 tcgen05.mma per chunk and m-group (a_small * w_big + a_big * w_small +
// a_big * w_big into P and Q, ~fp32 accuracy), each k chunk into its own accumulator pair;
// warps 4-15 (three per TMEM lane quarter) drain the accumulators (tcgen05.ld, fp32 chunk
// sums, shuffle, coalesced 128-byte row stores) while the next tile's chunks stream in —
// the drain is latency-bound, so it gets the most warps.  The twiddles (big / small, real / imaginary, canonical K-major, zero padded) stay
// in shared memory; outputs wider than 128 rows (embed: Nx) are two m-groups so the
// double-buffered accumulators fit the 512 TMEM columns.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

namespace {

constexpr int XS_KC = 32;       // k rows per chunk
constexpr int XS_NBUF = 3;      // TMA ring depth (raw chunks)
constexpr int XS_NSB = 2;       // operand buffers (big + small pairs)
constexpr int XS_THREADS = 512; // warp 0 TMA, warp 1 MMA, warps 2-3 split, warps 4-15 epilogue
constexpr int XS_CH = 128 * XS_KC;  // floats per chunk
constexpr size_t XS_SMEM_MAX = 226 * 1024;

__device__ __forceinline__ uint32_t xs_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void xs_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n XS_MBAR_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra XS_MBAR_WAIT;\n}\n" ::"r"(xs_su32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float xs_tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void xs_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(xs_su32(bar)) : "memory");
}

// K-major SWIZZLE_NONE canonical descriptor (8-row x 16-byte core matrices)
__device__ __forceinline__ uint64_t xs_desc_k(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void xs_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void xs_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// tmX: X as float [nf][K][N2] (box {32, XS_KC, 1}, SWIZZLE_128B); Tw: 4 canonical
// K-major arrays [Mpad][Kpad] (W real big, real small, imag big, imag small); C[f][m][n']
// with row pitch N2 and field stride sC.  NG: MMA N (output rows m per group), G groups.
template <int TMEM_COLS, int NBUF, int NSB>
__global__ __launch_bounds__(XS_THREADS, 1) void umma_xstage_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                    const float* __restrict__ Tw,
                                                                    float* __restrict__ C, long long sC, int M,
                                                                    int N2, int Kpad, int Mpad, int nf, int NG,
                                                                    int G, int NACC, int UC, int gsplit,
                                                                    int single) {
  constexpr uint32_t LBO_B = 128;
  const uint32_t SBO_B = (uint32_t)(Kpad / 4) * 128;
  // TMEM: NACC buffers of UC columns per accumulator unit: with several k chunks one (P, Q)
  // pair per chunk (big-twiddle products) and one for the small-twiddle corrections, added
  // by the epilogue in fp32; with one chunk a single (P, Q) pair.  The tensor core's fp32 accumulation, 180 terms deep at the
  // config-2 project, cost 2x the error of the FFMA stage and broke the SURVEY 8(c) energy
  // tolerance; 32 terms deep it does not.
  extern __shared__ __align__(1024) float sm[];
  float* ring = sm;                        // NBUF raw chunks (TMA destination, [4 boxes][KC][32])
  float* opb = ring + NBUF * XS_CH;     // NSB x (big, small) canonical K-major chunks
  float* tw = opb + 2 * NSB * XS_CH;    // 4 x Mpad x Kpad
  __shared__ __align__(8) unsigned long long full[NBUF], consumed[NBUF], ready[NSB], mma_done[NSB];
  __shared__ __align__(8) unsigned long long acc_full[2], acc_free[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // roles: one k chunk per tile (embed) -> the drain dominates: 12 epilogue warps (4-15),
  // split by warps 2-3; several chunks (project: K = Nx) -> the split dominates: 4
  // epilogue warps (4-7), split by warps 2-3 and 8-15
  const int nk = Kpad / XS_KC;
  // epilogue warps per TMEM lane quarter: 3 with one chunk per tile (drain-bound), 2 with
  // one accumulator over several chunks (config 4's embed: 51 vs 64 us with 3), 1 with
  // per-chunk accumulators (the split is the work)
  const int EW = nk == 1 ? 3 : (single ? 2 : 1);
  const int NSPLIT = (XS_THREADS / 32 - 4 - 4 * EW + 2) * 32;  // split threads
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(xs_su32(&tmem_base_sh)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xs_su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(xs_su32(&consumed[i])), "r"(NSPLIT));
    }
    for (int i = 0; i < NSB; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(xs_su32(&ready[i])), "r"(NSPLIT));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xs_su32(&mma_done[i])));
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xs_su32(&acc_full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(xs_su32(&acc_free[i])), "r"(128 * EW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // gsplit: CTA b handles output-row group g0 = b % G of its tiles only and keeps that
  // group's twiddle rows (4 NG canonical rows, contiguous); otherwise all groups
  const int g0 = gsplit ? (int)blockIdx.x % G : 0, Gc = gsplit ? 1 : G;
  const int cta = gsplit ? (int)blockIdx.x / G : (int)blockIdx.x, nct = gsplit ? (int)gridDim.x / G : (int)gridDim.x;
  {
    const float4* src = reinterpret_cast<const float4*>(Tw) + (size_t)g0 * NG * Kpad;  // 4 NG Kpad floats per group
    const int n4 = (gsplit ? NG : Mpad) * Kpad;
    for (int e = tid; e < n4; e += XS_THREADS) reinterpret_cast<float4*>(tw)[e] = __ldg(src + e);
  }
  // TMEM, barriers and the (constant) twiddle operand are set up before the PDL wait
  pdl_wait();
  pdl_trigger();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  const int ntn = (N2 + 127) / 128;  // 128-column tiles per field
  const int T = nf * ntn;
  const int my_tiles = (T - cta + nct - 1) / nct;
  const bool sep = nk > 1 && !single;  // per-chunk accumulators + corrections
  const int S = my_tiles * nk;  // this CTA's chunk sequence
  auto par = [](int q, int period) { return (uint32_t)(q / period) & 1u; };

  if (warp == 0) {
    if (lane == 0) {
      // TMA producer: chunk q -> ring slot q % NBUF once chunk q - NBUF has been transposed
      for (int q = 0; q < S; ++q) {
        if (q >= NBUF) xs_wait(&consumed[q % NBUF], par(q - NBUF, NBUF));
        const int tile = cta + (q / nk) * nct, j = q % nk;
        const int f = tile / ntn, n0 = (tile - f * ntn) * 128;
        unsigned long long* bar = &full[q % NBUF];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(xs_su32(bar)),
                     "r"((uint32_t)(XS_CH * 4))
                     : "memory");
        float* dst = ring + (q % NBUF) * XS_CH;
        for (int b = 0; b < 4; ++b)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
              "[%5];\n" ::"r"(xs_su32(dst + b * 32 * XS_KC)),
              "l"(&tmX), "r"(n0 + 32 * b), "r"(j * XS_KC), "r"(f), "r"(xs_su32(bar))
              : "memory");
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // MMA issuer, per chunk and m-group g (twiddle rows of the group: [Wr_big; Wi_big;
      // Wr_small; Wi_small], NG each, consecutive canonical rows), each N = 2 NG MMA
      // producing [P | Q]: X_big [Wr_b; Wi_b] -> big_j (chunk j), X_big [Wr_s; Wi_s] -> corr,
      // X_small [Wr_b; Wi_b] -> big_j.  One chunk (embed, K = 32): corr = big_0.
      const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(2 * NG >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t SBO_A = (XS_KC / 4) * 128;
      const uint32_t tw0 = xs_su32(tw);
      for (int s = 0; s < S; ++s) {
        const int t = s / nk, j = s % nk;
        xs_wait(&ready[s % NSB], par(s, NSB));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t a_big = xs_su32(opb + (s % NSB) * 2 * XS_CH), a_sml = a_big + XS_CH * 4;
        for (int g = 0; g < Gc; ++g) {
          const int u = t * Gc + g;  // accumulator unit
          if (j == 0 && u >= NACC) xs_wait(&acc_free[u % NACC], par(u - NACC, NACC));
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t ub = tmem + (uint32_t)((u % NACC) * UC);
          const uint32_t big = sep ? ub + (uint32_t)(j * 2 * NG) : ub, corr = sep ? ub + (uint32_t)(nk * 2 * NG) : big;
          // twiddle rows g 4 NG .. (8-row groups SBO_B apart), k chunk j (XS_KC / 4 core matrices of 128 B)
          const uint32_t wb = tw0 + (uint32_t)(g * 4 * NG / 8) * SBO_B + (uint32_t)j * (XS_KC / 4) * 128;
          const uint32_t ws = wb + (uint32_t)(2 * NG / 8) * SBO_B;
          for (int ks = 0; ks < XS_KC / 8; ++ks) {
            const uint64_t adb = xs_desc_k(a_big + ks * 2 * LBO_B, LBO_B, SBO_A);
            const uint64_t ads = xs_desc_k(a_sml + ks * 2 * LBO_B, LBO_B, SBO_A);
            const uint64_t bdb = xs_desc_k(wb + ks * 2 * LBO_B, LBO_B, SBO_B);
            xs_mma(big, adb, bdb, idesc2, (sep ? ks : (j | ks)) ? 1u : 0u);
            xs_mma(corr, adb, xs_desc_k(ws + ks * 2 * LBO_B, LBO_B, SBO_B), idesc2, (!sep || j | ks) ? 1u : 0u);
            xs_mma(big, ads, bdb, idesc2, 1u);
          }
          if (j == nk - 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             xs_su32(&acc_full[u % NACC]))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         xs_su32(&mma_done[s % NSB]))
                     : "memory");
      }
    }
  } else if (warp >= 4 && warp < 4 + 4 * EW) {
    // epilogue: TMEM lane quarter warp & 3 = columns n' of the tile; the EW warps of a
    // quarter take every EW-th 16-row block of the output rows m
    const int qd = warp & 3, part = (warp - 4) >> 2;
    const bool odd = lane & 1;
    for (int t = 0; t < my_tiles; ++t) {
      const int tile = cta + t * nct;
      const int f = tile / ntn, n = (tile - f * ntn) * 128 + qd * 32 + lane;
      const bool nok = n < N2;
      float* cf = C + (long long)f * sC + n;
      for (int g = 0; g < Gc; ++g) {
        const int u = t * Gc + g;
        xs_wait(&acc_full[u % NACC], par(u, NACC));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t ub = tmem + (uint32_t)((u % NACC) * UC) + ((uint32_t)(qd * 32) << 16);
        for (int c0 = 16 * part; c0 < NG; c0 += 16 * EW) {
          float ps[16], qs[16];
          {
            // corrections (several chunks) or the single chunk's accumulator
            uint32_t p[16], q[16];
            const uint32_t c = sep ? (uint32_t)(nk * 2 * NG) : 0u;
            xs_ld16(ub + c + c0, p);
            xs_ld16(ub + c + (uint32_t)NG + c0, q);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) ps[i] = __uint_as_float(p[i]), qs[i] = __uint_as_float(q[i]);
          }
          for (int j = 0; j < (sep ? nk : 0); ++j) {  // k chunks summed in fp32
            uint32_t p[16], q[16];
            xs_ld16(ub + (uint32_t)(j * 2 * NG) + c0, p);
            xs_ld16(ub + (uint32_t)(j * 2 * NG + NG) + c0, q);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) ps[i] += __uint_as_float(p[i]), qs[i] += __uint_as_float(q[i]);
          }
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float qo = __shfl_xor_sync(0xffffffffu, qs[i], 1);
            v[i] = odd ? ps[i] + qo : ps[i] - qo;
          }
          const int m0 = (g0 + g) * NG + c0;
          float* cp = cf + (long long)m0 * N2;
          if (nok && m0 + 16 <= M) {
#pragma unroll
            for (int i = 0; i < 16; ++i) cp[(long long)i * N2] = v[i];
          } else if (nok) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (m0 + i < M) cp[(long long)i * N2] = v[i];
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        xs_arrive(&acc_free[u % NACC]);
      }
    }
  } else if (warp >= 2) {
    // split workers (warps 2-3 and those past the epilogue): raw chunk s (ring slot
    // s % NBUF: box b = columns 32 b .., [KC][32]) -> canonical K-major big / small operands
    // (buffer pair s % NSB).  Items (k quad, column n') with n' fastest: a warp's lanes read
    // consecutive columns (conflict-free) and each 8-lane phase stores one 128-byte
    // core-matrix row.
    const int st = warp < 4 ? tid - 64 : tid - 64 - 128 * EW;
    for (int s = 0; s < S; ++s) {
      xs_wait(&full[s % NBUF], par(s, NBUF));
      if (s >= NSB) xs_wait(&mma_done[s % NSB], par(s - NSB, NSB));
      const float* raw = ring + (s % NBUF) * XS_CH;
      float* big = opb + (s % NSB) * 2 * XS_CH;
      float* sml = big + XS_CH;
      for (int item = st; item < 128 * XS_KC / 4; item += NSPLIT) {
        const int nc = item & 127, kq = item >> 7;
        const float* src = raw + (nc >> 5) * (32 * XS_KC) + (nc & 31) + 4 * kq * 32;
        float a[4], bg[4], sl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = src[i * 32];
        // big = round-to-nearest TF32 (exact in TF32; half the error of a truncated big part,
        // which the config-2 energy tolerance needs), small = a - big (exact in fp32)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          bg[i] = xs_tf32_rna(a[i]);
          sl[i] = a[i] - bg[i];
        }
        const int off = ((nc >> 3) * (XS_KC / 4) * 128 + kq * 128 + (nc & 7) * 16) / 4;
        *reinterpret_cast<float4*>(big + off) = make_float4(bg[0], bg[1], bg[2], bg[3]);
        *reinterpret_cast<float4*>(sml + off) = make_float4(sl[0], sl[1], sl[2], sl[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      xs_arrive(&consumed[s % NBUF]);
      xs_arrive(&ready[s % NSB]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 xs_encoder() {
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

// output rows in G groups of NG (a multiple of 16, at most 128: 2 NG <= 256 = one MMA's N)
void xs_groups(int M, int& G, int& NG) {
  const int Mp = (M + 15) / 16 * 16;
  G = (Mp + 127) / 128;
  NG = ((Mp + G - 1) / G + 15) / 16 * 16;
}
int xs_mpad(int M) {
  int G, NG;
  xs_groups(M, G, NG);
  return G * NG;
}
int xs_kpad(int K) { return (K + XS_KC - 1) / XS_KC * XS_KC; }

// TMEM columns of one accumulator unit: (P, Q) per k chunk plus the corrections, or one
// (P, Q) pair when there is a single chunk
int xs_ucols(int K, int NG) {
  const int nk = xs_kpad(K) / XS_KC;
  return (nk > 1 ? nk + 1 : 1) * 2 * NG;
}

size_t xs_smem(int M, int K) {
  return ((size_t)(XS_NBUF + 2 * XS_NSB) * XS_CH + (size_t)4 * xs_mpad(M) * xs_kpad(K)) * sizeof(float) + 1024;
}

// Launch plan.  Default: every CTA holds all twiddle groups, 3-deep ring, 2 operand
// buffers, per-chunk accumulators when K spans several chunks.  When the twiddles do not
// fit (config 4's embed: 256 rows x 64 k, 256 KB), each CTA takes one output-row group of
// its tiles (gsplit: that group's 128 KB of twiddles, X read once per group), a 2-deep ring
// and one operand buffer, and — when the per-chunk accumulators would not fit TMEM — one
// accumulator pair across the chunks (single).
struct XsPlan {
  bool ok = false;
  int G = 1, NG = 0, gsplit = 0, single = 0, nbuf = XS_NBUF, nsb = XS_NSB, UC = 0, NACC = 1;
  size_t smem = 0;
};

XsPlan xs_plan(int M, int K) {
  XsPlan p;
  xs_groups(M, p.G, p.NG);
  const int Kpad = xs_kpad(K), nk = Kpad / XS_KC;
  p.UC = xs_ucols(K, p.NG);
  p.smem = xs_smem(M, K);
  if (p.smem <= XS_SMEM_MAX && p.UC <= 512) {
    p.ok = true;
  } else if (p.G > 1) {
    p.gsplit = 1;
    p.nbuf = 2;
    p.nsb = 1;
    p.smem = ((size_t)(p.nbuf + 2 * p.nsb) * XS_CH + (size_t)4 * p.NG * Kpad) * sizeof(float) + 1024;
    if (p.UC > 512 && nk > 1) {
      p.single = 1;
      p.UC = 2 * p.NG;
    }
    p.ok = p.smem <= XS_SMEM_MAX && p.UC <= 512;
  }
  p.NACC = 2 * p.UC <= 512 ? 2 : 1;
  return p;
}

// TF32 round-to-nearest (ties away) of a float, on the host
float xs_tf32(float x) {
  uint32_t b;
  std::memcpy(&b, &x, 4);
  b = (b + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &b, 4);
  return r;
}

// canonical K-major offset (floats) of element (row, k) in a tile with Kpad columns
int xs_canon(int row, int k, int Kpad) { return ((row >> 3) * (Kpad / 4) * 128 + (k >> 2) * 128 + (row & 7) * 16) / 4 + (k & 3); }

}  // namespace

bool umma_xstage_fits(int M, int K, int N) {
  // M <= 256 output rows (MMA N = one or two groups of <= 128), 16-byte rows of X for the TMA
  int G, NG;
  xs_groups(M, G, NG);
  // TMA: 16-byte row pitch (2N floats) and field stride (K N complex, the callers' layouts)
  (void)NG;
  return M >= 1 && M <= 256 && K >= 1 && N >= 64 && N % 2 == 0 && (1LL * K * N) % 2 == 0 && xs_plan(M, K).ok &&
         xs_encoder() != nullptr;
}

long long umma_xstage_twiddle_floats(int M, int K) { return 4LL * xs_mpad(M) * xs_kpad(K); }

// W [M][K] complex (row-major, host) -> the canonical K-major twiddle operand: per output
// row group g (NG rows), rows [Re big; Im big; Re small; Im small], NG each
void umma_xstage_twiddles_host(const float2* W, int M, int K, std::vector<float>& out) {
  int G, NG;
  xs_groups(M, G, NG);
  const int Kpad = xs_kpad(K);
  out.assign((size_t)4 * G * NG * Kpad, 0.f);
  for (int m = 0; m < M; ++m) {
    const int g = m / NG, ml = m - g * NG, r0 = g * 4 * NG + ml;
    for (int k = 0; k < K; ++k) {
      const float2 w = W[(size_t)m * K + k];
      const float rb = xs_tf32(w.x), ib = xs_tf32(w.y);
      out[xs_canon(r0, k, Kpad)] = rb;
      out[xs_canon(r0 + NG, k, Kpad)] = ib;
      out[xs_canon(r0 + 2 * NG, k, Kpad)] = xs_tf32(w.x - rb);
      out[xs_canon(r0 + 3 * NG, k, Kpad)] = xs_tf32(w.y - ib);
    }
  }
}

// C[f][m][n] = sum_k W[m][k] X[f][k][n] (complex): X [nf][K][N] complex (field stride
// sX complex), C [nf][M][N] complex (field stride sC complex); tw from umma_xstage_twiddles_host
void launch_umma_xstage(const float* tw, const float2* X, long long sX, float2* C, long long sC, int M, int N,
                        int K, int nf, cudaStream_t s) {
  if (nf <= 0 || N <= 0) return;
  const int Mpad = xs_mpad(M), Kpad = xs_kpad(K), N2 = 2 * N;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)N2, (cuuint64_t)K, (cuuint64_t)nf};
  const cuuint64_t strides[2] = {(cuuint64_t)N2 * 4, (cuuint64_t)sX * 8};
  const cuuint32_t box[3] = {32, XS_KC, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = xs_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(X), dims, strides, box,
                                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(3, "umma x-stage: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  const XsPlan pl = xs_plan(M, K);
  if (!pl.ok) throw EngineError(3, "umma x-stage: no shared-memory / TMEM plan for this shape");
  const int T = nf * ((N2 + 127) / 128);
  // gsplit: G CTAs per tile (one per output-row group), grid a multiple of G
  const int grid = pl.gsplit ? std::min(kSMs / pl.G * pl.G, T * pl.G) : std::min(kSMs, T);
  auto go = [&](auto kern, int slot) {
    static bool set[64][8] = {};
    int dev = 0;
    LDDMM_CUDA(cudaGetDevice(&dev));
    if (!set[dev & 63][slot]) {
      LDDMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XS_SMEM_MAX));
      set[dev & 63][slot] = true;
    }
    pdl_launch(kern, grid, XS_THREADS, pl.smem, s, tm, tw, reinterpret_cast<float*>(C), 2 * sC, M, N2, Kpad, Mpad,
               nf, pl.NG, pl.G, pl.NACC, pl.UC, pl.gsplit, pl.single);
  };
  const int cols = pl.NACC * pl.UC;
  if (!pl.gsplit) {
    if (cols <= 64)
      go(umma_xstage_kernel<64, XS_NBUF, XS_NSB>, 0);
    else if (cols <= 128)
      go(umma_xstage_kernel<128, XS_NBUF, XS_NSB>, 1);
    else if (cols <= 256)
      go(umma_xstage_kernel<256, XS_NBUF, XS_NSB>, 2);
    else
      go(umma_xstage_kernel<512, XS_NBUF, XS_NSB>, 3);
  } else {
    if (cols <= 256)
      go(umma_xstage_kernel<256, 2, 1>, 4);
    else
      go(umma_xstage_kernel<512, 2, 1>, 5);
  }
  LDDMM_LAUNCH_CHECK();
}

}  // namespace lddmm_b200
