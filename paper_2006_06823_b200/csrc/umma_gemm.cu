// tcgen05 (5th-generation tensor core) 3xTF32 GEMMs for the z stages of the
// truncated DFT, accumulators in tensor memory (TMEM).
//
// embed-z:  C[b][m][n] = sum_k A[b][m][k] * B[k][n],  A = E2 viewed as float
//           [Nx*Ny][2H] (K = 2H), B = Tz_e [2H][Nz], C = the grid field [Nx*Ny][Nz].
//
// Persistent kernel, one CTA per SM: the CTA keeps B (TF32 big + small parts, in
// the canonical K-major no-swizzle UMMA layout: 8-row x 16-byte core matrices) in
// shared memory and one 128 x N fp32 accumulator in TMEM, and walks 128-row tiles:
//   1. the tile's A rows (loaded into registers during the previous tile) are
//      split into TF32 big + small and stored in the canonical layout;
//   2. one thread issues 3 x K/8 tcgen05.mma (a_small*b_big + a_big*b_small +
//      a_big*b_big, ~fp32 accuracy) and commits them to an mbarrier;
//   3. the next tile's A rows are loaded while the MMAs run;
//   4. the accumulator is read with tcgen05.ld into two 64-row shared stages that
//      are the tile's contiguous image in C, each written by one 1-D bulk copy
//      (cp.async.bulk, TMA engine) that overlaps the following tile.
// The output write (4 N bytes per row) dominates the traffic; the kernel runs at
// ~70% of the measured HBM bandwidth where the mma.sync version ran at ~37%.
//
// project-z (umma_zproject_kernel, below): the grid is the streaming operand, brought
// in by TMA tensor copies (SWIZZLE_128B) through a ring, with warp-specialised split /
// MMA / epilogue roles handing off through mbarriers.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t tf32_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE (canonical ((8,m),(T,2)) layout:
// LBO = byte stride between the two 16-byte K chunks of an MMA step, SBO = byte stride
// between 8-row groups), sm_100 version bit.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// K-major SWIZZLE_128B descriptor (8-row x 128-byte atoms, 1024-byte aligned; the
// start address moves by 32 bytes per 8-element TF32 K step inside the atom row)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n UMMA_MBAR_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra UMMA_MBAR_WAIT;\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}

// canonical K-major offset (floats) of element (row, k) in a tile with K columns
__host__ __device__ __forceinline__ int canon_off(int row, int k, int K) {
  return ((row >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (row & 7) * 16) / 4 + (k & 3);
}

}  // namespace

constexpr int UZ_THREADS = 256;

// nsplit > 1 (large Nz, e.g. config 4's 256 x K = 64, whose whole-row plan needs 320 KB):
// each CTA owns the output columns [h NS, (h+1) NS), h = blockIdx.x % nsplit, NS = N /
// nsplit (gridDim.x a multiple of nsplit, so h is fixed per CTA); its B slice is the
// contiguous canonical rows h NS ..; the 64-row stages (64 x NS) are written with a 3-D
// TMA tensor store (tmC: [nb][M][N], box {NS, 64, 1}) instead of one 1-D bulk copy.
template <int TMEM_COLS>
__global__ __launch_bounds__(UZ_THREADS, 1) void umma_zembed_kernel(const float* __restrict__ A, long long sA,
                                                                    const float* __restrict__ Bbig_c,
                                                                    const float* __restrict__ Bsm_c,
                                                                    float* __restrict__ C, long long sC, int M,
                                                                    int N, int NP, int K, int nb, int nsplit,
                                                                    const __grid_constant__ CUtensorMap tmC) {
  const int KC = K / 4;
  const uint32_t LBO = 128, SBO = (uint32_t)KC * 128;
  const int half = (int)blockIdx.x % nsplit;
  const int NS = nsplit > 1 ? N / nsplit : N;   // output columns of this CTA (stage row pitch)
  const int NPS = nsplit > 1 ? NS : NP;          // MMA N (padded)
  extern __shared__ __align__(1024) float sm[];
  float* Bb = sm;
  float* Bs = Bb + NPS * K;
  float* Ab = Bs + NPS * K;
  float* As = Ab + 128 * K;
  float* stage0 = As + 128 * K;  // two 64-row halves, each the half tile's image in C
  float* stage1 = stage0 + 64 * NS;
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    // canonical K-major rows n0 .. n0 + NPS - 1 are contiguous (n0 a multiple of 8)
    const float4* bg = reinterpret_cast<const float4*>(Bbig_c + (size_t)half * NPS * K);
    const float4* bs = reinterpret_cast<const float4*>(Bsm_c + (size_t)half * NPS * K);
    for (int e = tid; e < NPS * K / 4; e += UZ_THREADS) {
      reinterpret_cast<float4*>(Bb)[e] = __ldg(bg + e);
      reinterpret_cast<float4*>(Bs)[e] = __ldg(bs + e);
    }
  }
  // TMEM, barriers and the (constant) twiddle operand are set up before the PDL wait
  pdl_wait();
  pdl_trigger();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  const int mtiles = (M + 127) / 128;
  const int ntiles = mtiles * nb * nsplit;  // work items: (tile, column slice)
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NPS >> 3) << 17) | ((128u >> 4) << 24);
  constexpr int MAXPER = 128 * 16 / UZ_THREADS;  // K <= 64
  const int per = 128 * KC / UZ_THREADS;
  float4 v[MAXPER];
  auto load_tile = [&](int item) {
    const int tile = item / nsplit;
    const int b = tile / mtiles, m0 = (tile - b * mtiles) * 128;
    const float* Ag = A + b * sA;
#pragma unroll
    for (int q = 0; q < MAXPER; ++q) {
      if (q >= per) break;
      const int e = tid + q * UZ_THREADS;
      const int r = e & 127, kc = e >> 7;
      const int gm = m0 + r;
      v[q] = (item < ntiles && gm < M) ? __ldg(reinterpret_cast<const float4*>(Ag + (long long)gm * K) + kc)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  uint32_t phase = 0;
  load_tile(blockIdx.x);
  for (int item = blockIdx.x; item < ntiles; item += gridDim.x) {
    const int tile = item / nsplit;
    const int b = tile / mtiles, m0 = (tile - b * mtiles) * 128;
#pragma unroll
    for (int q = 0; q < MAXPER; ++q) {
      if (q >= per) break;
      const int e = tid + q * UZ_THREADS;
      const int r = e & 127, kc = e >> 7;
      float4 bg, sl;
      bg.x = __uint_as_float(tf32_bits(v[q].x));
      bg.y = __uint_as_float(tf32_bits(v[q].y));
      bg.z = __uint_as_float(tf32_bits(v[q].z));
      bg.w = __uint_as_float(tf32_bits(v[q].w));
      sl.x = __uint_as_float(tf32_bits(v[q].x - bg.x));
      sl.y = __uint_as_float(tf32_bits(v[q].y - bg.y));
      sl.z = __uint_as_float(tf32_bits(v[q].z - bg.z));
      sl.w = __uint_as_float(tf32_bits(v[q].w - bg.w));
      const int off = ((r >> 3) * (int)SBO + kc * (int)LBO + (r & 7) * 16) / 4;
      *reinterpret_cast<float4*>(Ab + off) = bg;
      *reinterpret_cast<float4*>(As + off) = sl;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid == 0) {
      const float* aops[3] = {As, Ab, Ab};
      const float* bops[3] = {Bb, Bs, Bb};
      for (int pass = 0; pass < 3; ++pass)
        for (int ks = 0; ks < K / 8; ++ks)
          umma_tf32(tmem, umma_desc(su32(aops[pass]) + ks * 2 * LBO, LBO, SBO),
                    umma_desc(su32(bops[pass]) + ks * 2 * LBO, LBO, SBO), idesc, (pass | ks) ? 1u : 0u);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       su32(&mbar))
                   : "memory");
    }
    load_tile(item + gridDim.x);  // next operand rows in flight under the MMAs and the epilogue
    mbar_wait(&mbar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    for (int h = 0; h < 2; ++h) {
      float* stage = h ? stage1 : stage0;
      // the bulk copy issued from this buffer one tile ago must have finished reading it
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      __syncthreads();
      const int q = warp & 3;
      if ((q >> 1) == h) {
        const int part = warp >> 2;  // two warps per lane quarter split the column chunks
        const int lr = (q & 1) * 32 + lane;
        const int chunks = NPS / 32 + ((NPS & 31) ? 1 : 0);
        for (int ci = part; ci < chunks; ci += UZ_THREADS / 128) {
          const int c0 = ci * 32;
          uint32_t r[32];
          const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + c0;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          float* srow = stage + lr * NS + c0;
          if ((NS & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              if (c0 + j < NS)
                *reinterpret_cast<float4*>(srow + j) =
                    make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                __uint_as_float(r[j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < NS) srow[j] = __uint_as_float(r[j]);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        const int r0 = m0 + 64 * h;
        const int nrows = min(64, M - r0);
        if (nrows > 0 && nsplit == 1) {
          float* dst = C + b * sC + (long long)r0 * N;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
                       "r"(su32(stage)), "r"((uint32_t)(nrows * N * 4))
                       : "memory");
        } else if (nrows > 0) {
          // rows beyond M are clipped by the TMA unit
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                           &tmC),
                       "r"(half * NS), "r"(r0), "r"(b), "r"(su32(stage))
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}

// project-z:  C[m][n] = sum_k A[m][k] * B[k][n],  A = nf grid fields viewed as one
// float [nf*Nx*Ny][Nz] (K = Nz; fields are contiguous), B = Tz_p [Nz][2H] (N = 2H),
// C = G1 [nf*Nx*Ny][2H].
//
// The streaming operand is A (the grid).  One TMA tensor copy per 128-row x ZP_KC
// (= 128-byte) chunk brings it from HBM straight into the K-major SWIZZLE_128B layout
// the UMMA descriptor reads (8-row x 128-byte atoms); the K tail and the last
// tile's missing rows are zero-filled by the TMA unit.  A ZP_NBUF-deep
// ring keeps ZP_NBUF - 1 chunks in flight while the current one is split in place
// into TF32 big (mantissa-masked, exact in TF32) + small (a - big, exact in fp32) and
// fed to 3 x ZP_KC/8 tcgen05.mma.  B (big + small, canonical, K zero-padded to whole
// chunks) stays in shared memory.  Two TMEM accumulators alternate between 128-row
// tiles; a tile's epilogue (tcgen05.ld, 16-byte stores of its rows) runs while the
// next tile's chunks stream in.
constexpr int ZP_KC = 32;
constexpr int ZP_NBUF = 6;  // TMA ring depth (whole-band plans; 3 when B is large, e.g. config 4)

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

constexpr int ZP_THREADS = 512;  // warp 0 TMA, warp 1 MMA, warps 4-7 epilogue, warps 8-15 split
constexpr int ZP_NS = 4;         // small-part buffers (2 with the shallow ring)

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}

template <int NT, int NBUF, int NSB>
__global__ __launch_bounds__(ZP_THREADS, 1) void umma_zproject_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                      const float* __restrict__ Bbig_c,
                                                                      const float* __restrict__ Bsm_c,
                                                                      float* __restrict__ C, int M, int Kpad) {
  constexpr int CH = 128 * ZP_KC;  // floats per chunk buffer
  constexpr uint32_t LBO_B = 128;
  constexpr int TMEM_COLS = 2 * NT < 32 ? 32 : 2 * NT;
  const uint32_t SBO_B = (uint32_t)(Kpad / 4) * 128;
  extern __shared__ __align__(1024) float sm[];
  float* ring = sm;                     // NBUF chunks: TMA destination, split in place to big
  float* smallb = ring + NBUF * CH;  // NSB small chunks
  float* Bb = smallb + NSB * CH;
  float* Bs = Bb + NT * Kpad;
  __shared__ __align__(8) unsigned long long full[NBUF], split_done[NBUF], mma_done[NBUF];
  __shared__ __align__(8) unsigned long long acc_full[2], acc_free[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base_sh)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 256;\n" ::"r"(su32(&split_done[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&mma_done[i])));
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&acc_full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;\n" ::"r"(su32(&acc_free[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int e = tid; e < NT * Kpad / 4; e += ZP_THREADS) {
    reinterpret_cast<float4*>(Bb)[e] = __ldg(reinterpret_cast<const float4*>(Bbig_c) + e);
    reinterpret_cast<float4*>(Bs)[e] = __ldg(reinterpret_cast<const float4*>(Bsm_c) + e);
  }
  // TMEM, barriers and the (constant) twiddle operand are set up before the PDL wait
  pdl_wait();
  pdl_trigger();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  const int mtiles = (M + 127) / 128;
  const int nk = Kpad / ZP_KC;
  const int my_tiles = (mtiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int S = my_tiles * nk;  // this CTA's chunk sequence
  auto par = [](int q, int period) { return (uint32_t)(q / period) & 1u; };

  if (warp == 0) {
    if (lane == 0) {
      // TMA producer: chunk q -> ring slot q % NBUF once chunk q - NBUF's MMAs are done
      for (int q = 0; q < S; ++q) {
        if (q >= NBUF) mbar_wait(&mma_done[q % NBUF], par(q - NBUF, NBUF));
        const int tile = (int)blockIdx.x + (q / nk) * (int)gridDim.x, j = q % nk;
        unsigned long long* bar = &full[q % NBUF];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)),
                     "r"((uint32_t)(CH * 4))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];\n" ::"r"(su32(ring + (q % NBUF) * CH)),
            "l"(&tmA), "r"(j * ZP_KC), "r"(tile * 128), "r"(su32(bar))
            : "memory");
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // MMA issuer
      const uint32_t idesc1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(2 * NT >> 3) << 17) | ((128u >> 4) << 24);
      for (int s = 0; s < S; ++s) {
        const int t = s / nk, j = s % nk;
        if (j == 0 && t >= 2) mbar_wait(&acc_free[t & 1], par(t - 2, 2));
        mbar_wait(&split_done[s % NBUF], par(s, NBUF));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)((t & 1) * 2 * NT);
        const uint32_t a_big = su32(ring + (s % NBUF) * CH), a_sml = su32(smallb + (s % NSB) * CH);
        const uint32_t b_off = (uint32_t)j * (ZP_KC / 4) * 128;
        const uint32_t b_big = su32(Bb) + b_off;  // B_small follows as canonical rows NT .. 2 NT - 1
        for (int ks = 0; ks < ZP_KC / 8; ++ks) {
          const uint64_t bd = umma_desc(b_big + ks * 2 * LBO_B, LBO_B, SBO_B);
#ifndef ZP_NOMMA  // lab: the pipeline without the MMAs (tools/lab/build_variant.sh)
          umma_tf32(acc, umma_desc_sw128(a_big + ks * 32), bd, idesc2, (j | ks) ? 1u : 0u);  // [Ab Bb | Ab Bs]
          umma_tf32(acc, umma_desc_sw128(a_sml + ks * 32), bd, idesc1, 1u);                 // += As Bb
#endif
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(&mma_done[s % NBUF]))
                     : "memory");
        if (j == nk - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           su32(&acc_full[t & 1]))
                       : "memory");
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // epilogue: TMEM lane quarter warp & 3 -> C rows
    const int qd = warp & 3;
    for (int t = 0; t < my_tiles; ++t) {
      mbar_wait(&acc_full[t & 1], par(t, 2));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t acc = tmem + (uint32_t)((t & 1) * 2 * NT);
      const int m = ((int)blockIdx.x + t * (int)gridDim.x) * 128 + qd * 32 + lane;
      float* crow = C + (long long)m * NT;
#pragma unroll
      for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t r[16], r2[16];
        tmem_ld16(acc + ((uint32_t)(qd * 32) << 16) + c0, r);
        tmem_ld16(acc + ((uint32_t)(qd * 32) << 16) + NT + c0, r2);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (m < M) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(crow + c0 + i) =
                make_float4(__uint_as_float(r[i]) + __uint_as_float(r2[i]),
                            __uint_as_float(r[i + 1]) + __uint_as_float(r2[i + 1]),
                            __uint_as_float(r[i + 2]) + __uint_as_float(r2[i + 2]),
                            __uint_as_float(r[i + 3]) + __uint_as_float(r2[i + 3]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      mbar_arrive(&acc_free[t & 1]);
    }
  } else if (warp >= 8) {
    // split workers: chunk s in place -> TF32 big; small -> small buffer s % NSB
    const int st = tid - 256;
    for (int s = 0; s < S; ++s) {
      mbar_wait(&full[s % NBUF], par(s, NBUF));
      if (s >= NSB) mbar_wait(&mma_done[(s - NSB) % NBUF], par(s - NSB, NBUF));
      float* big = ring + (s % NBUF) * CH;
      float* sml = smallb + (s % NSB) * CH;
#pragma unroll
      for (int u = 0; u < CH / 4 / 256; ++u) {
        const int e = st + u * 256;
        const float4 a = reinterpret_cast<const float4*>(big)[e];
        // TF32 parts: big = round-to-nearest TF32 (exact in TF32), small = a - big (exact in
        // fp32; the tensor core reads its leading 19 bits)
        float4 bg;
        bg.x = __uint_as_float(tf32_bits(a.x));
        bg.y = __uint_as_float(tf32_bits(a.y));
        bg.z = __uint_as_float(tf32_bits(a.z));
        bg.w = __uint_as_float(tf32_bits(a.w));
        reinterpret_cast<float4*>(big)[e] = bg;
        reinterpret_cast<float4*>(sml)[e] = make_float4(a.x - bg.x, a.y - bg.y, a.z - bg.z, a.w - bg.w);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive(&split_done[s % NBUF]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// Tz_p big/small [K][N] row-major -> canonical K-major [N][Kpad], rows k >= K zero
__global__ void umma_zproj_prep_kernel(const float* __restrict__ Bbig, const float* __restrict__ Bsm, int K, int N,
                                       int Kpad, float* __restrict__ Cbig, float* __restrict__ Csm) {
  pdl_prologue();
  const long long total = (long long)N * Kpad;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(e / Kpad), k = (int)(e - (long long)n * Kpad);
    const bool in = k < K;
    Cbig[canon_off(n, k, Kpad)] = in ? Bbig[(long long)k * N + n] : 0.f;
    Csm[canon_off(n, k, Kpad)] = in ? Bsm[(long long)k * N + n] : 0.f;
  }
}

int umma_zproject_kpad(int K) { return (K + ZP_KC - 1) / ZP_KC * ZP_KC; }

static size_t umma_zproject_smem_ring(int N, int K, int nbuf, int ns) {
  return ((size_t)2 * N * umma_zproject_kpad(K) + (size_t)(nbuf + ns) * 128 * ZP_KC) * sizeof(float);
}

// deep ring (6 TMA slots + 4 small buffers) when it fits, else the shallow one (3 + 2)
static bool umma_zproject_deep(int N, int K) { return umma_zproject_smem_ring(N, K, ZP_NBUF, ZP_NS) <= 226 * 1024; }

static size_t umma_zproject_smem(int N, int K) {
  return umma_zproject_deep(N, K) ? umma_zproject_smem_ring(N, K, ZP_NBUF, ZP_NS) : umma_zproject_smem_ring(N, K, 3, 2);
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

bool umma_zproject_fits(int K, int N) {
  // K = Nz (rows 16-byte aligned, whole 16-byte chunks), N = 2H in {32, 64}
  return K % 4 == 0 && (N == 32 || N == 64) && umma_zproject_smem(N, K) <= 226 * 1024 &&
         tensor_map_encoder() != nullptr;
}

void launch_umma_zproj_prep(const float* Bbig, const float* Bsm, int K, int N, float* Cbig, float* Csm,
                            cudaStream_t s) {
  const int Kpad = umma_zproject_kpad(K);
  pdl_launch(umma_zproj_prep_kernel, grid_for((long long)N * Kpad, 256), 256, 0, s, Bbig, Bsm, K, N, Kpad, Cbig, Csm);
  LDDMM_LAUNCH_CHECK();
}

// A: M rows of K floats (contiguous), C: M rows of N floats (contiguous)
void launch_umma_zproject(const float* A, const float* Bbig_c, const float* Bsm_c, float* C, int M, int K, int N,
                          cudaStream_t s) {
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  const cuuint32_t box[2] = {ZP_KC, 128};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(3, "umma z-project: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  const size_t smem = umma_zproject_smem(N, K);
  const int mtiles = (M + 127) / 128;
  const int grid = std::min(kSMs, mtiles);
  auto go = [&](auto kern, int slot) {
    static bool set[64][4] = {};
    int dev = 0;
    LDDMM_CUDA(cudaGetDevice(&dev));
    if (!set[dev & 63][slot]) {
      LDDMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
      set[dev & 63][slot] = true;
    }
    pdl_launch(kern, grid, ZP_THREADS, smem, s, tm, Bbig_c, Bsm_c, C, M, umma_zproject_kpad(K));
  };
  const bool deep = umma_zproject_deep(N, K);
  if (N == 32)
    deep ? go(umma_zproject_kernel<32, ZP_NBUF, ZP_NS>, 0) : go(umma_zproject_kernel<32, 3, 2>, 2);
  else
    deep ? go(umma_zproject_kernel<64, ZP_NBUF, ZP_NS>, 1) : go(umma_zproject_kernel<64, 3, 2>, 3);
  LDDMM_LAUNCH_CHECK();
}

// B [K][N] (big / small TF32 parts, row-major) -> canonical K-major [NP][K], zero padded
__global__ void umma_canon_b_kernel(const float* __restrict__ Bbig, const float* __restrict__ Bsm, int K, int N,
                                    int NP, float* __restrict__ Cbig, float* __restrict__ Csm) {
  pdl_prologue();
  const long long total = (long long)NP * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(e / K), k = (int)(e - (long long)n * K);
    const bool in = n < N;
    Cbig[canon_off(n, k, K)] = in ? Bbig[(long long)k * N + n] : 0.f;
    Csm[canon_off(n, k, K)] = in ? Bsm[(long long)k * N + n] : 0.f;
  }
}

int umma_padded_n(int N) { return (N + 15) & ~15; }

static size_t umma_zembed_smem_split(int N, int K, int nsplit) {
  const int NPS = nsplit > 1 ? N / nsplit : umma_padded_n(N);
  const int NS = nsplit > 1 ? N / nsplit : N;
  return ((size_t)2 * NPS * K + (size_t)2 * 128 * K + (size_t)128 * NS) * sizeof(float);
}

// column slices per CTA: 1 (whole rows, 1-D bulk stores) when that plan fits, else 2 or 4
// (each slice a multiple of 16 columns, TMA tensor stores)
static int umma_zembed_nsplit(int N, int K) {
  for (int ns : {1, 2, 4}) {
    if (ns > 1 && (N % (16 * ns) != 0)) continue;
    if (umma_zembed_smem_split(N, K, ns) <= 226 * 1024) return ns;
  }
  return 0;
}

size_t umma_zembed_smem(int N, int K) { return umma_zembed_smem_split(N, K, std::max(1, umma_zembed_nsplit(N, K))); }

bool umma_zembed_fits(int N, int K) {
  // UMMA M = 128 needs N % 16 == 0 (padded), N <= 256; K a multiple of 8 and <= 64; the
  // staged tile and operands must fit the 227 KB shared-memory budget (column slices
  // when whole rows do not); rows 16-byte aligned
  return N >= 16 && umma_padded_n(N) <= 256 && K % 8 == 0 && K <= 64 && (K % 4) == 0 && (N % 4) == 0 &&
         umma_zembed_nsplit(N, K) > 0 && tensor_map_encoder() != nullptr;
}

void launch_umma_canon_b(const float* Bbig, const float* Bsm, int K, int N, float* Cbig, float* Csm,
                         cudaStream_t s) {
  const int NP = umma_padded_n(N);
  pdl_launch(umma_canon_b_kernel, grid_for((long long)NP * K, 256), 256, 0, s, Bbig, Bsm, K, N, NP, Cbig, Csm);
  LDDMM_LAUNCH_CHECK();
}

void launch_umma_zembed(const float* A, long long sA, const float* Bbig_c, const float* Bsm_c, float* C,
                        long long sC, int M, int N, int K, int nb, cudaStream_t s) {
  const int NP = umma_padded_n(N);
  const int nsplit = umma_zembed_nsplit(N, K);
  if (nsplit < 1) throw EngineError(3, "umma z-embed: no shared-memory plan for N = " + std::to_string(N));
  const size_t smem = umma_zembed_smem_split(N, K, nsplit);
  const int mtiles = (M + 127) / 128;
  // a multiple of nsplit, so every CTA keeps one column slice
  const int grid = std::min(kSMs / nsplit * nsplit, mtiles * nb * nsplit);
  CUtensorMap tmC;
  std::memset(&tmC, 0, sizeof(tmC));
  if (nsplit > 1) {
    const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)nb};
    const cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)sC * 4};
    const cuuint32_t box[3] = {(cuuint32_t)(N / nsplit), 64, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = tensor_map_encoder()(&tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, C, dims, strides, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      throw EngineError(3, "umma z-embed: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  }
  auto go = [&](auto kern, int slot) {  // one attribute flag per instantiation (same pointer type)
    static bool set[64][4] = {};
    int dev = 0;
    LDDMM_CUDA(cudaGetDevice(&dev));
    if (!set[dev & 63][slot]) {
      LDDMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
      set[dev & 63][slot] = true;
    }
    pdl_launch(kern, grid, UZ_THREADS, smem, s, A, sA, Bbig_c, Bsm_c, C, sC, M, N, NP, K, nb, nsplit, tmC);
  };
  const int NPS = nsplit > 1 ? N / nsplit : NP;
  if (NPS <= 32)
    go(umma_zembed_kernel<32>, 0);
  else if (NPS <= 64)
    go(umma_zembed_kernel<64>, 1);
  else if (NPS <= 128)
    go(umma_zembed_kernel<128>, 2);
  else
    go(umma_zembed_kernel<256>, 3);
  LDDMM_LAUNCH_CHECK();
}

}  // namespace lddmm_b200
