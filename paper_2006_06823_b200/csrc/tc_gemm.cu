// Tensor-core (3xTF32) real GEMMs for the z stages of the truncated DFT.
//
//   C[b][m][n] = sum_k A[b][m][k] * B[k][n]      (fp32 in, fp32 out)
//
// embed-z:   A = E2 viewed as float [Nx*Ny][2H], B = Tz_e [2H][Nz]  (K = 2H)
// project-z: A = grid field [Nx*Ny][Nz],        B = Tz_p [Nz][2H]  (K = Nz)
//
// Each product is evaluated as a_big*b_big + a_big*b_small + a_small*b_big with
// a = a_big + a_small split into two TF32 numbers (cvt.rna), accumulated in fp32
// on the tensor cores (mma.sync m16n8k8 .tf32): ~fp32 accuracy (dropped term
// a_small*b_small ~ 2^-22 relative).  B (the twiddle table) is split once on
// the host side of the call; A is split in registers.  The kernels are
// HBM-bound at the z-stage shapes (K = 32 / N = 32), so the simpler warp-level
// MMA suffices; the FFMA version (sgemm_kernel) remains for reference.
#include "common.cuh"
#include "kernels.cuh"

namespace lddmm_b200 {

__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int TC_BK = 32;

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_tc() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_tc() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// CTA: 256 threads = 8 warps.  BN = 64: warps 4 (m) x 2 (n), warp tile 32 x 32.
//                               BN = 32: warps 8 (m) x 1 (n), warp tile 16 x 32.
// A k-chunks (128 x 32) are double-buffered with 16-byte cp.async when the rows are
// 16-byte aligned (lda % 4 == 0), so the next chunk streams in under the MMAs.
template <int BN>
__global__ __launch_bounds__(256) void tc3_gemm_kernel(const float* __restrict__ A, int lda, long long sA,
                                                       const float* __restrict__ Bbig,
                                                       const float* __restrict__ Bsmall, int ldb,
                                                       float* __restrict__ C, int ldc, long long sC, int M, int N,
                                                       int K) {
  pdl_prologue();
  constexpr int BM = 128;
  constexpr int WN = BN == 64 ? 2 : 1;  // warps along n
  constexpr int WMW = 8 / WN;           // warps along m
  constexpr int WM = BM / WMW;          // warp tile rows: 32 or 16
  constexpr int MT = WM / 16;           // m16 tiles per warp
  constexpr int AS = TC_BK + 4;         // smem strides (bank-conflict free fragments, 16-B rows)
  constexpr int BS = BN + 8;
  constexpr int NB = BN == 64 ? 1 : 2;  // A buffers (static smem limit 48 KB)
  __shared__ __align__(16) float As[NB][BM * AS];
  __shared__ __align__(16) float Bb[TC_BK * BS];
  __shared__ __align__(16) float Bl[TC_BK * BS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WMW, wn = warp / WMW;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  A += blockIdx.z * sA;
  C += blockIdx.z * sC;
  const bool vec = (lda & 3) == 0;
  float acc[MT][4][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.f;

  auto load_a = [&](int buf, int k0) {
    float* dst = As[buf % NB];
    if (vec) {
      // 128 rows x 8 float4 = 1024 chunks, 4 per thread
      for (int e = tid; e < BM * (TC_BK / 4); e += 256) {
        const int r = e >> 3, c4 = (e & 7) * 4;
        const int gm = m0 + r, gk = k0 + c4;
        float* d = dst + r * AS + c4;
        if (gm < M && gk + 3 < K) {
          cp_async16(d, A + (long long)gm * lda + gk);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) d[q] = (gm < M && gk + q < K) ? __ldg(A + (long long)gm * lda + gk + q) : 0.f;
        }
      }
    } else {
      for (int e = tid; e < BM * TC_BK; e += 256) {
        const int r = e / TC_BK, kk = e % TC_BK;
        const int gm = m0 + r, gk = k0 + kk;
        dst[r * AS + kk] = (gm < M && gk < K) ? __ldg(A + (long long)gm * lda + gk) : 0.f;
      }
    }
    cp_async_commit_tc();
  };

  load_a(0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += TC_BK, buf ^= 1) {
    __syncthreads();  // previous iteration's MMAs are done with Bb/Bl and As[buf ^ 1]
    if (NB == 2) {
      if (k0 + TC_BK < K) load_a(buf ^ 1, k0 + TC_BK);
    } else if (k0 > 0) {
      load_a(0, k0);
    }
    for (int e = tid; e < TC_BK * BN; e += 256) {
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      const bool in = gk < K && gn < N;
      Bb[kk * BS + nn] = in ? __ldg(Bbig + (long long)gk * ldb + gn) : 0.f;
      Bl[kk * BS + nn] = in ? __ldg(Bsmall + (long long)gk * ldb + gn) : 0.f;
    }
    if (NB == 2 && k0 + TC_BK < K)
      cp_async_wait_tc<1>();
    else
      cp_async_wait_tc<0>();
    __syncthreads();
    const float* Acur = As[buf % NB];
#pragma unroll
    for (int ks = 0; ks < TC_BK; ks += 8) {
      uint32_t bb[4][2], bl[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + g;
        bb[j][0] = __float_as_uint(Bb[(ks + t) * BS + n]);
        bb[j][1] = __float_as_uint(Bb[(ks + t + 4) * BS + n]);
        bl[j][0] = __float_as_uint(Bl[(ks + t) * BS + n]);
        bl[j][1] = __float_as_uint(Bl[(ks + t + 4) * BS + n]);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = wm * WM + i * 16 + g;
        const float x0 = Acur[r * AS + ks + t], x1 = Acur[(r + 8) * AS + ks + t];
        const float x2 = Acur[r * AS + ks + t + 4], x3 = Acur[(r + 8) * AS + ks + t + 4];
        uint32_t ab[4] = {f2tf32(x0), f2tf32(x1), f2tf32(x2), f2tf32(x3)};
        uint32_t al[4] = {f2tf32(x0 - __uint_as_float(ab[0])), f2tf32(x1 - __uint_as_float(ab[1])),
                          f2tf32(x2 - __uint_as_float(ab[2])), f2tf32(x3 - __uint_as_float(ab[3]))};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mma_tf32(acc[i][j], al, bb[j][0], bb[j][1]);
          mma_tf32(acc[i][j], ab, bl[j][0], bl[j][1]);
          mma_tf32(acc[i][j], ab, bb[j][0], bb[j][1]);
        }
      }
    }
  }
  // C fragment: (g, 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)
#pragma unroll
  for (int i = 0; i < MT; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + wn * 32 + j * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm * WM + i * 16 + g + 8 * h;
        if (m >= M) continue;
        float* crow = C + (long long)m * ldc;
        const float v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
        if (n + 1 < N && (ldc & 1) == 0) {
          *reinterpret_cast<float2*>(crow + n) = make_float2(v0, v1);
        } else {
          if (n < N) crow[n] = v0;
          if (n + 1 < N) crow[n + 1] = v1;
        }
      }
    }
  }
}

__global__ void tf32_split_kernel(const float* __restrict__ in, float* __restrict__ big, float* __restrict__ small,
                                  long long n) {
  pdl_prologue();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float x = in[i];
    const uint32_t b = f2tf32(x);
    big[i] = __uint_as_float(b);
    small[i] = __uint_as_float(f2tf32(x - __uint_as_float(b)));
  }
}

void launch_tf32_split(const float* in, float* big, float* small, long long n, cudaStream_t s) {
  pdl_launch(tf32_split_kernel, grid_for(n, 256), 256, 0, s, in, big, small, n);
  LDDMM_LAUNCH_CHECK();
}

void launch_tc3_gemm(const float* A, int lda, long long sA, const float* Bbig, const float* Bsmall, int ldb, float* C,
                     int ldc, long long sC, int M, int N, int K, int batch, cudaStream_t s) {
  if (N <= 32) {
    dim3 grid(ceil_div(N, 32), ceil_div(M, 128), batch);
    pdl_launch(tc3_gemm_kernel<32>, grid, 256, 0, s, A, lda, sA, Bbig, Bsmall, ldb, C, ldc, sC, M, N, K);
  } else {
    dim3 grid(ceil_div(N, 64), ceil_div(M, 128), batch);
    pdl_launch(tc3_gemm_kernel<64>, grid, 256, 0, s, A, lda, sA, Bbig, Bsmall, ldb, C, ldc, sC, M, N, K);
  }
  LDDMM_LAUNCH_CHECK();
}

}  // namespace lddmm_b200
