// Microbenchmark (B200, sm_100a): FP32 FMA pipe throughput for scalar 3-register FFMA
// vs packed FFMA2, and LDS.128 throughput.  Decides how the SL gather's inner loop is
// written.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_pipe fma_pipe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ unsigned long long g_cyc[4096];
template <int CH>
__global__ void k_ffma(float* out, float a, float b) {
  const long long c0 = clock64();
  float x[CH], w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3f + c; w[c] = a + c * 1e-4f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], w[c], w[(c + 1) % CH]);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == b) out[threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - c0;
}

template <int CH>
__global__ void k_ffma2(float* out, float a, float b) {
  const long long c0 = clock64();
  float2 x[CH], w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = make_float2(threadIdx.x * 1e-3f + c, c); w[c] = make_float2(a + c * 1e-4f, a - c * 1e-4f); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(x[c], w[c], w[(c + 1) % CH]);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c].x + x[c].y;
  if (s == b) out[threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - c0;
}

// FFMA2 with a broadcast scalar data operand (R.F32 form)
template <int CH>
__global__ void k_ffma2b(float* out, float a, float b) {
  const long long c0 = clock64();
  float2 x[CH], w[CH];
  float d[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = make_float2(threadIdx.x * 1e-3f + c, c); w[c] = make_float2(a + c * 1e-4f, a - c * 1e-4f); d[c] = a * c; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(w[c], make_float2(d[(c + 3) % CH], d[(c + 3) % CH]), x[c]);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c].x + x[c].y;
  if (s == b) out[threadIdx.x] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - c0;
}

__global__ void k_lds128(float* out, float b) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x & 1023;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = sm[(idx + u * 32) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    idx += 1;
  }
  if (acc.x + acc.y + acc.z + acc.w == b) out[threadIdx.x] = acc.x;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d MHz\n", sms, clk / 1000);
  auto cyc = [&](int blocks) {
    static unsigned long long h[4096];
    cudaMemcpyFromSymbol(h, g_cyc, blocks * sizeof(unsigned long long));
    double s = 0; for (int i = 0; i < blocks; ++i) s += h[i];
    return s / blocks;
  };
  for (int th : {128, 256, 512, 1024}) {
    const int blocks = sms * (1024 / th) * 2;
    double fmas = (double)blocks * th * ITERS;
    float t;
    t = timeit([&] { k_ffma<8><<<blocks, th>>>(out, 1.0001f, -1); });
    printf("FFMA  x8 chains th=%4d: %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM\n", th, t, fmas * 8 / t / 1e9,
           fmas * 8 / (t * 1e-3) / sms / (clk * 1e3));
    t = timeit([&] { k_ffma2<4><<<blocks, th>>>(out, 1.0001f, -1); });
    printf("FFMA2 x4 chains th=%4d: %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM\n", th, t, fmas * 8 / t / 1e9,
           fmas * 8 / (t * 1e-3) / sms / (clk * 1e3));
    t = timeit([&] { k_ffma<16><<<blocks, th>>>(out, 1.0001f, -1); });
    printf("FFMA  x16 chains th=%4d: %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM\n", th, t, fmas * 16 / t / 1e9,
           fmas * 16 / (t * 1e-3) / sms / (clk * 1e3));
    t = timeit([&] { k_ffma2<8><<<blocks, th>>>(out, 1.0001f, -1); });
    printf("FFMA2 x8 chains th=%4d: %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM\n", th, t, fmas * 16 / t / 1e9,
           fmas * 16 / (t * 1e-3) / sms / (clk * 1e3));
    {
      // per-SM cycle based: one resident wave (blocks = sms * (2048/th)), ops per SM / cycles per block
      const int wave = sms * (2048 / th);
      double ops = (double)(2048 / th) * th * ITERS;  // per SM per chain-iteration
      k_ffma<16><<<wave, th>>>(out, 1.0001f, -1); cudaDeviceSynchronize();
      printf("  [cyc] FFMA  x16: %.1f FMA/clk/SM\n", ops * 16 / cyc(wave));
      k_ffma2<8><<<wave, th>>>(out, 1.0001f, -1); cudaDeviceSynchronize();
      printf("  [cyc] FFMA2 x8 : %.1f FMA/clk/SM\n", ops * 16 / cyc(wave));
      k_ffma2b<8><<<wave, th>>>(out, 1.0001f, -1); cudaDeviceSynchronize();
      printf("  [cyc] FFMA2 bcast x8 : %.1f FMA/clk/SM\n", ops * 16 / cyc(wave));
    }
    t = timeit([&] { k_lds128<<<blocks, th>>>(out, -1); });
    double bytes = (double)blocks * th * ITERS * 8 * 16;
    printf("LDS.128 th=%4d: %.3f ms  %.1f B/clk/SM\n", th, t, bytes / (t * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
