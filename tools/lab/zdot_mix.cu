// Microbenchmark: throughput of the gather's per-row arithmetic (register-only, no
// shared memory): (a) gw_item's mixed FFMA2 / scalar FFMA z-dot + FFMA2 accumulate,
// (b) all-scalar FFMA, (c) all-FFMA2 with broadcast data operands (zero-weight lanes).
// Reports useful FMAs (24 per row per 4 nodes) per clock per SM at 1965 MHz.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ROWS = 2048;

__device__ __forceinline__ void zdot_mix(const float (&win)[8], const float2 (&wz)[2][5], float2& pa, float2& pb) {
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
__device__ __forceinline__ void zdot_scalar(const float (&win)[8], const float2 (&wz)[2][5], float2& pa, float2& pb) {
  pa.x = wz[0][0].x * win[0]; pa.y = wz[0][0].y * win[1]; pb.x = wz[1][0].x * win[2]; pb.y = wz[1][0].y * win[3];
#pragma unroll
  for (int k = 1; k < 5; ++k) {
    pa.x = fmaf(wz[0][k].x, win[k], pa.x);
    pa.y = fmaf(wz[0][k].y, win[k + 1], pa.y);
    pb.x = fmaf(wz[1][k].x, win[k + 2], pb.x);
    pb.y = fmaf(wz[1][k].y, win[k + 3], pb.y);
  }
}
// broadcast form: for window element q, nodes m with q-m in [0,4]: pairs (0,1), (2,3)
__device__ __forceinline__ void zdot_bcast(const float (&win)[8], const float2 (&wz)[2][6], float2& pa, float2& pb) {
  // wz[h][q'] = (w_{2h}[q' ], w_{2h+1}[q'-1]) with zeros outside; q' = q - 2h in 0..5
  pa = __fmul2_rn(wz[0][0], make_float2(win[0], win[0]));
  pb = __fmul2_rn(wz[1][0], make_float2(win[2], win[2]));
#pragma unroll
  for (int q = 1; q < 6; ++q) {
    pa = __ffma2_rn(wz[0][q], make_float2(win[q], win[q]), pa);
    pb = __ffma2_rn(wz[1][q], make_float2(win[q + 2], win[q + 2]), pb);
  }
}

template <int MODE, int NC>
__global__ void __launch_bounds__(512, 1) k(const float* in, float* out) {
  float win[NC][8];
  float2 wz[2][6], w01 = make_float2(in[threadIdx.x & 7], in[(threadIdx.x + 1) & 7]);
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int i = 0; i < 8; ++i) win[c][i] = in[(threadIdx.x + i + c) & 63];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 6; ++i) wz[h][i] = make_float2(in[i + h], in[i + 3 + h]);
  float2 acc[NC][2];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c][0] = acc[c][1] = make_float2(0, 0);
  for (int r = 0; r < ROWS; ++r) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float2 pa, pb;
      if (MODE == 0) zdot_mix(win[c], reinterpret_cast<const float2(&)[2][5]>(wz), pa, pb);
      if (MODE == 1) zdot_scalar(win[c], reinterpret_cast<const float2(&)[2][5]>(wz), pa, pb);
      if (MODE == 2) zdot_bcast(win[c], wz, pa, pb);
      acc[c][0] = __ffma2_rn(w01, pa, acc[c][0]);
      acc[c][1] = __ffma2_rn(w01, pb, acc[c][1]);
      // perturb the window so the compiler cannot hoist the z-dots
      win[c][0] += 1e-7f; win[c][5] -= 1e-7f;
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += acc[c][0].x + acc[c][0].y + acc[c][1].x + acc[c][1].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, float* in, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int th : {256, 384, 512}) {
    k<MODE, 3><<<148, th>>>(in, out);
    cudaEventRecord(a);
    k<MODE, 3><<<148, th>>>(in, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double useful = 148.0 * th * ROWS * 3 * 24;
    printf("%-28s th=%d: %.3f ms  useful %.1f FMA/clk/SM\n", name, th, ms, useful / (ms * 1e-3) / 148 / 1.965e9);
  }
}
int main() {
  float *in, *out;
  cudaMalloc(&in, 64 * 4); cudaMalloc(&out, 148 * 512 * 4);
  cudaMemset(in, 0, 256);
  run<0>("mixed FFMA2/FFMA (gw_item)", in, out);
  run<1>("scalar FFMA", in, out);
  run<2>("FFMA2 broadcast", in, out);
}
