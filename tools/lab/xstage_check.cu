// Standalone check of the tcgen05 x-stage complex GEMM (umma_xstage.cu) against a CPU
// reference: C[f][m][n] = sum_k W[m][k] X[f][k][n].
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -lcuda \
//        tools/lab/xstage_check.cu -o /tmp/xs && /tmp/xs M K N nf
// (add -DWITH_FFMA -Lpaper_2006_06823_b200 -llddmm_cuda to time the FFMA x stage too)
#include "../../paper_2006_06823_b200/csrc/umma_xstage.cu"

#include <cmath>
#include <cstdio>
#include <random>

using namespace lddmm_b200;

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 180, K = argc > 2 ? atoi(argv[2]) : 32;
  const int N = argc > 3 ? atoi(argv[3]) : 3360, nf = argc > 4 ? atoi(argv[4]) : 2;
  printf("M %d K %d N %d nf %d fits %d\n", M, K, N, nf, (int)umma_xstage_fits(M, K, N));
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float2> W((size_t)M * K), X((size_t)nf * K * N), C((size_t)nf * M * N);
  for (auto& w : W) w = make_float2(U(rng), U(rng));
  for (auto& x : X) x = make_float2(U(rng), U(rng));
  std::vector<float> tw;
  umma_xstage_twiddles_host(W.data(), M, K, tw);
  float *dtw;
  float2 *dX, *dC;
  cudaMalloc(&dtw, tw.size() * 4);
  cudaMalloc(&dX, X.size() * 8);
  cudaMalloc(&dC, C.size() * 8);
  cudaMemcpy(dtw, tw.data(), tw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, C.size() * 8);
  try {
    launch_umma_xstage(dtw, dX, (long long)K * N, dC, (long long)M * N, M, N, K, nf, 0);
  } catch (std::exception& e) {
    printf("launch: %s\n", e.what());
    return 1;
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(err));
  cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  int shown = 0;
  for (int f = 0; f < nf; ++f)
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double re = 0, im = 0;
        for (int k = 0; k < K; ++k) {
          const float2 w = W[(size_t)m * K + k], x = X[((size_t)f * K + k) * N + n];
          re += (double)w.x * x.x - (double)w.y * x.y;
          im += (double)w.x * x.y + (double)w.y * x.x;
        }
        const float2 c = C[((size_t)f * M + m) * N + n];
        const double e = std::max(std::fabs(c.x - re), std::fabs(c.y - im));
        if (e > 1e-3 && shown < 8) {
          printf("f %d m %d n %d: got (%g, %g) want (%g, %g)\n", f, m, n, c.x, c.y, re, im);
          ++shown;
        }
        maxerr = std::max(maxerr, e);
        maxref = std::max(maxref, std::max(std::fabs(re), std::fabs(im)));
      }
  printf("max abs err %.3e (max |C| %.3e, rel %.3e)\n", maxerr, maxref, maxerr / maxref);
  // timing
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) launch_umma_xstage(dtw, dX, (long long)K * N, dC, (long long)M * N, M, N, K, nf, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)nf * (K + M) * N * 8;
  printf("%.2f us per launch, %.0f GB/s\n", ms * 1e3 / 20, bytes / (ms / 20 * 1e-3) / 1e9);
#ifdef WITH_FFMA
  // the FFMA x stage (spectral.cu launch_cgemm) on the same operands, from liblddmm_cuda.so
  float2* dW;
  cudaMalloc(&dW, W.size() * 8);
  cudaMemcpy(dW, W.data(), W.size() * 8, cudaMemcpyHostToDevice);
  launch_cgemm(dW, K, dX, (long long)K * N, N, dC, (long long)M * N, N, M, N, K, nf, 0);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) launch_cgemm(dW, K, dX, (long long)K * N, N, dC, (long long)M * N, N, M, N, K, nf, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("FFMA cgemm: %.2f us per launch\n", ms * 1e3 / 20);
#endif
  return 0;
}
