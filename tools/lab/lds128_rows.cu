// LDS.128 wavefronts when the 32 lanes of a warp read 16-byte chunks whose bank groups
// are all distinct per 8-lane phase but that lie in different 128-byte rows.
// mode 0: lane l reads row 0, chunk l              (contiguous 512 B)
// mode 1: lane l reads row (l % 8) * 3, chunk l    (distinct rows, banks as mode 0)
// mode 2: lane l reads row l, chunk l % 8          (all lanes of a phase distinct banks)
// mode 3: lane l reads row l, chunk (l * 5) % 32   (bank groups balanced, 4 per group)
// mode 4: lane l reads row hash(l), chunk l        (random rows, contiguous chunks)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lab/lds128_rows.cu -o /tmp/lds && /tmp/lds
#include <cstdio>
#include <cuda_runtime.h>
constexpr int P = 192;  // floats per row (multiple of 32)
__global__ void k(float* out, int mode, int iters) {
  __shared__ __align__(16) float sm[40 * P];
  for (int i = threadIdx.x; i < 40 * P; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int l = threadIdx.x & 31;
  int row, chunk;
  if (mode == 0) { row = 0; chunk = l; }
  else if (mode == 1) { row = (l % 8) * 3; chunk = l; }
  else if (mode == 2) { row = l; chunk = l % 8; }
  else if (mode == 3) { row = l; chunk = (l * 5) % 32; }
  else { row = (l * 13 + 7) % 37; chunk = l; }
  const float* p = sm + row * P + 4 * chunk;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    float4 v;
    asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"((unsigned)__cvta_generic_to_shared(p)));
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    asm volatile("" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 4 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 5; ++mode) {
    k<<<148 * 4, 512>>>(o, mode, 4096);
    if (cudaDeviceSynchronize() != cudaSuccess) printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a);
    k<<<148 * 4, 512>>>(o, mode, 4096);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (cudaGetLastError() != cudaSuccess) printf("launch error\n");
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // wavefronts per LDS.128 ~ SM clocks per warp-instruction: 148 SMs, 1 LDS wavefront / clk
    const double inst = 148.0 * 4 * 16 * 4096;
    printf("mode %d: %.3f ms, %.2f clk per warp LDS.128 (at 1.965 GHz)\n", mode, ms, ms * 1e-3 * 1.965e9 * 148 / inst);
  }
  return 0;
}
