// Shared device/host helpers for the B200 band-limited SL-LDDMM engine.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <stdexcept>
#include <string>

namespace lddmm_b200 {

// Error classes mirror the reference (core.hpp:21-38): ShapeError -> status 1,
// DivergenceError(step) -> status 2, anything CUDA/other -> status 3.
struct EngineError : std::runtime_error {
  int status;
  int step;
  EngineError(int st, const std::string& m, int s = -1) : std::runtime_error(m), status(st), step(s) {}
};

inline void shape_require(bool ok, const std::string& msg) {
  if (!ok) throw EngineError(1, msg);
}

#define LDDMM_CUDA(call)                                                                            \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw ::lddmm_b200::EngineError(3, std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                                             " at " + __FILE__ + ":" + std::to_string(__LINE__));  \
  } while (0)

// Every kernel launch in the engine is followed by LDDMM_LAUNCH_CHECK(), which
// also counts it (reported as gpu_launches by bench.py).
inline long long& launch_counter() {
  static long long c = 0;
  return c;
}
#define LDDMM_LAUNCH_CHECK()                    \
  do {                                          \
    ++::lddmm_b200::launch_counter();           \
    LDDMM_CUDA(cudaGetLastError());             \
  } while (0)

// NVTX range for the host-side phases (forward / gradient / hessvec / GN iteration /
// PCG): visible in any NVTX-aware profiler timeline; header-only (nvtx3), no-ops when
// no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define LDDMM_NVTX_CAT2(a, b) a##b
#define LDDMM_NVTX_CAT(a, b) LDDMM_NVTX_CAT2(a, b)
#define LDDMM_NVTX(name) ::lddmm_b200::NvtxRange LDDMM_NVTX_CAT(nvtx_range_, __LINE__)(name)

// Programmatic dependent launch (PDL).  Every engine kernel starts with pdl_prologue()
// (kernels with constant set-up — twiddle tables, TMEM allocation, mbarriers — do that
// first and call pdl_wait() / pdl_trigger() after it):
// griddepcontrol.wait (no access to global memory before the preceding kernel in the
// stream has completed and its writes are visible), then launch_dependents (the next
// kernel may be scheduled now).  Kernels are launched through pdl_launch(), which sets
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's launch and CTA
// ramp-up overlap its predecessor's tail instead of following it.  Without the
// attribute (LDDMM_PDL=0) the two instructions are no-ops and launches are ordinary.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_prologue() {
  pdl_wait();
  pdl_trigger();
}

inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("LDDMM_PDL");
    v = e ? std::atoi(e) : 1;
  }
  return v != 0;
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);  // errors surface in LDDMM_LAUNCH_CHECK
}

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// grid-stride loop over [0, n)
#define GRID_STRIDE(i, n) \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

// Grid-stride launch size: a multiple of the SM count, capped.
inline int grid_for(long long n, int block, int per_sm = 8) {
  long long g = (n + block - 1) / block;
  long long cap = (long long)kSMs * per_sm;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

// Number of partial slots used by the deterministic two-pass reductions.
constexpr int kReduceBlocks = kSMs * 4;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reductions (blockDim a multiple of 32); result valid in every thread.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double r = (lane < nw) ? sh[lane] : 0.0;
  r = warp_sum(r);
  return r;
}

__device__ __forceinline__ double block_max(double v) {
  __shared__ double sh[32];
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double r = (lane < nw) ? sh[lane] : -INFINITY;
  r = warp_max(r);
  return r;
}

}  // namespace lddmm_b200
