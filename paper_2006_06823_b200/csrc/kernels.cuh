// Kernel launch interfaces shared by the engine translation units.
#pragma once

#include <vector>

#include <cuda_runtime.h>

#include "common.cuh"

namespace lddmm_b200 {

// ---- spectral ---------------------------------------------------------------

enum : int {
  SYM_NONE = 0,
  SYM_DERIV_X = 1,  // i * omega_0
  SYM_DERIV_Y = 2,
  SYM_DERIV_Z = 3,
  SYM_DERIV_MASK = 3,
  SYM_PREFILTER = 4,  // 1 / B(k)
};

constexpr int kMaxPrep = 64;

struct PrepField {
  const double2* src;  // band field [Kx][Ky][Kz] (null -> zero)
  int sym;
  double scale;
};
struct PrepArgs {
  PrepField f[kMaxPrep];
  int nf;
};

struct FinField {
  double2* dst;        // band field [Kx][Ky][Kz]
  double alpha;        // dst = alpha * projected + beta * add
  const double2* add;  // may alias dst; may be null
  double beta;
};
struct FinArgs {
  FinField f[kMaxPrep];
  int nf;
};

// One (grid, band) pair: twiddle tables for the separable truncated DFTs.
struct DftPlan {
  int N[3];               // grid the transform lives on (parent grid or the small product grid)
  int K[3];               // band bounds
  double omega_unit[3];   // 2 pi / (N_a h_a) of the PARENT grid (spectral.hpp:77-79)
  float2* wy_e = nullptr;  // [Ny][Ky]  exp(+2 pi i ky y / Ny)
  float2* wx_e = nullptr;  // [Nx][Kx]
  float* tz_e = nullptr;   // [2H][Nz]  (cos, -sin)(2 pi kz z / Nz) / Ntot
  float* tz_p = nullptr;   // [Nz][2H]  (cos, -sin)(2 pi kz z / Nz)
  float2* wx_p = nullptr;  // [Kx][Nx]  exp(-2 pi i kx x / Nx)
  float2* wy_p = nullptr;  // [Ky][Ny]
  // TF32 big/small splits of the z tables for the tensor-core (3xTF32) z stages
  float *tz_e_big = nullptr, *tz_e_small = nullptr, *tz_p_big = nullptr, *tz_p_small = nullptr;
  // Tz_e big/small in the canonical K-major UMMA layout (tcgen05 embed-z), or null
  float *uz_e_big = nullptr, *uz_e_small = nullptr;
  // Tz_p in the canonical UMMA layout, K zero-padded to whole chunks (tcgen05 z-project), or null
  float *uz_p_big = nullptr, *uz_p_small = nullptr;
  // Wx_e / Wx_p as the tcgen05 x-stage twiddle operand (umma_xstage.cu: real / imaginary x
  // TF32 big / small, canonical K-major), or null (FFMA x stage)
  float *ux_e = nullptr, *ux_p = nullptr;
  // B(k) factors of the prefilter symbol per axis [Kx | Ky | Kz] (launch_band_symbols)
  double* bsym = nullptr;
  long long npts() const { return (long long)N[0] * N[1] * N[2]; }
  long long half() const { return (long long)K[0] * K[1] * (K[2] / 2); }
  long long kprod() const { return (long long)K[0] * K[1] * K[2]; }
};

void launch_band_prep(const PrepArgs& a, const DftPlan& p, float2* D, cudaStream_t s);
void launch_band_symbols(const int* K, const int* N, double* out, cudaStream_t s);
void launch_band_finalize(const FinArgs& a, const DftPlan& p, const float2* G, cudaStream_t s);
void dft_embed_prep(const DftPlan& p, const PrepArgs& a, float2* D, float2* E1, float2* E2, float* out,
                    cudaStream_t s);
void dft_embed(const DftPlan& p, const float2* D, int nf, float2* E1, float2* E2, float* out, cudaStream_t s);
void dft_project_fin(const DftPlan& p, const float* f, const FinArgs& a, float2* G1, float2* G2, float2* G3,
                     cudaStream_t s);
void dft_project(const DftPlan& p, const float* f, int nf, float2* G1, float2* G2, float2* G3, cudaStream_t s);
void launch_sgemm(const float* A, int lda, long long sA, const float* B, int ldb, float* C, int ldc,
                  long long sC, int M, int N, int K, int batch, cudaStream_t s);
void launch_cgemm(const float2* A, int lda, const float2* B, long long sB, int ldb, float2* C, long long sC,
                  int ldc, int M, int N, int K, int batch, cudaStream_t s);
// 3xTF32 tensor-core GEMM C[b] = A[b] * B with B given as TF32 big/small parts (tc_gemm.cu)
void launch_tc3_gemm(const float* A, int lda, long long sA, const float* Bbig, const float* Bsmall, int ldb, float* C,
                     int ldc, long long sC, int M, int N, int K, int batch, cudaStream_t s);
void launch_tf32_split(const float* in, float* big, float* small, long long n, cudaStream_t s);
// tcgen05 3xTF32 complex x-stage GEMM (umma_xstage.cu): C[f] = W X[f], W [M][K], X [K][N],
// C [M][N] complex; twiddle operand prepared on the host
bool umma_xstage_fits(int M, int K, int N);
long long umma_xstage_twiddle_floats(int M, int K);
void umma_xstage_twiddles_host(const float2* W, int M, int K, std::vector<float>& out);
void launch_umma_xstage(const float* tw, const float2* X, long long sX, float2* C, long long sC, int M, int N, int K,
                        int nf, cudaStream_t s);
// tcgen05 3xTF32 embed-z GEMM (umma_gemm.cu): C[b] = A[b] * B, A [M][K] rows, C [M][N] rows
int umma_padded_n(int N);
bool umma_zembed_fits(int N, int K);
void launch_umma_canon_b(const float* Bbig, const float* Bsm, int K, int N, float* Cbig, float* Csm, cudaStream_t s);
// tcgen05 3xTF32 z-project GEMM (A streamed by cp.async into the canonical layout)
bool umma_zproject_fits(int K, int N);
int umma_zproject_kpad(int K);
void launch_umma_zproj_prep(const float* Bbig, const float* Bsm, int K, int N, float* Cbig, float* Csm,
                            cudaStream_t s);
void launch_umma_zproject(const float* A, const float* Bbig_c, const float* Bsm_c, float* C, int M, int K, int N,
                          cudaStream_t s);
void launch_umma_zembed(const float* A, long long sA, const float* Bbig_c, const float* Bsm_c, float* C, long long sC,
                        int M, int N, int K, int nb, cudaStream_t s);

// ---- interpolation / transport -------------------------------------------------

// out[c][i] = cubic B-spline sample of coef[c] at node i + disp[:, i] (grid units), c < ncomp
void launch_gather_cubic(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                         cudaStream_t s);
// alternative implementations of the same gather (tests / ablations)
void launch_gather_cubic_tiled(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                               cudaStream_t s);
void launch_gather_cubic_global(const float* coef, int ncomp, const float* disp, float* out, const int* N,
                                cudaStream_t s);
// grid-unit departure displacements for both directions (transport.hpp:83-102)
void launch_departure(const float* vgrid, const float* vcoef, double dt, const double* h, float* dep_fwd,
                      float* dep_bwd, float* scratch, const int* N, cudaStream_t s);
// one direction: X* = x + sg dt vgrid, out = sg dt/2 (vcoef-sample(X*) + vgrid) in grid units;
// vm: [3][N] scratch (separate arrival / traced nodes for nonstationary velocities)
void launch_departure_dir(const float* vgrid, const float* vcoef, double dt, const double* h, float sg, float* out,
                          float* vm, const int* N, cudaStream_t s);
// pipelined marching gather (gather_pipe.cu); false when the shape is not supported
bool gather_pipe_supported(const int* N);
bool launch_gather_pipe(const float* coef, int ncomp, const float* disp, float* out, const int* N, float3 sc,
                        cudaStream_t s);
// gather with the displacement scaled per axis: samples coef at node + (sx dx, sy dy, sz dz)
void launch_gather_scaled(const float* coef, int ncomp, const float* disp, float sx, float sy, float sz, float* out,
                          const int* N, cudaStream_t s, bool march = true);
// cubic pull-back of coef at x - disp_phys where disp is a grid field in physical units
// (points_from_displacement, variants.hpp:49-51); out[c] for ncomp coefficient fields
void launch_warp_by_displacement(const float* coef, int ncomp, const float* disp_phys, const double* h,
                                 float* out, const int* N, cudaStream_t s, bool large = false);
// nearest-neighbour pull-back (warp_nearest, interp.hpp:213-225): out[c](x) =
// f[c](wrap(llround((x - disp(x)) / h))), fp64 index arithmetic
void launch_warp_nearest(const float* f, int ncomp, const float* disp_phys, const double* h, float* out,
                         const int* N, cudaStream_t s);
// exact periodic prefilter (interp.hpp:23-63) along every axis, fp64, in place
void launch_prefilter3d(double* f, const int* N, cudaStream_t s);
void launch_prefilter3d_f32(float* f, const int* N, cudaStream_t s);
// out = spectral derivative of in along `axis` (fp64), D = circulant kernel [N[axis]]
void launch_circulant_axis_f64(const double* in, double* out, const double* D, int axis, const int* N,
                               cudaStream_t s);

// ---- band algebra (fp64) ----------------------------------------------------------

void launch_axpy(long long n, double a, const double2* x, const double2* y, double2* out, cudaStream_t s);
// out = sum_{j < count} w_j (x + j stride), in order (= launch_scale + count - 1 launch_axpy)
void launch_weighted_sum(long long n, int count, const double* w, const double2* x, long long stride, double2* out,
                         cudaStream_t s);
void launch_axpby(long long n, double a, const double2* x, double b, const double2* y, double2* out,
                  cudaStream_t s);
void launch_scale(long long n, double a, const double2* x, double2* out, cudaStream_t s);
// out[c] = in[c] * (1 + alpha |omega|^2)^(+-s)  (SobolevOperator::apply, spectral.hpp:527-544)
void launch_sobolev(const double2* in, double2* out, int ncomp, const int* K, const double* wunit, double alpha,
                    int s, bool inverse, cudaStream_t st);
// div = sum_a i omega_a v_a  (band_divergence, spectral.hpp:440-451)
void launch_band_divergence(const double2* v, double2* out, const int* K, const double* wunit, cudaStream_t s);
// partial reductions into part[0..g) (g returned); finished by launch_reduce_final into slot
int launch_inner_partial(long long n, const double2* x, const double2* y, double* part, cudaStream_t s);
int launch_linf_partial(long long n, const double2* x, double* part, cudaStream_t s);
int launch_nonfinite_partial(long long n, const double2* x, double* part, cudaStream_t s);
// 1.0 into *slot when x holds a non-finite value, else 0.0; part needs kReduceBlocks + 1
// doubles, the last one a zero-initialised counter
void launch_nonfinite_flag(long long n, const double2* x, double* part, double* slot, cudaStream_t s);
// flags of `count` consecutive nodes base + j V into slots[step], step = step0 + j (or
// step0 + count - 1 - j backward), one launch (the slots are zeroed first)
void launch_nonfinite_series(const double2* base, long long V, int count, int step0, bool backward, double* slots,
                             cudaStream_t s);
void launch_reduce_final(const double* part, int nparts, int op /*0 sum 1 max*/, double* slot, cudaStream_t s);

// ---- grid pointwise (fp32 fields, fp64 reductions) --------------------------------

void launch_f64_to_f32(long long n, const double* in, float* out, cudaStream_t s);
void launch_f32_to_f64(long long n, const float* in, double* out, cudaStream_t s);
// res = m1 - I1 ; part <- sum res^2
int launch_residual(long long n, const float* m1, const float* I1, float* res, double* part, cudaStream_t s);
int launch_sumsq_partial(long long n, const float* x, double* part, cudaStream_t s);
int launch_absmax_partial(long long n, const float* x, double* part, cudaStream_t s);
// r1_a = (c * res) * g_a    (variants.hpp:431)
void launch_scale_vec(long long n, const float* res, double c, const float* g, float* out, cudaStream_t s);
// dr1_a = ((-1 * sum_b g_b du_b) * c) * g_a   (variants.hpp:326-336)
void launch_dr1(long long n, const float* g, const float* du, double c, float* out, cudaStream_t s);
// dlam1 = ((-1 * sum_b g_b du_b) * c)   (variants.hpp:326-327)
void launch_dlam1(long long n, const float* g, const float* du, double c, float* out, cudaStream_t s);
// product kernels on the small grid, accumulate with weight w: op 0 jac, 1 jacT, 2 s*vec, 3 dot, 4 s*s
void launch_products(int op, long long n, const float* a, const float* b, float* acc, float w, bool init,
                     cudaStream_t s);
// node-batched Jacobian products on the small grid (band_jac_mul / band_jacT_mul integrands,
// spectral.hpp:480-510).  derivs [nn][9][M] (d_b u_a at index a*3+b), w [nn|1][3][M].
// out_stride == 0: acc[3][M] (+)= sum_n wts[n] * prod_n ; else out[n][3][M] = prod_n.
struct NodeWeights {
  float w[8];
};
void launch_equal_flag(long long n, const double* a, const double* b, unsigned long long* mismatch, cudaStream_t s);
void launch_jac_batch(bool transpose, int nn, long long M, const float* derivs, const float* w,
                      long long w_node_stride, float* out, long long out_stride, NodeWeights wts, bool init,
                      cudaStream_t s);
// det(I - Du) min/max from 9 derivative fields [a][b][N] (metrics.hpp:40-65)
int launch_jacdet_minmax(long long n, const float* du, double* part_min, double* part_max, cudaStream_t s);
void launch_jacdet(long long n, const float* du, float* out, cudaStream_t s);
// Dice counts (metrics.hpp:100-118) for nl label values (device array): counts[3 l + 0..2] =
// |a == l|, |b == l|, |a == l && b == l|; counts zeroed by the launcher
void launch_dice_counts(long long n, const float* a, const float* b, const float* labels, int nl,
                        unsigned long long* counts, cudaStream_t s);
// affine: out = a * x + b  (fp32 grid)
void launch_affine_f32(long long n, const float* x, float a, float b, float* out, cudaStream_t s);
void launch_mul_f32(long long n, const float* x, const float* y, float* out, cudaStream_t s);

}  // namespace lddmm_b200
