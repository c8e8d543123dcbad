/* lddmm_cuda.h — C ABI of the B200-native band-limited SL-RK2 GN-Krylov engine
 * (liblddmm_cuda.so, built from paper_2006_06823_b200/csrc for sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (arxiv 2006.06823, /root/reference/proj/include/lddmm) is a header-only C++
 * template library with no FFI; its operator surface for this path is
 * Model<BandAlgebra> + optimize<BandAlgebra> (variants.hpp:229-548,
 * optimizer.hpp:18-262).  Each entry point below names the reference
 * interface it replaces.  Plain C types only: pointers, sizes, doubles.
 *
 * Layouts (identical to the reference):
 *   grid scalar  double[N], row-major, axis 0 slowest      (core.hpp:8-9,133-146)
 *   grid vector  double[3][N], component-major             (core.hpp:148-160)
 *   band vector  double[3][Kx*Ky*Kz][2] interleaved re/im, DFT order, band-Nyquist
 *                planes zero                                 (spectral.hpp:8-12,95-107)
 *   velocity     stationary: one band vector; nonstationary: nt+1 of them
 *                (core.hpp:275-317)
 * "dev" pointers are CUDA device pointers on the context's device; "host"
 * pointers are ordinary host memory.
 *
 * Errors mirror the reference exceptions (core.hpp:21-38): every int-returning
 * call returns LDDMM_OK, LDDMM_ESHAPE (ShapeError/Error), LDDMM_EDIVERGENCE
 * (DivergenceError; *step receives its step index where a step pointer is
 * taken) or LDDMM_ECUDA; lddmm_last_error() returns the message.
 * Threading: one host thread per context; contexts are independent.
 */
#ifndef LDDMM_CUDA_H
#define LDDMM_CUDA_H

#ifdef __cplusplus
extern "C" {
#endif

enum { LDDMM_OK = 0, LDDMM_ESHAPE = 1, LDDMM_EDIVERGENCE = 2, LDDMM_ECUDA = 3 };

/* Variant (variants.hpp:34) */
enum { LDDMM_ORIGINAL = 0, LDDMM_STATE_EQUATION = 1, LDDMM_DEFORMATION_STATE_EQUATION = 2 };
/* Parameterization (core.hpp:271) */
enum { LDDMM_STATIONARY = 0, LDDMM_NONSTATIONARY = 1 };
/* Integrator (variants.hpp:35; note the reference enum order is {rk4, sl}: these
 * values are the engine's, with the SL default at 0) */
enum { LDDMM_SL = 0, LDDMM_RK4 = 1 };
/* StopReason (optimizer.hpp:29-36), same order */
enum {
  LDDMM_STOP_GRADIENT = 0,
  LDDMM_STOP_ENERGY_CHANGE,
  LDDMM_STOP_STEP_SIZE,
  LDDMM_STOP_ZERO_GRADIENT,
  LDDMM_STOP_MAX_ITERATIONS,
  LDDMM_STOP_LINE_SEARCH_FAILURE
};

typedef struct lddmm_ctx lddmm_ctx;

/* Model<BandAlgebra> construction data: GridSpec (core.hpp:42-122), BandSpec
 * (spectral.hpp:22-83), Model fields variant/nt/sigma2/lop (variants.hpp:237-244),
 * SobolevOperator (spectral.hpp:518-525), Model::integrator (variants.hpp:241).
 * d = 3 or 2, band representation; SL-RK2 (default) or RK4 transport; all three
 * variants; stationary and nonstationary.  d = 2: dims/spacing/band[2] are ignored;
 * every host-side layout of the ABI (images, fields, displacements, band velocities,
 * series) is the reference's 2-D one (2 vector components, Kx x Ky band); the engine
 * runs the problem z-replicated internally, so device velocity buffers and the
 * lddmm_op_* primitives use the internal 3-D layout. */
typedef struct {
  int d;
  int dims[3];
  double spacing[3];
  int band[3];
  int nt;
  int variant;
  int parameterization;
  double alpha;
  int s;
  double sigma2;
  int integrator; /* LDDMM_SL or LDDMM_RK4 (RK4 needs nt >= 2, transport.hpp:236) */
} lddmm_problem;

/* ForwardCache energies + cfl (variants.hpp:196-198) */
typedef struct {
  double energy, energy_reg, energy_data, cfl;
} lddmm_energies;

/* OptimizeOptions (optimizer.hpp:18-27) */
typedef struct {
  int max_iter;
  int pcg_max_iter;
  double pcg_tol, grad_tol, energy_tol, step_tol, armijo_c;
  int armijo_max_trials;
} lddmm_options;

/* IterationRecord (optimizer.hpp:50-61); pcg_residuals truncated at 16 */
typedef struct {
  int iter;
  double energy, energy_data, energy_reg, mse_rel, rel_grad;
  int pcg_iters;
  int pcg_fallback;
  double epsilon, cfl, wall_ms;
  int n_pcg_residuals;
  double pcg_residuals[16];
} lddmm_iteration_record;

/* OptimizeResult scalars (optimizer.hpp:63-74) + operation counts */
typedef struct {
  int stop_reason;
  int converged;
  int iterations;
  int n_history;
  double final_energy, rel_grad;
  int hessvecs, trials, forwards;
} lddmm_result;

void lddmm_default_options(lddmm_options* opt); /* OptimizeOptions{} defaults */

/* Model(dom, I0, I1) (variants.hpp:246-250) minus the images; owns device memory
 * and one CUDA stream on `device`. */
int lddmm_create(const lddmm_problem* problem, int device, lddmm_ctx** out);
void lddmm_destroy(lddmm_ctx* ctx);
const char* lddmm_last_error(const lddmm_ctx* ctx);
int lddmm_sync(lddmm_ctx* ctx);
long long lddmm_launch_count(void); /* kernels launched by this library (process-wide) */
/* the context's CUDA stream (cudaStream_t), for events / external synchronisation */
void* lddmm_stream(lddmm_ctx* ctx);
/* live timing (measurement only): mode bit 0 = CUDA events around every SL-gather
 * launch, bit 1 = around every full-grid truncated-DFT call; 0 = off (resets the
 * window).  gather stats = device ms summed over launches, launch count, algorithmic
 * bytes sum of N * (12 + 8 C) */
int lddmm_gather_timing(lddmm_ctx* ctx, int mode);
int lddmm_gather_stats(lddmm_ctx* ctx, double* ms, long long* launches, double* bytes);
/* same timing window: full-grid truncated DFT calls (embed / project pipelines of nf
 * fields), with their algorithmic flops (8 (y + x stage complex MACs)
 * + 4 (z stage real-complex MACs) per field). */
int lddmm_dft_stats(lddmm_ctx* ctx, double* ms, long long* launches, double* flops);

/* Model::source / Model::target (variants.hpp:238-239): host fp64 ScalarFields */
int lddmm_set_images(lddmm_ctx* ctx, const double* host_I0, const double* host_I1);
/* same, already resident: device fp32 */
int lddmm_set_images_dev_f32(lddmm_ctx* ctx, const float* dev_I0, const float* dev_I1);

/* TimeVaryingVelocity<BandVectorField> storage (core.hpp:275-317) as device buffers */
long long lddmm_velocity_doubles(const lddmm_ctx* ctx); /* doubles per velocity (re/im counted) */
int lddmm_vel_alloc(lddmm_ctx* ctx, double** dev_v);    /* zero-initialised (Model::zero_velocity) */
int lddmm_vel_free(lddmm_ctx* ctx, double* dev_v);
int lddmm_vel_upload(lddmm_ctx* ctx, double* dev_v, const double* host_v);
int lddmm_vel_download(lddmm_ctx* ctx, const double* dev_v, double* host_v);
/* tv_axpy / tv_scaled / tv_inner / tv_linf / tv_all_finite (variants.hpp:70-117) */
int lddmm_vel_axpy(lddmm_ctx* ctx, double a, const double* dev_x, const double* dev_y, double* dev_out);
int lddmm_vel_scale(lddmm_ctx* ctx, const double* dev_x, double a, double* dev_out);
int lddmm_vel_inner(lddmm_ctx* ctx, const double* dev_x, const double* dev_y, double* out);
int lddmm_vel_linf(lddmm_ctx* ctx, const double* dev_x, double* out);
int lddmm_vel_all_finite(lddmm_ctx* ctx, const double* dev_x, int* out);

/* Model::forward(v, with_adjoint) (variants.hpp:262-276); keeps the cache in ctx */
int lddmm_forward(lddmm_ctx* ctx, const double* dev_v, int with_adjoint, lddmm_energies* out, int* step);
/* Model::energy(v) (variants.hpp:278); does not disturb the cache */
int lddmm_energy(lddmm_ctx* ctx, const double* dev_v, double* energy, int* step);
/* Model::gradient(cache) (variants.hpp:291-309) */
int lddmm_gradient(lddmm_ctx* ctx, double* dev_out);
/* Model::hessvec(cache, dv) (variants.hpp:313-344) */
int lddmm_hessvec(lddmm_ctx* ctx, const double* dev_dv, double* dev_out, int* step);
/* Model::precondition(g) (variants.hpp:347-353) */
int lddmm_precondition(lddmm_ctx* ctx, const double* dev_in, double* dev_out);
/* ForwardCache::m1 / residual (variants.hpp:200-201) as host fp64 (either may be NULL) */
int lddmm_get_fields(lddmm_ctx* ctx, double* host_m1, double* host_residual);
/* cached grid field as host fp64 [N]: 0 m1, 1 residual, 2-4 grad_src_warped (variants.hpp:220),
 * 5 I0 spline coefficients, 6-8 spline coefficients of spectral_gradient(I0), 9 I1 */
int lddmm_get_grid(lddmm_ctx* ctx, int which, double* host_out);
/* 0: u series, 1: rho series (nt+1 band vectors), host fp64 (ForwardCache::u / rho) */
int lddmm_get_series(lddmm_ctx* ctx, int which, double* host_out);

/* optimize(model, v0, opt) (optimizer.hpp:143-262): dev_v is v0 on entry and the
 * result velocity on exit.  history may be NULL. */
int lddmm_optimize(lddmm_ctx* ctx, double* dev_v, const lddmm_options* opt, lddmm_iteration_record* history,
                   int history_cap, lddmm_result* result);

/* End-to-end call from host buffers (lddmm_cli.cpp:101-125 run_registration):
 * images in, zero velocity, optimize, velocity out (host_v may be NULL). */
int lddmm_register(lddmm_ctx* ctx, const double* host_I0, const double* host_I1, const lddmm_options* opt,
                   double* host_v, lddmm_iteration_record* history, int history_cap, lddmm_result* result);

/* compute_maps + map_jacobian_determinant + value_range (metrics.hpp:24-79):
 * jac = {fwd min, fwd max, inv min, inv max}; displacement outputs host fp64
 * [3][N] (either may be NULL). */
int lddmm_maps(lddmm_ctx* ctx, const double* dev_v, double* host_disp_fwd, double* host_disp_inv,
               double jac[4]);

/* ---- primitives on device buffers (parity tests; fp64 band, fp32 grid) ---- */
/* embed (spectral.hpp:262-285); prefilter != 0 returns the cubic spline
 * coefficients of the embedded field (spline_coefficients, interp.hpp:80-84) */
int lddmm_op_embed(lddmm_ctx* ctx, const double* dev_band, int ncomp, float* dev_grid, int prefilter);
/* project (spectral.hpp:242-260) */
int lddmm_op_project(lddmm_ctx* ctx, const float* dev_grid, int ncomp, double* dev_band);
/* advect_state (transport.hpp:67-73) at departure displacements dev_dep [3][N]
 * (grid units: X = x + dep * h) */
int lddmm_op_advect(lddmm_ctx* ctx, const double* dev_band, int ncomp, const float* dev_dep, double* dev_out);
/* VelocityProvider::departure fwd/bwd + cfl (transport.hpp:83-102,176-194), stationary v */
int lddmm_op_departure(lddmm_ctx* ctx, const double* dev_v, float* dev_dep_fwd, float* dev_dep_bwd, double* cfl);
/* truncated products (spectral.hpp:460-510): op 0 star(s,s) 1 star(s,vec)
 * 2 star_dot 3 band_jac_mul 4 band_jacT_mul ; 5 band_divergence(vec) */
int lddmm_op_band(lddmm_ctx* ctx, int op, const double* dev_a, const double* dev_b, double* dev_out);
/* the SL cubic gather alone (ScalarSampler::eval_cubic at departure points, interp.hpp:119-159):
 * dev_coef [ncomp][N] spline coefficients, dev_dep [3][N] grid-unit displacements;
 * impl 0 production (marching window), 1 smem-tiled, 2 global-memory, 3 8x4-tile register window
 * (the pull-back path); all bitwise equal */
int lddmm_op_gather(lddmm_ctx* ctx, int impl, const float* dev_coef, int ncomp, const float* dev_dep,
                    float* dev_out);
/* cubic pull-back of grid scalar fields through x - disp (warp with
 * points_from_displacement, interp.hpp:178-210, variants.hpp:49-51); disp phys units */
int lddmm_op_warp(lddmm_ctx* ctx, const float* dev_field, int ncomp, const float* dev_disp, float* dev_out);

/* ---- evaluation path (metrics.hpp:24-131, interp.hpp:178-225) ---- */
/* Interp (interp.hpp:14) plus the nearest-neighbour label warp */
enum { LDDMM_INTERP_LINEAR = 0, LDDMM_INTERP_CUBIC = 1, LDDMM_INTERP_NEAREST = 2 };
/* warp_nearest(f, x - disp) (interp.hpp:213-225) on device fp32 buffers, disp phys units */
int lddmm_op_warp_nearest(lddmm_ctx* ctx, const float* dev_field, int ncomp, const float* dev_disp, float* dev_out);
/* map_jacobian_determinant + value_range (metrics.hpp:40-79) of a device grid displacement
 * [3][N] (phys units); full-grid spectral derivatives in fp64; dev_det may be NULL */
int lddmm_op_jacobian(lddmm_ctx* ctx, const float* dev_disp, float* dev_det, double minmax[2]);
/* mean_dice (metrics.hpp:92-131) of two device label fields: inventory = distinct nonzero
 * values of dev_target, exact integer counts on the device */
int lddmm_op_mean_dice(lddmm_ctx* ctx, const float* dev_warped, const float* dev_target, double* out);

/* Host-buffer forms (fp64, ScalarField / VectorField layouts) used by the CLI
 * (lddmm_cli.cpp:101-235).  warp: kind LDDMM_INTERP_CUBIC (warp, interp.hpp:178-210)
 * or LDDMM_INTERP_NEAREST; ncomp fields of N; disp [3][N] phys units. */
int lddmm_warp(lddmm_ctx* ctx, int kind, const double* host_field, int ncomp, const double* host_disp,
               double* host_out);
int lddmm_jacobian(lddmm_ctx* ctx, const double* host_disp, double* host_det, double minmax[2]);
int lddmm_mean_dice(lddmm_ctx* ctx, const double* host_warped, const double* host_target, double* out);
/* Alg::from_spatial (= project) of a host vector field into every node of dev_v (--v0,
 * lddmm_cli.cpp:111-117); Alg::to_spatial (= embed) of node `node` to a host vector field */
int lddmm_vel_from_spatial(lddmm_ctx* ctx, const double* host_vec, double* dev_v);
int lddmm_vel_to_spatial(lddmm_ctx* ctx, const double* dev_v, int node, double* host_vec);

#ifdef __cplusplus
}
#endif

#endif /* LDDMM_CUDA_H */
