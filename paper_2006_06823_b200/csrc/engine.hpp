// Device-resident band-limited SL-LDDMM model (the reference's Model<BandAlgebra>
// with the semi-Lagrangian integrator, variants.hpp:229-548) for one
// registration on one B200.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace lddmm_b200 {

struct Problem {
  int dims[3];
  double spacing[3];
  int band[3];
  int nt = 5;
  int variant = 2;     // 0 original, 1 state_equation, 2 deformation_state_equation (variants.hpp:34)
  int stationary = 1;  // Parameterization (core.hpp:271)
  int rk4 = 0;         // Integrator: 0 SL-RK2, 1 RK4 (variants.hpp:35,241)
  double alpha = 0.0025;
  int s = 2;
  double sigma2 = 1.0;
  // 2-D problems (core.hpp:49-52 allows d = 2) run as 3-D problems with the z axis
  // replicated zrep times at spacing 1/zrep: every field is z-constant, only the kz = 0
  // band plane is non-zero, and all reference quantities (inner products, energies,
  // Jacobians) are exactly the 2-D ones; d sets which axes enter h_min (cfl) and
  // zrep rescales the band coefficients' max norm (the 3-D coefficients are zrep times
  // the 2-D ones).
  int d = 3;
  int zrep = 1;
};

struct Energies {
  double energy = 0, energy_reg = 0, energy_data = 0, cfl = 0;
};

// LDDMM_POISON=1: fill every new device buffer with NaNs, so reads of memory
// no kernel wrote show up deterministically (debug aid; off by default).
inline bool poison_allocations() {
  static const int v = [] {
    const char* e = std::getenv("LDDMM_POISON");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      LDDMM_CUDA(cudaMalloc(&p, count * sizeof(T)));
      if (poison_allocations()) LDDMM_CUDA(cudaMemset(p, 0xff, count * sizeof(T)));  // NaN fill (debug)
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  T* get() const { return p; }
  operator T*() const { return p; }
};

// Provider state for one velocity (VelocityProvider, transport.hpp:109-218),
// stationary: one slot.
struct ProviderState {
  DevBuf<double2> v;     // band velocity copy [3][Kprod]
  DevBuf<double2> div;   // band divergence [Kprod]
  DevBuf<float> dep_fwd; // departure displacement, grid units [3][N]
  DevBuf<float> dep_bwd;
  double cfl = 0;
  bool has_bwd = false;
};

class Engine {
 public:
  Engine(const Problem& p, int device);
  ~Engine();

  const Problem& problem() const { return prob_; }
  int nodes() const { return prob_.stationary ? 1 : prob_.nt + 1; }
  long long kprod() const { return full_.kprod(); }
  long long npts() const { return full_.npts(); }
  long long vec_elems() const { return 3 * kprod(); }          // one band vector (double2 count)
  long long vel_elems() const { return nodes() * vec_elems(); }  // one velocity
  cudaStream_t stream() const { return stream_; }
  int device() const { return device_; }
  const int* small_dims() const { return small_.N; }

  // images (reference ScalarField layout, fp64 host or fp32 device)
  void set_images_host(const double* I0, const double* I1);
  void set_images_device_f32(const float* I0, const float* I1);

  // ---- Model API (variants.hpp:262-353) ----
  Energies forward(const double2* v, bool with_adjoint);
  double energy(const double2* v);  // forward(v, false).energy on a separate trial state
  void gradient(double2* out);
  void hessvec(const double2* dv, double2* out);
  void precondition(const double2* in, double2* out);
  double reg_energy(const double2* v);
  const float* m1() const { return m1_.p; }
  const float* residual() const { return res_.p; }
  // cached grid fields: 0 m1, 1 residual, 2-4 grad_src_warped, 5 I0 spline coefficients,
  // 6-8 grad I0 spline coefficients, 9 I1
  const float* grid_field(int which) const {
    const long long N = npts();
    if (which == 0) return m1_.p;
    if (which == 1) return res_.p;
    if (which >= 2 && which <= 4) return m1_.p + (which - 1) * N;
    if (which >= 5 && which <= 8) return I0coef_.p + (which - 5) * N;
    if (which == 9) return I1_.p;
    return nullptr;
  }
  double residual_sumsq();
  double mse_denominator();  // l2_inner(I0 - I1, I0 - I1)

  // ---- TimeVaryingVelocity algebra (variants.hpp:65-117) ----
  void tv_axpy(double a, const double2* x, const double2* y, double2* out);
  void tv_scaled(const double2* x, double a, double2* out);
  double tv_inner(const double2* a, const double2* b);
  double tv_linf(const double2* a);
  bool tv_all_finite(const double2* a);

  // ---- primitives (parity tests / tools) ----
  void embed(const double2* c, int ncomp, float* out, bool prefilter = false);  // full grid
  void project(const float* f, int ncomp, double2* out);
  void advect(const double2* q, int ncomp, const float* dep, double2* out);
  void departure(const double2* v, float* dep_fwd, float* dep_bwd, double* cfl);
  void star_sv(const double2* s, const double2* x, double2* out, double alpha);
  void star_ss(const double2* a, const double2* b, double2* out, double alpha);
  void star_dot(const double2* a, const double2* b, double2* out, double alpha);
  void jac_mul(const double2* u, const double2* w, double2* out, double alpha, bool transpose);
  void band_divergence(const double2* v, double2* out);
  // cubic pull-back of grid fields (ncomp <= 6) through x - disp_phys (warp, interp.hpp:178-210)
  void warp_grid(const float* f, int ncomp, const float* disp_phys, float* out);
  // endpoint maps and Jacobian ranges (metrics.hpp:24-65); disp outputs optional (device, [3][N] fp32)
  void maps(const double2* v, float* disp_fwd, float* disp_inv, double jac[4]);
  // ---- evaluation path (metrics.hpp:40-131, interp.hpp:213-225) ----
  // nearest-neighbour pull-back of grid fields (labels) through x - disp_phys
  void warp_nearest(const float* f, int ncomp, const float* disp_phys, float* out);
  // det(I - Du) of a grid displacement [3][N] (phys units), full-grid spectral
  // derivatives in fp64; det optional (device fp32 [N]); mm = {min, max}
  void jacobian_grid(const float* disp_phys, float* det, double mm[2]);
  // Dice counts of `nl` label values: counts[3*l + {0,1,2}] = |a=l|, |b=l|, |a=l & b=l|
  void dice_counts(const float* a, const float* b, const float* labels, int nl, unsigned long long* counts);
  void series(int which, double2* out);  // 0 u, 1 rho (nt+1 band vectors)

  // counters (kernel launches issued by this engine)
  long long launches() const { return launches_; }
  void sync();
  double2* opt_ws(int i) const { return opt_ws_.p + (long long)i * vel_elems(); }

  // Live per-launch timing of the SL gather kernel (CUDA events on the engine
  // stream around every gather launch while enabled).  stats: total device ms,
  // launch count, algorithmic bytes N * (12 + 8 C) summed over launches.
  void set_gather_timing(int mode);  // bit 0 gathers, bit 1 full-grid DFTs
  void gather_stats(double* ms, long long* launches, double* bytes);
  // kind 0: SL gathers (amount = algorithmic bytes), 1: full-grid truncated DFTs (flops)
  void timing_stats(int kind, double* ms, long long* launches, double* amount);
  double dft_flops_per_field() const;

 private:
  Problem prob_;
  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  long long launches_ = 0;
  double h_[3];
  double cell_volume_ = 1;
  double small_ratio_ = 1;  // M / N (total points) for the small product grid

  DftPlan full_, small_;
  std::vector<void*> plan_allocs_;

  // images
  DevBuf<float> I1_, I0coef_, gI0coef_;  // I0 spline coefficients, grad I0 spline coefficients [3][N]
  DevBuf<float> I0f_;                    // I0 values (fp32) for mse denominators
  double mse_denom_ = -1;

  // scratch: full-grid DFT
  int fmax_full_ = 6, fmax_small_ = 12;
  DevBuf<float2> D_, E1_, E2_, G1_, G2_, G3_;
  DevBuf<float> gridA_, gridB_;  // [fmax][N]
  // scratch: small grid
  DevBuf<float2> sD_, sE1_, sE2_, sG1_, sG2_, sG3_;
  DevBuf<float> sgrid_, sacc_;  // [12][M], [3][M]

  // reductions
  DevBuf<double> part_, part2_, slots_;
  double* host_slots_ = nullptr;

  // forward cache (variants.hpp:188-224, deformation variant fields)
  ProviderState prov_, trial_prov_;
  bool have_cache_ = false, cache_adjoint_ = false;
  Energies cache_e_;
  DevBuf<double2> u_, rho_;   // (nt+1) x 3 x Kprod
  DevBuf<double2> tmp_u_;     // trial u running state [2][3][Kprod]
  DevBuf<float> m1_, res_, gsw_, ugrid_;  // m1, residual [N], grad_src_warped [3][N], u(1) embed [3][N]
  DevBuf<float> trial_m1_, trial_res_;
  // trial-state reuse (stationary SL, all variants): the last energy() keeps its u (or
  // image) series; a forward() at the bitwise-same velocity adopts it
  DevBuf<double2> trial_u_, trial_mser_;
  bool trial_valid_ = false;
  bool trial_reuse_ok() const { return prob_.stationary && !prob_.rk4 && std::getenv("LDDMM_NO_TRIAL_REUSE") == nullptr; }
  bool same_velocity(const double2* a, const double2* b);
  void adopt_trial_provider(bool with_bwd);
  DevBuf<double2> btmp_;      // band temporaries: 12 band vectors
  DevBuf<double2> src_;       // (nt+1) band vectors (incremental sources)
  DevBuf<double2> dseries_;   // (nt+1) band vectors (hessvec du / drho series)
  // original / state_equation caches (variants.hpp:203-217), allocated on first use
  DevBuf<double2> m_ser_;     // image state m_i (original) / reconstructed m_i (state), band scalars
  DevBuf<double2> lam_ser_;   // lambda_i (original) / lambda nodes (state), band scalars
  DevBuf<double2> dm_ser_;    // hessvec incremental scalar series (dm, dlambda)
  DevBuf<double2> nu_ser_;    // state: nu series (band vectors)
  DevBuf<double2> bigU_ser_;  // state: U series (band scalars)
  DevBuf<float> jac_f_;       // state: J_i = 1 - iota(U_i), [nt+1][N]
  DevBuf<float> psi_f_;       // state: iota(nu_i) displacement, [nt+1][3][N]
  DevBuf<float> fgI0coef_;    // state: spline coefficients of filtered_gradient(I0), [3][N]
  DevBuf<float> lcoef_;       // state: spline coefficients of lambda1 / dlambda1, [N]
  DevBuf<double2> m0_;        // original: pi(I0)
  DevBuf<double> f64a_, f64b_, f64c_, dker_;  // fp64 grid scratch (image constants), derivative kernels
  bool dker_ready_ = false;
  void ensure_dker();  // per-axis circulant spectral-derivative kernels (spectral.hpp:326-370)
  DevBuf<float> maps_du_;     // 9 derivative fields for the Jacobian (allocated on first use)
 public:
  // velocity of lddmm_register (host-buffer path), allocated on first use and reused
  double2* register_velocity() {
    if (!reg_v_.p) reg_v_.alloc(vel_elems());
    return reg_v_.p;
  }

 private:
  DevBuf<double2> reg_v_;
  DevBuf<double2> opt_ws_;    // optimizer workspace: 9 velocities

  void build_plan(DftPlan& p, const int* Ngrid, const int* K, const double* parent_wunit);
  void free_plans();
  double2* bt(int i) const { return btmp_.p + (long long)i * vec_elems(); }
  // per-node / per-step views (stationary: one slot, transport.hpp:124-130)
  const float* depf(const ProviderState& ps, int step) const {
    return ps.dep_fwd.p + (prob_.stationary ? 0 : (long long)step * 3 * npts());
  }
  const float* depb(const ProviderState& ps, int step) const {
    return ps.dep_bwd.p + (prob_.stationary ? 0 : (long long)step * 3 * npts());
  }
  const double2* vnode(const ProviderState& ps, int i) const {
    return ps.v.p + (prob_.stationary ? 0 : (long long)i * vec_elems());
  }
  const double2* divnode(const ProviderState& ps, int i) const {
    return ps.div.p + (prob_.stationary ? 0 : (long long)i * kprod());
  }
  const double2* tvnode(const double2* tv, int i) const {  // tv_node (variants.hpp:65-68)
    return tv + (prob_.stationary ? 0 : (long long)i * vec_elems());
  }
  DevBuf<float> pscratch_;  // nonstationary provider scratch [9][N]
  double2* node(DevBuf<double2>& s, int i) const { return s.p + (long long)i * vec_elems(); }

  void provider_build(const double2* v, ProviderState& ps, bool with_bwd);
  // ---- RK4 integrator (transport.hpp:234-258), band representation (rk4.cu) ----
  using RkRhs = std::function<void(const double2* q, double t, double2* out)>;
  void rk4_run(long long C, const double2* init, double2* series, double2* last, bool forward, const RkRhs& rhs);
  const double2* rk_vel_at(const ProviderState& ps, double t, double2* scratch);
  const double2* rk_div_at(const ProviderState& ps, double t, double2* scratch);
  const double2* rk_tv_at(const double2* tv, double t, double2* scratch);
  const double2* rk_series_at(const double2* series, long long C, double t, double2* scratch);
  void graddot(const double2* q, const double2* w, double2* out, double alpha, const double2* add, double beta);
  double2* rk(int i) const { return rk_.p + (long long)i * vec_elems(); }
  DevBuf<double2> rk_;  // RK4 stages and samples: 12 band vectors
  void enqueue_finite(const double2* p, long long n, int step);
  void rk4_displacement(ProviderState& ps, bool forward, double2* series, double2* last);
  void rk4_vector_continuity_bwd(ProviderState& ps, const double2* q1, double2* series);
  void rk4_incremental_displacement(ProviderState& ps, const double2* dv, double2* series);
  void rk4_image_forward(ProviderState& ps, const double2* m0, double2* series, double2* last);
  void rk4_scalar_continuity_bwd(ProviderState& ps, const double2* q1, double2* series, bool jf);
  void rk4_incremental_image(ProviderState& ps, const double2* dv, double2* series);
  void solve_displacement_fwd(ProviderState& ps, double2* series, bool keep_all, double2* last);
  void solve_vector_continuity_bwd(ProviderState& ps, const double2* q1, double2* series);
  void solve_incremental_displacement(ProviderState& ps, const double2* dv, double2* series);
  void warp_m1(const double2* u1, float* m1, float* res, bool want_gsw, double* data_sumsq);
  // variants.cu: original and state_equation (variants.hpp:373-422,444-527)
  void ensure_variant_buffers();
  void solve_displacement(ProviderState& ps, bool forward, double2* series);
  void solve_image_forward(ProviderState& ps, const double2* m0, double2* series, bool keep_all, double2* last);
  void solve_scalar_continuity_bwd(ProviderState& ps, const double2* q1, double2* series, bool jacobian_factor);
  void solve_incremental_image(ProviderState& ps, const double2* dv, double2* series);
  void small_custom(const PrepArgs& pa, int prodop, double2* out, int nout, double alpha, const double2* add,
                    double beta);
  void assemble_star_grad(const double2* Lam, const double2* Mser, const double2* like, double2* out);
  void grid_spline(const float* f, float* coef);
  void lambda_nodes_state(const float* lam1, double2* out_series);
  double forward_original(bool with_adjoint, const double2* v, bool have_m = false);
  double forward_state(bool with_adjoint, bool have_u = false);
  double energy_original(const double2* v);
  void hessvec_original(const double2* dv, double2* out);
  void hessvec_state(const double2* dv, double2* out);
  void assemble_jacT_terms(const double2* series_u, const double2* series_q, const double2* like,
                           double2* out);
  void check_series_finite(const double2* series, int count, int first_step_offset, bool backward);
  void enqueue_finite_check(const double2* node, int step);
  void finish_finite_checks(int nsteps);
  void set_images_impl(const double* I0d);

  // generic pipelines
  void embed_fields(const DftPlan& p, const PrepArgs& a, float* out, float2* D, float2* E1, float2* E2);
  void project_fields(const DftPlan& p, const float* f, const FinArgs& a, float2* G1, float2* G2, float2* G3);
  void advect_multi(const double2* const* in, int nf, const float* dep, const FinField* outs);
  void small_product(int op, const double2* a, const double2* b, double2* out, double alpha,
                     const double2* add, double beta);

  double reduce(int nparts, int op);
  void timed_gather(const float* coef, int ncomp, const float* dep, float* out);

  int gt_on_ = 0;
  bool pullback_large_ = false;  // set by provider_build: whole-map pull-backs exceed a voxel
  std::vector<cudaEvent_t> gt_events_;
  std::vector<double> gt_bytes_;
  std::vector<int> gt_kind_;
  void timing_begin();
  void timing_end(int kind, double amount);
  size_t gt_used_ = 0;
  void count(int n = 1) { launches_ += n; }
};

}  // namespace lddmm_b200
