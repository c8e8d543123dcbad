// Device orchestration of the band-limited SL-RK2 model (deformation-state
// variant), restating variants.hpp / transport.hpp on top of the kernels.
//
// Exact algebraic levers used (each exact in real arithmetic):
//  * prefilter = 1/B(k) in band: spline coefficients of embed(q) are
//    embed(q / B) (interp.hpp:23-63 vs a diagonal symbol), fused into the
//    embed prep;
//  * small product grid: every truncated product of two band fields
//    (star, star_dot, band_jac(T)_mul, spectral.hpp:460-510) is alias-free on
//    an M grid with M_a >= 3K_a/2 - 2 and equals (M/N) * pi_M(iota_M a * iota_M b);
//    when the parent grid itself aliases (N_a < 3K_a/2 - 2) M_a = N_a;
//  * stationary invariants: departure points and advect(v) are step-invariant
//    (transport.hpp:178, variants.hpp:471);
//  * merged advects for q-independent sources (incremental displacement):
//    advect(q) + dt/2 advect(src) = advect(q + dt/2 src);
//  * linear assembly: sum_i w_i jacT(u_i, q_i) is accumulated on the small grid
//    and projected once;
//  * hoisting: I0 and grad I0 spline coefficients are per-registration constants.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"

namespace lddmm_b200 {

namespace {

int small_dim(int N, int K) {
  int m = (3 * K) / 2 - 2;
  if (m % 2) ++m;
  if (m < K) m = K;
  if (N < m) return N;  // the parent grid aliases; reproduce it exactly
  return m;
}

std::vector<double> trapezoid_weights(int nt) {  // variants.hpp:40-46
  std::vector<double> w(nt + 1, 1.0 / nt);
  w.front() *= 0.5;
  w.back() *= 0.5;
  return w;
}

}  // namespace

Engine::Engine(const Problem& p, int device) : prob_(p), device_(device) {
  for (int a = 0; a < 3; ++a) {
    shape_require(p.dims[a] >= 4 && p.dims[a] % 2 == 0, "grid dims must be even and >= 4");
    shape_require(p.spacing[a] > 0.0, "grid spacing must be positive");
    shape_require(p.band[a] % 2 == 0 && p.band[a] >= 4 && p.band[a] <= p.dims[a],
                  "band bounds must be even and in [4, dims]");
  }
  shape_require(p.nt >= 1, "nt must be >= 1");
  shape_require(p.alpha > 0.0 && p.s >= 1, "sobolev: alpha > 0 and s >= 1 required");
  shape_require(p.variant >= 0 && p.variant <= 2, "unknown variant");
  shape_require(!p.rk4 || p.nt >= 2, "rk4 requires nt >= 2");
  LDDMM_CUDA(cudaSetDevice(device));
  // A blocking stream: it is ordered against the legacy default stream, so device
  // buffers a caller fills or allocates there (torch tensors, cudaMemset) are
  // complete before the engine reads them, and a caller's later default-stream
  // work waits for the engine's writes.
  LDDMM_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamDefault));
  double wunit[3];
  cell_volume_ = 1.0;
  for (int a = 0; a < 3; ++a) {
    h_[a] = p.spacing[a];
    wunit[a] = 2.0 * M_PI / (p.dims[a] * p.spacing[a]);
    cell_volume_ *= p.spacing[a];
  }
  build_plan(full_, p.dims, p.band, wunit);
  int M[3];
  for (int a = 0; a < 3; ++a) M[a] = small_dim(p.dims[a], p.band[a]);
  build_plan(small_, M, p.band, wunit);
  small_ratio_ = (double)small_.npts() / (double)full_.npts();

  const long long N = full_.npts(), Kx = p.band[0], H = p.band[2] / 2;
  const int Nx = p.dims[0], Ny = p.dims[1];
  D_.alloc(fmax_full_ * full_.half());
  E1_.alloc(fmax_full_ * Kx * Ny * H);
  E2_.alloc(fmax_full_ * (long long)Nx * Ny * H);
  G1_.alloc(fmax_full_ * (long long)Nx * Ny * H);
  G2_.alloc(fmax_full_ * Kx * Ny * H);
  G3_.alloc(fmax_full_ * full_.half());
  gridA_.alloc(fmax_full_ * N);
  gridB_.alloc(fmax_full_ * N);

  fmax_small_ = 60;
  const long long Ms = small_.npts();
  sD_.alloc(fmax_small_ * small_.half());
  sE1_.alloc(fmax_small_ * Kx * small_.N[1] * H);
  sE2_.alloc(fmax_small_ * (long long)small_.N[0] * small_.N[1] * H);
  sG1_.alloc(fmax_small_ * (long long)small_.N[0] * small_.N[1] * H);
  sG2_.alloc(fmax_small_ * Kx * small_.N[1] * H);
  sG3_.alloc(fmax_small_ * small_.half());
  sgrid_.alloc(fmax_small_ * Ms);
  sacc_.alloc(fmax_small_ * Ms);

  part_.alloc(kReduceBlocks);
  part2_.alloc(kReduceBlocks + 1);  // + the counter of launch_nonfinite_flag
  LDDMM_CUDA(cudaMemset(part2_.p, 0, (kReduceBlocks + 1) * sizeof(double)));
  // 16 scalar slots, then one per time step / node (cfl per node, non-finite flag per step)
  slots_.alloc(16 + p.nt + 1);
  LDDMM_CUDA(cudaMallocHost(&host_slots_, (16 + p.nt + 1) * sizeof(double)));

  const long long V = vec_elems();
  const int nsteps = p.stationary ? 1 : p.nt;  // departure slots per direction
  for (ProviderState* ps : {&prov_, &trial_prov_}) {
    ps->v.alloc(nodes() * V);
    ps->div.alloc(nodes() * kprod());
    if (!p.rk4) ps->dep_fwd.alloc(nsteps * 3 * N);  // RK4 never samples departure points
  }
  if (!p.rk4) prov_.dep_bwd.alloc(nsteps * 3 * N);
  if (!p.stationary) pscratch_.alloc(9 * N);
  u_.alloc((p.nt + 1) * V);
  rho_.alloc((p.nt + 1) * V);
  src_.alloc((p.nt + 1) * V);
  dseries_.alloc((p.nt + 1) * V);
  tmp_u_.alloc(2 * V);
  btmp_.alloc(12 * V);
  if (p.rk4) rk_.alloc(12 * V);
  m1_.alloc(4 * N);  // m1 followed by grad_src_warped [3][N]
  res_.alloc(N);
  ugrid_.alloc(3 * N);
  trial_m1_.alloc(N);
  trial_res_.alloc(N);
  if (trial_reuse_ok() && p.variant != 0) trial_u_.alloc((p.nt + 1) * V);
  I1_.alloc(N);
  I0f_.alloc(N);
  I0coef_.alloc(4 * N);  // I0 spline coefficients followed by grad I0 spline coefficients
  f64a_.alloc(N);
  f64b_.alloc(N);
  f64c_.alloc(N);
  dker_.alloc(3 * 1024);
  shape_require(p.dims[0] <= 1024 && p.dims[1] <= 1024 && p.dims[2] <= 1024, "grid dims must be <= 1024");
  opt_ws_.alloc(9 * vel_elems());
  if (p.variant == 0) m0_.alloc(kprod());
  ensure_variant_buffers();
}

Engine::~Engine() {
  for (cudaEvent_t e : gt_events_) cudaEventDestroy(e);
  free_plans();
  if (host_slots_) cudaFreeHost(host_slots_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::free_plans() {
  for (void* q : plan_allocs_) cudaFree(q);
  plan_allocs_.clear();
}

void Engine::sync() { LDDMM_CUDA(cudaStreamSynchronize(stream_)); }

// Twiddle tables in fp64 (exact integer phase reduction), rounded to fp32.
void Engine::build_plan(DftPlan& p, const int* Ng, const int* K, const double* wunit) {
  for (int a = 0; a < 3; ++a) {
    p.N[a] = Ng[a];
    p.K[a] = K[a];
    p.omega_unit[a] = wunit[a];
  }
  const int Nx = Ng[0], Ny = Ng[1], Nz = Ng[2], Kx = K[0], Ky = K[1], H = K[2] / 2;
  const double Ntot = (double)Nx * Ny * Nz;
  auto sf = [](int f, int Kb) { return f < Kb / 2 ? f : f - Kb; };
  auto ang = [](long long k, long long x, long long n) {
    long long r = ((k * x) % n + n) % n;
    return 2.0 * M_PI * (double)r / (double)n;
  };
  auto upload = [&](const void* host, size_t bytes) {
    void* d = nullptr;
    LDDMM_CUDA(cudaMalloc(&d, bytes));
    LDDMM_CUDA(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice));
    plan_allocs_.push_back(d);
    return d;
  };
  std::vector<float2> wy_e((size_t)Ny * Ky), wx_e((size_t)Nx * Kx), wx_p((size_t)Kx * Nx), wy_p((size_t)Ky * Ny);
  for (int y = 0; y < Ny; ++y)
    for (int f = 0; f < Ky; ++f) {
      const double t = ang(sf(f, Ky), y, Ny);
      wy_e[(size_t)y * Ky + f] = make_float2((float)cos(t), (float)sin(t));
      wy_p[(size_t)f * Ny + y] = make_float2((float)cos(t), (float)-sin(t));
    }
  for (int x = 0; x < Nx; ++x)
    for (int f = 0; f < Kx; ++f) {
      const double t = ang(sf(f, Kx), x, Nx);
      wx_e[(size_t)x * Kx + f] = make_float2((float)cos(t), (float)sin(t));
      wx_p[(size_t)f * Nx + x] = make_float2((float)cos(t), (float)-sin(t));
    }
  std::vector<float> tz_e((size_t)2 * H * Nz), tz_p((size_t)Nz * 2 * H);
  for (int kz = 0; kz < H; ++kz)
    for (int z = 0; z < Nz; ++z) {
      const double t = ang(kz, z, Nz);
      tz_e[(size_t)(2 * kz) * Nz + z] = (float)(cos(t) / Ntot);
      tz_e[(size_t)(2 * kz + 1) * Nz + z] = (float)(-sin(t) / Ntot);
      tz_p[(size_t)z * 2 * H + 2 * kz] = (float)cos(t);
      tz_p[(size_t)z * 2 * H + 2 * kz + 1] = (float)-sin(t);
    }
  p.wy_e = (float2*)upload(wy_e.data(), wy_e.size() * sizeof(float2));
  p.wx_e = (float2*)upload(wx_e.data(), wx_e.size() * sizeof(float2));
  p.wx_p = (float2*)upload(wx_p.data(), wx_p.size() * sizeof(float2));
  p.wy_p = (float2*)upload(wy_p.data(), wy_p.size() * sizeof(float2));
  p.tz_e = (float*)upload(tz_e.data(), tz_e.size() * sizeof(float));
  p.tz_p = (float*)upload(tz_p.data(), tz_p.size() * sizeof(float));
  auto alloc = [&](size_t n) {
    void* d = nullptr;
    LDDMM_CUDA(cudaMalloc(&d, n * sizeof(float)));
    plan_allocs_.push_back(d);
    return (float*)d;
  };
  {
    void* d = nullptr;
    LDDMM_CUDA(cudaMalloc(&d, (size_t)(Kx + Ky + K[2]) * sizeof(double)));
    plan_allocs_.push_back(d);
    p.bsym = (double*)d;
    launch_band_symbols(K, Ng, p.bsym, stream_);
  }
  p.tz_e_big = alloc(tz_e.size());
  p.tz_e_small = alloc(tz_e.size());
  p.tz_p_big = alloc(tz_p.size());
  p.tz_p_small = alloc(tz_p.size());
  launch_tf32_split(p.tz_e, p.tz_e_big, p.tz_e_small, (long long)tz_e.size(), stream_);
  launch_tf32_split(p.tz_p, p.tz_p_big, p.tz_p_small, (long long)tz_p.size(), stream_);
  if (umma_zproject_fits(Nz, 2 * H)) {
    const size_t nc = (size_t)2 * H * umma_zproject_kpad(Nz);
    p.uz_p_big = alloc(nc);
    p.uz_p_small = alloc(nc);
    launch_umma_zproj_prep(p.tz_p_big, p.tz_p_small, Nz, 2 * H, p.uz_p_big, p.uz_p_small, stream_);
  }
  // x stage on tcgen05 (twiddles as the canonical K-major operand) where the plan fits and
  // a field has enough 128-column tiles (2 Ny H >= 4096: config 2's full grid, config 4's
  // 94^3 product grid); narrower transforms (config 2's 46^3 product grid) are
  // launch-latency-bound and stay on FFMA
  const bool narrow = 2LL * Ny * H < 4096 && !std::getenv("LDDMM_UMMA_X_SMALL");
  if (!narrow && !(std::getenv("LDDMM_UMMA_X") && std::getenv("LDDMM_UMMA_X")[0] == '0')) {
    std::vector<float> tw;
    if (umma_xstage_fits(Nx, Kx, Ny * H)) {
      umma_xstage_twiddles_host(wx_e.data(), Nx, Kx, tw);
      p.ux_e = (float*)upload(tw.data(), tw.size() * sizeof(float));
    }
    if (umma_xstage_fits(Kx, Nx, Ny * H)) {
      umma_xstage_twiddles_host(wx_p.data(), Kx, Nx, tw);
      p.ux_p = (float*)upload(tw.data(), tw.size() * sizeof(float));
    }
  }
  if (umma_zembed_fits(Nz, 2 * H)) {
    const size_t nc = (size_t)umma_padded_n(Nz) * 2 * H;
    p.uz_e_big = alloc(nc);
    p.uz_e_small = alloc(nc);
    launch_umma_canon_b(p.tz_e_big, p.tz_e_small, 2 * H, Nz, p.uz_e_big, p.uz_e_small, stream_);
  }
  sync();
}

void Engine::timing_begin() {
  while (gt_events_.size() < 2 * (gt_used_ + 1)) {
    cudaEvent_t ev;
    LDDMM_CUDA(cudaEventCreate(&ev));
    gt_events_.push_back(ev);
  }
  LDDMM_CUDA(cudaEventRecord(gt_events_[2 * gt_used_], stream_));
}

void Engine::timing_end(int kind, double amount) {
  LDDMM_CUDA(cudaEventRecord(gt_events_[2 * gt_used_ + 1], stream_));
  if (gt_bytes_.size() <= gt_used_) {
    gt_bytes_.resize(gt_used_ + 1);
    gt_kind_.resize(gt_used_ + 1);
  }
  gt_bytes_[gt_used_] = amount;
  gt_kind_[gt_used_] = kind;
  ++gt_used_;
}

void Engine::timed_gather(const float* coef, int ncomp, const float* dep, float* out) {
  if (!(gt_on_ & 1)) {
    launch_gather_cubic(coef, ncomp, dep, out, full_.N, stream_);
    return;
  }
  timing_begin();
  launch_gather_cubic(coef, ncomp, dep, out, full_.N, stream_);
  // algorithmic bytes N (12 + 8 C): displacement, coefficient reads, output writes
  timing_end(0, (double)npts() * (12.0 + 8.0 * ncomp));
}

// algorithmic flops of one full-grid truncated transform (half band along z): complex
// MACs (8 flop) of the y stage Kx*H*Ky*Ny and x stage Ny*H*Kx*Nx, real-complex MACs
// (4 flop) of the z stage Nx*Ny*Nz*H
double Engine::dft_flops_per_field() const {
  const double Nx = full_.N[0], Ny = full_.N[1], Nz = full_.N[2];
  const double Kx = prob_.band[0], Ky = prob_.band[1], H = prob_.band[2] / 2;
  return 8.0 * (Kx * H * Ky * Ny + Ny * H * Kx * Nx) + 4.0 * Nx * Ny * Nz * H;
}

void Engine::set_gather_timing(int mode) {
  gt_on_ = mode;
  gt_used_ = 0;
}

void Engine::timing_stats(int kind, double* ms, long long* launches, double* amount) {
  sync();
  double t = 0.0, b = 0.0;
  long long n = 0;
  for (size_t i = 0; i < gt_used_; ++i) {
    if (gt_kind_[i] != kind) continue;
    float el = 0.f;
    LDDMM_CUDA(cudaEventElapsedTime(&el, gt_events_[2 * i], gt_events_[2 * i + 1]));
    t += el;
    b += gt_bytes_[i];
    ++n;
  }
  *ms = t;
  *launches = n;
  *amount = b;
}

void Engine::gather_stats(double* ms, long long* launches, double* bytes) { timing_stats(0, ms, launches, bytes); }

double Engine::reduce(int nparts, int op) {
  launch_reduce_final(part_, nparts, op, slots_.p, stream_);
  LDDMM_CUDA(cudaMemcpyAsync(host_slots_, slots_.p, sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  return host_slots_[0];
}

// ---------------------------------------------------------------------------
// images: I0 spline coefficients (fp64 prefilter, interp.hpp:80-84) and the
// spline coefficients of the full-grid spectral gradient of I0 (spectral.hpp:356-370)

void Engine::set_images_host(const double* I0, const double* I1) {
  const long long N = npts();
  double* d0 = f64a_.p;
  double* d1 = f64b_.p;
  LDDMM_CUDA(cudaMemcpyAsync(d0, I0, N * sizeof(double), cudaMemcpyHostToDevice, stream_));
  LDDMM_CUDA(cudaMemcpyAsync(d1, I1, N * sizeof(double), cudaMemcpyHostToDevice, stream_));
  launch_f64_to_f32(N, d0, I0f_.p, stream_);
  launch_f64_to_f32(N, d1, I1_.p, stream_);
  set_images_impl(d0);
}

void Engine::set_images_device_f32(const float* I0, const float* I1) {
  const long long N = npts();
  LDDMM_CUDA(cudaMemcpyAsync(I1_.p, I1, N * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
  LDDMM_CUDA(cudaMemcpyAsync(I0f_.p, I0, N * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
  launch_f32_to_f64(N, I0, f64a_.p, stream_);
  set_images_impl(f64a_.p);
}

// I0 (fp64 on device) -> I0 spline coefficients, grad I0 spline coefficients,
// mse denominator.  I0f_ / I1_ already hold the fp32 images.
void Engine::set_images_impl(const double* I0d) {
  trial_valid_ = false;
  const long long N = npts();
  const float* I0 = I0f_.p;
  const float* I1 = I1_.p;
  // I0 spline coefficients (fp64 recursion, interp.hpp:80-84)
  double* c = f64c_.p;  // I0d is f64a_
  LDDMM_CUDA(cudaMemcpyAsync(c, I0d, N * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  launch_prefilter3d(c, full_.N, stream_);
  launch_f64_to_f32(N, c, I0coef_.p, stream_);
  // spectral_gradient(I0) (spectral.hpp:326-334,356-370) in fp64: per axis a real
  // circulant derivative kernel, then the spline prefilter.
  ensure_dker();
  for (int a = 0; a < 3; ++a) {
    double* g = f64b_.p;
    launch_circulant_axis_f64(I0d, g, dker_.p + 1024 * a, a, full_.N, stream_);
    launch_prefilter3d(g, full_.N, stream_);
    launch_f64_to_f32(N, g, I0coef_.p + (a + 1) * N, stream_);
  }
  // variant constants: m0 = pi(I0) (original, variants.hpp:374); spline coefficients of
  // filtered_gradient(I0) = iota(grad pi(I0)) (state, variants.hpp:176-178,421)
  if (prob_.variant == 0) project(I0, 1, m0_.p);
  if (prob_.variant == 1) {
    double2* pI0 = bt(11);
    project(I0, 1, pI0);
    PrepArgs pa{};
    pa.nf = 3;
    for (int a = 0; a < 3; ++a) pa.f[a] = PrepField{pI0, (SYM_DERIV_X + a) | SYM_PREFILTER, 1.0};
    embed_fields(full_, pa, fgI0coef_.p, D_.p, E1_.p, E2_.p);
  }
  // mse denominator l2_inner(I0 - I1) (optimizer.hpp:151-154)
  {
    const int g = launch_residual(N, I0, I1, gridB_.p, part_.p, stream_);
    mse_denom_ = reduce(g, 0) * cell_volume_;
  }
  have_cache_ = false;
}

double Engine::mse_denominator() { return mse_denom_; }

// ---------------------------------------------------------------------------
// generic pipelines

void Engine::embed_fields(const DftPlan& p, const PrepArgs& a, float* out, float2* D, float2* E1, float2* E2) {
  const bool timed = (gt_on_ & 2) && &p == &full_;
  if (timed) timing_begin();
  dft_embed_prep(p, a, D, E1, E2, out, stream_);
  if (timed) timing_end(1, a.nf * dft_flops_per_field());
}

void Engine::project_fields(const DftPlan& p, const float* f, const FinArgs& a, float2* G1, float2* G2,
                            float2* G3) {
  const bool timed = (gt_on_ & 2) && &p == &full_;
  if (timed) timing_begin();
  dft_project_fin(p, f, a, G1, G2, G3, stream_);
  if (timed) timing_end(1, a.nf * dft_flops_per_field());
}

// out_i = pi(gather(spline(iota(in_i)), dep)) combined per FinField (advect_state, transport.hpp:67-73)
void Engine::advect_multi(const double2* const* in, int nf, const float* dep, const FinField* outs) {
  const long long N = npts();
  for (int c0 = 0; c0 < nf; c0 += fmax_full_) {
    const int n = std::min(fmax_full_, nf - c0);
    PrepArgs pa{};
    pa.nf = n;
    for (int i = 0; i < n; ++i) pa.f[i] = PrepField{in[c0 + i], SYM_PREFILTER, 1.0};
    embed_fields(full_, pa, gridA_.p, D_.p, E1_.p, E2_.p);
    timed_gather(gridA_.p, n, dep, gridB_.p);
    FinArgs fa{};
    fa.nf = n;
    for (int i = 0; i < n; ++i) fa.f[i] = outs[c0 + i];
    project_fields(full_, gridB_.p, fa, G1_.p, G2_.p, G3_.p);
  }
  (void)N;
}

// truncated products on the small grid; op: 0 star(s,s) 1 star(s,vec) 2 star_dot 3 jac 4 jacT
// out = alpha * product + beta * add
void Engine::small_product(int op, const double2* a, const double2* b, double2* out, double alpha,
                           const double2* add, double beta) {
  const long long M = small_.npts(), K = kprod();
  PrepArgs pa{};
  int nb = 0;
  if (op == 0) {
    pa.f[0] = PrepField{a, SYM_NONE, 1.0};
    pa.f[1] = PrepField{b, SYM_NONE, 1.0};
    pa.nf = 2;
  } else if (op == 1) {
    pa.f[0] = PrepField{a, SYM_NONE, 1.0};
    for (int c = 0; c < 3; ++c) pa.f[1 + c] = PrepField{b + c * K, SYM_NONE, 1.0};
    pa.nf = 4;
  } else if (op == 2) {
    for (int c = 0; c < 3; ++c) pa.f[c] = PrepField{a + c * K, SYM_NONE, 1.0};
    for (int c = 0; c < 3; ++c) pa.f[3 + c] = PrepField{b + c * K, SYM_NONE, 1.0};
    pa.nf = 6;
  } else {
    for (int ac = 0; ac < 3; ++ac)
      for (int bc = 0; bc < 3; ++bc) pa.f[ac * 3 + bc] = PrepField{a + ac * K, SYM_DERIV_X + bc, 1.0};
    for (int c = 0; c < 3; ++c) pa.f[9 + c] = PrepField{b + c * K, SYM_NONE, 1.0};
    pa.nf = 12;
  }
  embed_fields(small_, pa, sgrid_.p, sD_.p, sE1_.p, sE2_.p);
  float* acc = sacc_.p;
  switch (op) {
    case 0: launch_products(4, M, sgrid_.p, sgrid_.p + M, acc, 1.f, true, stream_); nb = 1; break;
    case 1: launch_products(2, M, sgrid_.p, sgrid_.p + M, acc, 1.f, true, stream_); nb = 3; break;
    case 2: launch_products(3, M, sgrid_.p, sgrid_.p + 3 * M, acc, 1.f, true, stream_); nb = 1; break;
    case 3: launch_products(0, M, sgrid_.p, sgrid_.p + 9 * M, acc, 1.f, true, stream_); nb = 3; break;
    default: launch_products(1, M, sgrid_.p, sgrid_.p + 9 * M, acc, 1.f, true, stream_); nb = 3; break;
  }
  FinArgs fa{};
  fa.nf = nb;
  for (int c = 0; c < nb; ++c)
    fa.f[c] = FinField{out + c * K, alpha * small_ratio_, add ? add + c * K : nullptr, beta};
  project_fields(small_, acc, fa, sG1_.p, sG2_.p, sG3_.p);
}

void Engine::star_ss(const double2* a, const double2* b, double2* out, double alpha) {
  small_product(0, a, b, out, alpha, nullptr, 0.0);
}
void Engine::star_sv(const double2* s, const double2* x, double2* out, double alpha) {
  small_product(1, s, x, out, alpha, nullptr, 0.0);
}
void Engine::star_dot(const double2* a, const double2* b, double2* out, double alpha) {
  small_product(2, a, b, out, alpha, nullptr, 0.0);
}
void Engine::jac_mul(const double2* u, const double2* w, double2* out, double alpha, bool transpose) {
  small_product(transpose ? 4 : 3, u, w, out, alpha, nullptr, 0.0);
}
void Engine::band_divergence(const double2* v, double2* out) {
  launch_band_divergence(v, out, full_.K, full_.omega_unit, stream_);
}

void Engine::warp_grid(const float* f, int ncomp, const float* disp_phys, float* out) {
  const long long N = npts();
  shape_require(ncomp >= 1 && ncomp <= fmax_full_, "warp_grid: 1..6 components");
  LDDMM_CUDA(cudaMemcpyAsync(gridA_.p, f, ncomp * N * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
  double* c = f64c_.p;
  for (int k = 0; k < ncomp; ++k) {
    launch_f32_to_f64(N, gridA_.p + k * N, c, stream_);
    launch_prefilter3d(c, full_.N, stream_);
    launch_f64_to_f32(N, c, gridA_.p + k * N, stream_);
  }
  for (int k = 0; k < ncomp;) {
    const int n = (ncomp - k >= 4) ? 4 : (ncomp - k >= 3 ? 3 : 1);
    launch_warp_by_displacement(gridA_.p + k * N, n, disp_phys, h_, out + k * N, full_.N, stream_);
    k += n;
  }
}

void Engine::embed(const double2* c, int ncomp, float* out, bool prefilter) {
  const long long K = kprod(), N = npts();
  for (int c0 = 0; c0 < ncomp; c0 += fmax_full_) {
    const int n = std::min(fmax_full_, ncomp - c0);
    PrepArgs pa{};
    pa.nf = n;
    for (int i = 0; i < n; ++i) pa.f[i] = PrepField{c + (c0 + i) * K, prefilter ? SYM_PREFILTER : SYM_NONE, 1.0};
    embed_fields(full_, pa, out + c0 * N, D_.p, E1_.p, E2_.p);
  }
}

void Engine::project(const float* f, int ncomp, double2* out) {
  const long long K = kprod(), N = npts();
  for (int c0 = 0; c0 < ncomp; c0 += fmax_full_) {
    const int n = std::min(fmax_full_, ncomp - c0);
    FinArgs fa{};
    fa.nf = n;
    for (int i = 0; i < n; ++i) fa.f[i] = FinField{out + (c0 + i) * K, 1.0, nullptr, 0.0};
    project_fields(full_, f + c0 * N, fa, G1_.p, G2_.p, G3_.p);
  }
}

void Engine::advect(const double2* q, int ncomp, const float* dep, double2* out) {
  const long long K = kprod();
  std::vector<const double2*> in(ncomp);
  std::vector<FinField> outs(ncomp);
  for (int c = 0; c < ncomp; ++c) {
    in[c] = q + c * K;
    outs[c] = FinField{out + c * K, 1.0, nullptr, 0.0};
  }
  advect_multi(in.data(), ncomp, dep, outs.data());
}

// ---------------------------------------------------------------------------
// provider (transport.hpp:109-218, stationary): spatial node, spline coefficients,
// band divergence, departure points, cfl

bool Engine::same_velocity(const double2* a, const double2* b) {
  // slot 1 reinterpreted as the mismatch counter
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(slots_.p + 1);
  launch_equal_flag(2 * vel_elems(), reinterpret_cast<const double*>(a), reinterpret_cast<const double*>(b), cnt,
                    stream_);
  LDDMM_CUDA(cudaMemcpyAsync(host_slots_ + 1, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
  sync();
  unsigned long long m = 0;
  std::memcpy(&m, host_slots_ + 1, sizeof(m));
  return m == 0;
}

// trial provider + u series -> the forward cache (buffer swaps), then the backward
// departure of the same velocity (stationary SL: transport.hpp:176-187)
void Engine::adopt_trial_provider(bool with_bwd) {
  auto swapbuf = [](auto& a, auto& b) {
    std::swap(a.p, b.p);
    std::swap(a.n, b.n);
  };
  swapbuf(prov_.v, trial_prov_.v);
  swapbuf(prov_.div, trial_prov_.div);
  swapbuf(prov_.dep_fwd, trial_prov_.dep_fwd);
  if (prob_.variant == 0)
    swapbuf(m_ser_, trial_mser_);  // transported image series (original)
  else
    swapbuf(u_, trial_u_);  // displacement series (state / deformation-state)
  prov_.cfl = trial_prov_.cfl;
  pullback_large_ = prov_.cfl * prob_.nt > 1.0;
  prov_.has_bwd = false;
  if (with_bwd) {
    const long long N = npts(), K = kprod();
    PrepArgs pa{};
    pa.nf = 6;
    for (int c = 0; c < 3; ++c) {
      pa.f[c] = PrepField{prov_.v.p + c * K, SYM_NONE, 1.0};
      pa.f[3 + c] = PrepField{prov_.v.p + c * K, SYM_PREFILTER, 1.0};
    }
    embed_fields(full_, pa, gridA_.p, D_.p, E1_.p, E2_.p);
    launch_departure_dir(gridA_.p, gridA_.p + 3 * N, 1.0 / prob_.nt, h_, 1.f, prov_.dep_bwd.p, gridB_.p, full_.N,
                         stream_);
    prov_.has_bwd = true;
  }
}

void Engine::provider_build(const double2* v, ProviderState& ps, bool with_bwd) {
  const long long N = npts(), K = kprod(), V = vec_elems();
  const int nn = nodes(), nt = prob_.nt;
  const double dt = 1.0 / nt;
  LDDMM_CUDA(cudaMemcpyAsync(ps.v.p, v, vel_elems() * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  for (int i = 0; i < nn; ++i) launch_band_divergence(v + i * V, ps.div.p + i * K, full_.K, full_.omega_unit, stream_);
  // per node: spatial node iota(v_i) and its spline coefficients iota(v_i / B)
  auto embed_node = [&](int i, float* dst) {
    PrepArgs pa{};
    pa.nf = 6;
    for (int c = 0; c < 3; ++c) {
      pa.f[c] = PrepField{v + i * V + c * K, SYM_NONE, 1.0};
      pa.f[3 + c] = PrepField{v + i * V + c * K, SYM_PREFILTER, 1.0};
    }
    embed_fields(full_, pa, dst, D_.p, E1_.p, E2_.p);
    const int g = launch_absmax_partial(3 * N, dst, part_.p, stream_);
    launch_reduce_final(part_, g, 1, slots_.p + 16 + i, stream_);  // cfl: max over nodes (transport.hpp:189-194)
  };
  if (prob_.rk4) {
    // RK4 uses the band velocity and divergence only; iota(v_i) is embedded for the cfl
    for (int i = 0; i < nn; ++i) embed_node(i, gridA_.p);
  } else if (prob_.stationary) {
    embed_node(0, gridA_.p);
    launch_departure(gridA_.p, gridA_.p + 3 * N, dt, h_, ps.dep_fwd.p, with_bwd ? ps.dep_bwd.p : nullptr, gridB_.p,
                     full_.N, stream_);
  } else {
    // departure(step): forward from v_grid = node(step+1), v_traced = node(step); backward from
    // v_grid = node(step), v_traced = node(step+1) (transport.hpp:176-187)
    float* prev = pscratch_.p;         // grid + coefficients of node i-1 [6][N]
    float* vm = pscratch_.p + 6 * N;   // gathered traced velocity [3][N]
    for (int i = 0; i <= nt; ++i) {
      embed_node(i, gridA_.p);
      if (i >= 1) {
        launch_departure_dir(gridA_.p, prev + 3 * N, dt, h_, -1.f, ps.dep_fwd.p + (i - 1) * 3 * N, vm, full_.N,
                             stream_);
        if (with_bwd)
          launch_departure_dir(prev, gridA_.p + 3 * N, dt, h_, 1.f, ps.dep_bwd.p + (i - 1) * 3 * N, vm, full_.N,
                               stream_);
      }
      LDDMM_CUDA(cudaMemcpyAsync(prev, gridA_.p, 6 * N * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
    }
  }
  ps.has_bwd = with_bwd;
  LDDMM_CUDA(cudaMemcpyAsync(host_slots_ + 16, slots_.p + 16, nn * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  double vmax = 0.0;
  for (int i = 0; i < nn; ++i) vmax = std::max(vmax, host_slots_[16 + i]);
  const double hmin = prob_.d == 2 ? std::min(h_[0], h_[1]) : std::min(h_[0], std::min(h_[1], h_[2]));
  ps.cfl = vmax * dt / hmin;
  // whole-map pull-backs of this forward move nodes by up to max|v| T / h = cfl nt voxels
  pullback_large_ = ps.cfl * prob_.nt > 1.0;
}

void Engine::departure(const double2* v, float* dep_fwd, float* dep_bwd, double* cfl) {
  shape_require(!prob_.rk4, "departure points belong to the SL integrator");
  provider_build(v, prov_, true);
  const long long N = npts();
  if (dep_fwd)
    LDDMM_CUDA(cudaMemcpyAsync(dep_fwd, prov_.dep_fwd.p, 3 * N * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
  if (dep_bwd)
    LDDMM_CUDA(cudaMemcpyAsync(dep_bwd, prov_.dep_bwd.p, 3 * N * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
  if (cfl) *cfl = prov_.cfl;
  have_cache_ = false;
  sync();
}

// Non-finite check of the node filled at march step s (transport.hpp:225-228,285,293):
// enqueue one device flag per step, read all flags back once per solve.
void Engine::enqueue_finite_check(const double2* node, int step) {
  launch_nonfinite_flag(vec_elems(), node, part2_.p, slots_.p + 16 + step, stream_);
}

void Engine::finish_finite_checks(int nsteps) {
  LDDMM_CUDA(cudaMemcpyAsync(host_slots_ + 16, slots_.p + 16, nsteps * sizeof(double), cudaMemcpyDeviceToHost,
                             stream_));
  sync();
  for (int s = 0; s < nsteps; ++s)
    if (host_slots_[16 + s] != 0.0)
      throw EngineError(2, "transport produced non-finite values (step " + std::to_string(s) + ")", s);
}

void Engine::check_series_finite(const double2* series, int count, int first, bool backward) {
  const long long V = vec_elems();
  const int nt = prob_.nt;
  if (count > 0) {
    // steps first .. first + count - 1 fill nodes first + 1 .. (forward) or nt - first - 1
    // down to nt - first - count (backward): one contiguous range, one launch
    const int lo = backward ? nt - first - count : first + 1;
    launch_nonfinite_series(series + lo * V, V, count, first, backward, slots_.p + 16, stream_);
  }
  finish_finite_checks(first + count);
}

// D_t u = v forward from 0 (variants.hpp:468-472) with the stationary f_from
// cached: next = dt/2 f_from + (dt/2 v + A), A = advect(u_s) (A = 0 at s = 0).
void Engine::solve_displacement_fwd(ProviderState& ps, double2* series, bool keep_all, double2* last) {
  if (prob_.rk4) {
    rk4_displacement(ps, true, keep_all ? series : nullptr, last);
    return;
  }
  const long long V = vec_elems(), K = kprod();
  const int nt = prob_.nt;
  const double dt = 1.0 / nt;
  double2* F = bt(0);
  if (prob_.stationary) advect(ps.v.p, 3, ps.dep_fwd.p, F);
  double2* prev = nullptr;
  for (int s = 0; s < nt; ++s) {
    double2* dst = keep_all ? series + (s + 1) * V : tmp_u_.p + ((s + 1) & 1) * V;
    double2* tmp = bt(1);
    if (prob_.stationary) {
      if (s == 0) {
        launch_scale(V, 0.5 * dt, ps.v.p, tmp, stream_);  // 0.5 dt v + 0
      } else {
        const double2* in[3] = {prev, prev + K, prev + 2 * K};
        FinField outs[3];
        for (int c = 0; c < 3; ++c) outs[c] = FinField{tmp + c * K, 1.0, ps.v.p + c * K, 0.5 * dt};
        advect_multi(in, 3, ps.dep_fwd.p, outs);
      }
      launch_axpy(V, 0.5 * dt, F, tmp, dst, stream_);
    } else {
      // q-independent source v(t_i): merged advect, next = advect(u_s + dt/2 v_s) + dt/2 v_{s+1}
      if (s == 0)
        launch_scale(V, 0.5 * dt, vnode(ps, 0), tmp, stream_);
      else
        launch_axpy(V, 0.5 * dt, vnode(ps, s), prev, tmp, stream_);
      const double2* in[3] = {tmp, tmp + K, tmp + 2 * K};
      FinField outs[3];
      for (int c = 0; c < 3; ++c) outs[c] = FinField{dst + c * K, 1.0, vnode(ps, s + 1) + c * K, 0.5 * dt};
      advect_multi(in, 3, depf(ps, s), outs);
    }
    enqueue_finite_check(dst, s);
    prev = dst;
  }
  if (keep_all) LDDMM_CUDA(cudaMemsetAsync(series, 0, V * sizeof(double2), stream_));
  if (last) LDDMM_CUDA(cudaMemcpyAsync(last, prev, V * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  finish_finite_checks(nt);
}

// componentwise continuity D_t q = -(div v) q, backward from q1 (variants.hpp:499-503)
void Engine::solve_vector_continuity_bwd(ProviderState& ps, const double2* q1, double2* series) {
  if (prob_.rk4) {
    rk4_vector_continuity_bwd(ps, q1, series);
    return;
  }
  const long long V = vec_elems(), K = kprod();
  const int nt = prob_.nt;
  const double sdt = -1.0 / nt;
  LDDMM_CUDA(cudaMemcpyAsync(series + nt * V, q1, V * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  for (int s = 0; s < nt; ++s) {
    const int from = nt - s, to = nt - s - 1;
    const double2* q = series + from * V;
    double2 *sf = bt(0), *A = bt(1), *F = bt(2), *qs = bt(3), *ft = bt(4), *tmp = bt(5);
    small_product(1, divnode(ps, from), q, sf, -1.0, nullptr, 0.0);  // src(q_from) = -(div * q)
    const double2* in[6] = {q, q + K, q + 2 * K, sf, sf + K, sf + 2 * K};
    FinField outs[6];
    for (int c = 0; c < 3; ++c) {
      outs[c] = FinField{A + c * K, 1.0, nullptr, 0.0};
      outs[3 + c] = FinField{F + c * K, 1.0, nullptr, 0.0};
    }
    advect_multi(in, 6, depb(ps, to), outs);
    launch_axpy(V, sdt, F, A, qs, stream_);                          // q* = sdt f_from + A
    small_product(1, divnode(ps, to), qs, ft, -1.0, nullptr, 0.0);  // f_to = src(q*)
    launch_axpy(V, 0.5 * sdt, ft, A, tmp, stream_);           // 0.5 sdt f_to + A
    launch_axpy(V, 0.5 * sdt, F, tmp, series + to * V, stream_);
  }
  check_series_finite(series, nt, 0, true);
}

// D_t du = dv - (Du) dv forward from 0 (variants.hpp:530-540), merged advect:
// next = advect(du_s + dt/2 src_s) + dt/2 src_{s+1}.
void Engine::solve_incremental_displacement(ProviderState& ps, const double2* dv, double2* series) {
  if (prob_.rk4) {
    rk4_incremental_displacement(ps, dv, series);
    return;
  }
  const long long V = vec_elems(), K = kprod();
  const int nt = prob_.nt;
  const double dt = 1.0 / nt;
  // sources src_i = -jac(u_i, dv_i) + dv_i ; u_0 = 0 so src_0 = dv_0 exactly.  The
  // sources do not depend on du, so the nodes go through the small grid in batches (one
  // embed / product / project pipeline per batch instead of per node; every field takes
  // the same arithmetic as in a single small_product, so the values are identical)
  LDDMM_CUDA(cudaMemcpyAsync(src_.p, dv, V * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  {
    const long long M = small_.npts();
    const bool stat = prob_.stationary != 0;
    const int per = stat ? std::min((fmax_small_ - 3) / 9, 6) : std::min(fmax_small_ / 12, 5);
    for (int i0 = 1; i0 <= nt; i0 += per) {
      const int nn = std::min(per, nt + 1 - i0);
      PrepArgs pa{};
      for (int n = 0; n < nn; ++n)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            pa.f[n * 9 + a * 3 + b] = PrepField{u_.p + (i0 + n) * V + a * K, SYM_DERIV_X + b, 1.0};
      const int nw = stat ? 1 : nn;  // dv fields: one set (stationary) or one per node
      for (int n = 0; n < nw; ++n)
        for (int c = 0; c < 3; ++c) pa.f[9 * nn + n * 3 + c] = PrepField{tvnode(dv, i0 + n) + c * K, SYM_NONE, 1.0};
      pa.nf = 9 * nn + 3 * nw;
      embed_fields(small_, pa, sgrid_.p, sD_.p, sE1_.p, sE2_.p);
      launch_jac_batch(false, nn, M, sgrid_.p, sgrid_.p + 9 * nn * M, stat ? 0 : 3 * M, sacc_.p, 3 * M,
                       NodeWeights{}, true, stream_);
      FinArgs fa{};
      fa.nf = 3 * nn;
      for (int n = 0; n < nn; ++n)
        for (int c = 0; c < 3; ++c)
          fa.f[n * 3 + c] = FinField{src_.p + (i0 + n) * V + c * K, -small_ratio_, tvnode(dv, i0 + n) + c * K, 1.0};
      project_fields(small_, sacc_.p, fa, sG1_.p, sG2_.p, sG3_.p);
    }
  }
  LDDMM_CUDA(cudaMemsetAsync(series, 0, V * sizeof(double2), stream_));
  for (int s = 0; s < nt; ++s) {
    double2* in = bt(0);
    launch_axpy(V, 0.5 * dt, src_.p + s * V, series + s * V, in, stream_);
    const double2* ins[3] = {in, in + K, in + 2 * K};
    FinField outs[3];
    for (int c = 0; c < 3; ++c)
      outs[c] = FinField{series + (s + 1) * V + c * K, 1.0, src_.p + (s + 1) * V + c * K, 0.5 * dt};
    advect_multi(ins, 3, depf(ps, s), outs);
  }
  check_series_finite(series, nt, 0, false);
}

// m1 = I0 o (x - iota(u1)) (cubic), residual, optionally grad_src_warped (variants.hpp:426-430)
void Engine::warp_m1(const double2* u1, float* m1, float* res, bool want_gsw, double* data_sumsq) {
  const long long N = npts();
  embed(u1, 3, ugrid_.p, false);
  launch_warp_by_displacement(I0coef_.p, want_gsw ? 4 : 1, ugrid_.p, h_, m1, full_.N, stream_, pullback_large_);
  const int g = launch_residual(N, m1, I1_.p, res, part_.p, stream_);
  *data_sumsq = reduce(g, 0);
}

// terms_i = q_i - jacT(u_i, q_i); out = L like + sum_i w_i terms_i (variants.hpp:291-309,357-362)
void Engine::assemble_jacT_terms(const double2* U, const double2* Q, const double2* like, double2* out) {
  const long long V = vec_elems(), K = kprod(), M = small_.npts();
  const int nt = prob_.nt;
  const auto w = trapezoid_weights(nt);
  if (!prob_.stationary) {
    // nonstationary: out_i = L like_i + (q_i - jacT(u_i, q_i)) (variants.hpp:364-368)
    for (int i = 0; i <= nt; ++i) {
      double2* tmp = bt(7);
      if (i == 0)
        LDDMM_CUDA(cudaMemcpyAsync(tmp, Q, V * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
      else
        small_product(4, U + i * V, Q + i * V, tmp, -1.0, Q + i * V, 1.0);
      double2* lv = bt(8);
      launch_sobolev(like + i * V, lv, 3, full_.K, full_.omega_unit, prob_.alpha, prob_.s, false, stream_);
      launch_axpy(V, 1.0, lv, tmp, out + i * V, stream_);
    }
    return;
  }
  // band part: acc = sum_i w_i q_i
  double2* acc = bt(6);
  launch_weighted_sum(V, nt + 1, w.data(), Q, V, acc, stream_);
  // product part on the small grid, nodes 1..nt (u_0 = 0)
  const int per_chunk = std::min(5, fmax_small_ / 12);
  bool first = true;
  for (int i0 = 1; i0 <= nt; i0 += per_chunk) {
    const int nn = std::min(per_chunk, nt + 1 - i0);
    PrepArgs pa{};
    pa.nf = 12 * nn;
    for (int n = 0; n < nn; ++n) {
      const double2* u = U + (i0 + n) * V;
      const double2* q = Q + (i0 + n) * V;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) pa.f[n * 9 + a * 3 + b] = PrepField{u + a * K, SYM_DERIV_X + b, 1.0};
      for (int c = 0; c < 3; ++c) pa.f[9 * nn + n * 3 + c] = PrepField{q + c * K, SYM_NONE, 1.0};
    }
    embed_fields(small_, pa, sgrid_.p, sD_.p, sE1_.p, sE2_.p);
    NodeWeights nw{};
    for (int n = 0; n < nn; ++n) nw.w[n] = (float)w[i0 + n];
    launch_jac_batch(true, nn, M, sgrid_.p, sgrid_.p + 9 * nn * M, 3 * M, sacc_.p, 0, nw, first, stream_);
    first = false;
  }
  double2* tmp = bt(7);
  FinArgs fa{};
  fa.nf = 3;
  for (int c = 0; c < 3; ++c) fa.f[c] = FinField{tmp + c * K, -small_ratio_, acc + c * K, 1.0};
  project_fields(small_, sacc_.p, fa, sG1_.p, sG2_.p, sG3_.p);
  double2* lv = bt(8);
  launch_sobolev(like, lv, 3, full_.K, full_.omega_unit, prob_.alpha, prob_.s, false, stream_);
  launch_axpy(V, 1.0, lv, tmp, out, stream_);
}

// ---------------------------------------------------------------------------
// Model API

double Engine::reg_energy(const double2* v) {  // variants.hpp:280-287
  const long long V = vec_elems();
  const auto w = trapezoid_weights(prob_.nt);
  double acc = 0.0;
  for (int i = 0; i < nodes(); ++i) {
    double2* lv = bt(9);
    launch_sobolev(v + i * V, lv, 3, full_.K, full_.omega_unit, prob_.alpha, prob_.s, false, stream_);
    const int g = launch_inner_partial(V, lv, v + i * V, part_.p, stream_);
    const double s = reduce(g, 0) * cell_volume_ / (double)npts();
    if (prob_.stationary) return 0.5 * s;
    acc += w[i] * s;
  }
  return 0.5 * acc;
}

Energies Engine::forward(const double2* v, bool with_adjoint) {
  LDDMM_NVTX(with_adjoint ? "forward+adjoint" : "forward");
  const long long V = vec_elems(), N = npts();
  have_cache_ = false;
  // The forward at the velocity of the line search's accepted trial (optimizer.hpp:219,
  // after trial_energy at the same tv_axpy result) adopts the trial's provider and u
  // series instead of recomputing them: the same kernels on the same inputs, so the
  // values are identical; only the backward departures are added.
  const bool reuse = trial_reuse_ok() && trial_valid_ && same_velocity(v, trial_prov_.v.p);
  trial_valid_ = false;
  if (reuse) {
    adopt_trial_provider(with_adjoint);
  } else {
    provider_build(v, prov_, with_adjoint);
  }
  Energies e;
  e.cfl = prov_.cfl;
  double ss = 0.0;
  if (prob_.variant == 0) {
    ss = forward_original(with_adjoint, v, reuse);
  } else if (prob_.variant == 1) {
    ss = forward_state(with_adjoint, reuse);
  } else {
    if (!reuse) solve_displacement_fwd(prov_, u_.p, true, nullptr);
    warp_m1(u_.p + prob_.nt * V, m1_.p, res_.p, with_adjoint, &ss);
  }
  if (with_adjoint && prob_.variant == 2) {
    float* gsw = m1_.p + N;
    launch_scale_vec(N, res_.p, -2.0 / prob_.sigma2, gsw, gridB_.p, stream_);  // r1
    double2* r1 = bt(10);
    project(gridB_.p, 3, r1);
    solve_vector_continuity_bwd(prov_, r1, rho_.p);
  }
  e.energy_reg = reg_energy(v);
  e.energy_data = ss * cell_volume_ / prob_.sigma2;
  e.energy = e.energy_reg + e.energy_data;
  cache_e_ = e;
  have_cache_ = true;
  cache_adjoint_ = with_adjoint;
  return e;
}

double Engine::energy(const double2* v) {
  LDDMM_NVTX("energy (trial)");
  if (prob_.variant == 0) return energy_original(v);
  trial_valid_ = false;  // set again only when this trial completes
  provider_build(v, trial_prov_, false);
  double ss = 0.0;
  if (trial_reuse_ok()) {  // state / deformation-state variants
    // keep the whole u series: if this trial is accepted, the forward at the same
    // velocity (optimizer.hpp:219) adopts it instead of recomputing (forward())
    solve_displacement_fwd(trial_prov_, trial_u_.p, true, nullptr);
    warp_m1(trial_u_.p + prob_.nt * vec_elems(), trial_m1_.p, trial_res_.p, false, &ss);
    trial_valid_ = true;
  } else {
    solve_displacement_fwd(trial_prov_, nullptr, false, bt(11));
    warp_m1(bt(11), trial_m1_.p, trial_res_.p, false, &ss);
  }
  const double er = reg_energy(v);
  return er + ss * cell_volume_ / prob_.sigma2;
}

void Engine::gradient(double2* out) {
  LDDMM_NVTX("gradient");
  shape_require(have_cache_ && cache_adjoint_, "gradient requires an adjoint-enabled forward cache");
  if (prob_.variant == 2)
    assemble_jacT_terms(u_.p, rho_.p, prov_.v.p, out);
  else
    assemble_star_grad(lam_ser_.p, m_ser_.p, prov_.v.p, out);
}

void Engine::hessvec(const double2* dv, double2* out) {
  LDDMM_NVTX("hessvec");
  shape_require(have_cache_ && cache_adjoint_, "hessvec requires an adjoint-enabled forward cache");
  if (prob_.variant == 0) return hessvec_original(dv, out);
  if (prob_.variant == 1) return hessvec_state(dv, out);
  const long long V = vec_elems(), N = npts();
  const int nt = prob_.nt;
  DevBuf<double2>& series = dseries_;  // du series, then reused for the drho series
  solve_incremental_displacement(prov_, dv, series.p);
  embed(series.p + nt * V, 3, ugrid_.p, false);  // du1 (ugrid_ is scratch here)
  launch_dr1(N, m1_.p + N, ugrid_.p, -2.0 / prob_.sigma2, gridB_.p, stream_);
  double2* dr1 = bt(10);
  project(gridB_.p, 3, dr1);
  solve_vector_continuity_bwd(prov_, dr1, series.p);
  assemble_jacT_terms(u_.p, series.p, dv, out);
}

void Engine::precondition(const double2* in, double2* out) {  // variants.hpp:347-353
  launch_sobolev(in, out, 3 * nodes(), full_.K, full_.omega_unit, prob_.alpha, prob_.s, true, stream_);
}

void Engine::tv_axpy(double a, const double2* x, const double2* y, double2* out) {
  launch_axpy(vel_elems(), a, x, y, out, stream_);
}
void Engine::tv_scaled(const double2* x, double a, double2* out) { launch_scale(vel_elems(), a, x, out, stream_); }
double Engine::tv_inner(const double2* a, const double2* b) {  // variants.hpp:94-103
  if (prob_.stationary) {
    const int g = launch_inner_partial(vel_elems(), a, b, part_.p, stream_);
    return reduce(g, 0) * cell_volume_ / (double)npts();
  }
  const long long V = vec_elems();
  const auto w = trapezoid_weights(prob_.nt);
  double s = 0.0;
  for (int i = 0; i <= prob_.nt; ++i) {
    const int g = launch_inner_partial(V, a + i * V, b + i * V, part_.p, stream_);
    s += w[i] * (reduce(g, 0) * cell_volume_ / (double)npts());
  }
  return s;
}
double Engine::tv_linf(const double2* a) {
  const int g = launch_linf_partial(vel_elems(), a, part_.p, stream_);
  return reduce(g, 1) / prob_.zrep;  // 2-D: the 2-D coefficients' max norm
}
bool Engine::tv_all_finite(const double2* a) {
  const int g = launch_nonfinite_partial(vel_elems(), a, part_.p, stream_);
  return reduce(g, 1) == 0.0;
}

double Engine::residual_sumsq() {
  const int g = launch_sumsq_partial(npts(), res_.p, part_.p, stream_);
  return reduce(g, 0);
}

void Engine::series(int which, double2* out) {
  const long long V = vec_elems();
  LDDMM_CUDA(cudaMemcpyAsync(out, which == 0 ? u_.p : rho_.p, (prob_.nt + 1) * V * sizeof(double2),
                             cudaMemcpyDeviceToDevice, stream_));
  sync();
}

// Circulant spectral-derivative kernels D_a[d] = (1/n) sum_k i omega_k e^{2 pi i k d / n}
// (grid Nyquist k = n/2 excluded, omega = 2 pi k / (n h)): a full-grid
// spectral_derivative (spectral.hpp:326-334,339-354) as an exact real convolution.
void Engine::ensure_dker() {
  if (dker_ready_) return;
  for (int a = 0; a < 3; ++a) {
    const int n = full_.N[a];
    shape_require(n <= 1024, "spectral derivative: axis length > 1024");
    std::vector<double> Dh(n);
    for (int d = 0; d < n; ++d) {
      long double acc = 0.0L;
      for (int k = -n / 2 + 1; k < n / 2; ++k) {
        const long double om = 2.0L * 3.14159265358979323846264338327950288L * k / (n * h_[a]);
        const long long r = (((long long)k * d) % n + n) % n;
        acc += -om * sinl(2.0L * 3.14159265358979323846264338327950288L * r / n);
      }
      Dh[d] = (double)(acc / n);
    }
    LDDMM_CUDA(cudaMemcpyAsync(dker_.p + 1024 * a, Dh.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream_));
    LDDMM_CUDA(cudaStreamSynchronize(stream_));
  }
  dker_ready_ = true;
}

void Engine::warp_nearest(const float* f, int ncomp, const float* disp_phys, float* out) {
  launch_warp_nearest(f, ncomp, disp_phys, h_, out, full_.N, stream_);
}

// map_jacobian_determinant + value_range (metrics.hpp:40-79) of a grid displacement
void Engine::jacobian_grid(const float* disp, float* det, double mm[2]) {
  const long long N = npts();
  ensure_dker();
  if (maps_du_.n < (size_t)(9 * N)) maps_du_.alloc(9 * N);
  for (int a = 0; a < 3; ++a) {
    launch_f32_to_f64(N, disp + a * N, f64a_.p, stream_);
    for (int b = 0; b < 3; ++b) {
      launch_circulant_axis_f64(f64a_.p, f64b_.p, dker_.p + 1024 * b, b, full_.N, stream_);
      launch_f64_to_f32(N, f64b_.p, maps_du_.p + (3 * a + b) * N, stream_);
    }
  }
  if (det) launch_jacdet(N, maps_du_.p, det, stream_);
  const int g = launch_jacdet_minmax(N, maps_du_.p, part_.p, part2_.p, stream_);
  launch_reduce_final(part_.p, g, 1, slots_.p + 2, stream_);
  launch_reduce_final(part2_.p, g, 1, slots_.p + 3, stream_);
  LDDMM_CUDA(cudaMemcpyAsync(host_slots_ + 2, slots_.p + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  mm[0] = -host_slots_[2];
  mm[1] = host_slots_[3];
}

void Engine::dice_counts(const float* a, const float* b, const float* labels, int nl, unsigned long long* counts) {
  launch_dice_counts(npts(), a, b, labels, nl, counts, stream_);
}

// compute_maps + map_jacobian_determinant + value_range (metrics.hpp:24-79)
void Engine::maps(const double2* v, float* disp_fwd, float* disp_inv, double jac[4]) {
  const long long V = vec_elems(), N = npts(), K = kprod();
  const int nt = prob_.nt;
  const double dt = 1.0 / nt;
  provider_build(v, prov_, true);
  have_cache_ = false;
  // u(1): forward displacement; nu(0): backward displacement (same SL scheme, src = v)
  double2* u1 = bt(11);
  solve_displacement_fwd(prov_, u_.p, true, u1);
  solve_displacement(prov_, false, rho_.p);
  const double2* nu0 = rho_.p;
  for (int which = 0; which < 2; ++which) {
    const double2* d = which == 0 ? u1 : nu0;
    float* dst = which == 0 ? disp_fwd : disp_inv;
    if (dst) embed(d, 3, dst, false);
    // 9 derivative embeds d_b u_a: spectral_derivative of a band-limited field is
    // embed(i omega_b u_a) (its grid-Nyquist content is zero)
    if (maps_du_.n < (size_t)(9 * N)) maps_du_.alloc(9 * N);
    DevBuf<float>& du = maps_du_;
    int done = 0;
    while (done < 9) {
      const int n = std::min(fmax_full_, 9 - done);
      PrepArgs p2{};
      p2.nf = n;
      for (int i = 0; i < n; ++i) {
        const int ab = done + i, a = ab / 3, b = ab % 3;
        p2.f[i] = PrepField{d + a * K, SYM_DERIV_X + b, 1.0};
      }
      embed_fields(full_, p2, du.p + done * N, D_.p, E1_.p, E2_.p);
      done += n;
    }
    const int g = launch_jacdet_minmax(N, du.p, part_.p, part2_.p, stream_);
    launch_reduce_final(part_.p, g, 1, slots_.p + 2, stream_);
    launch_reduce_final(part2_.p, g, 1, slots_.p + 3, stream_);
    LDDMM_CUDA(cudaMemcpyAsync(host_slots_ + 2, slots_.p + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    sync();
    jac[2 * which] = -host_slots_[2];
    jac[2 * which + 1] = host_slots_[3];
  }
}

}  // namespace lddmm_b200
