// C entry points over the UNMODIFIED reference headers (test infrastructure).
//
// Compiled by oracle/Makefile straight from /root/reference/proj/include (no
// reference source is copied into this repo) together with the FFTW3-API
// shim in oracle/fftw_shim.cpp, into oracle/_ref/libref_lddmm.so.  Tests,
// tests/golden/make_golden.py and bench.py's reference/cpu_baseline legs load
// it through oracle/ref.py.  The product (paper_2006_06823_b200) never links
// or calls anything here.
//
// Conventions of this shim ABI:
//   grid fields  : double[ncomp][N], row-major, axis 0 slowest (core.hpp:8-9)
//   band fields  : double[ncomp][Kprod][2] interleaved re/im in the reference
//                  BandSpec DFT order (spectral.hpp:8-12)
//   velocities   : stationary -> one band vector field; nonstationary ->
//                  nt+1 of them back to back
//   return value : 0 ok, 1 ShapeError/Error, 2 DivergenceError (step in *step)

#include <lddmm/lddmm.hpp>

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

using namespace lddmm;

namespace {

thread_local std::string g_err;

GridSpec make_grid(int d, const int* dims, const double* h) {
  std::vector<int> n(dims, dims + d);
  std::vector<double> s(h, h + d);
  return GridSpec(n, s);
}

BandSpec make_band(const GridSpec& g, const int* band) {
  std::array<int, kMaxDim> b{1, 1, 1};
  for (int a = 0; a < g.d; ++a) b[a] = band[a];
  return BandSpec(g, b);
}

ScalarField scalar_in(const GridSpec& g, const double* p) {
  return ScalarField(g, std::vector<double>(p, p + g.size()));
}
void scalar_out(const ScalarField& f, double* p) { std::memcpy(p, f.v.data(), f.size() * 8); }

VectorField vector_in(const GridSpec& g, const double* p) {
  VectorField f(g);
  for (int a = 0; a < g.d; ++a) std::memcpy(f.comp[a].data(), p + (size_t)a * g.size(), g.size() * 8);
  return f;
}
void vector_out(const VectorField& f, double* p) {
  for (int a = 0; a < f.grid.d; ++a)
    std::memcpy(p + (size_t)a * f.grid.size(), f.comp[a].data(), f.grid.size() * 8);
}

BandScalarField bscalar_in(const BandSpec& b, const double* p) {
  BandScalarField f(b);
  std::memcpy(reinterpret_cast<double*>(f.c.data()), p, b.size() * 16);
  return f;
}
void bscalar_out(const BandScalarField& f, double* p) {
  std::memcpy(p, reinterpret_cast<const double*>(f.c.data()), f.size() * 16);
}
BandVectorField bvector_in(const BandSpec& b, const double* p) {
  BandVectorField f(b);
  for (int a = 0; a < b.d(); ++a)
    std::memcpy(reinterpret_cast<double*>(f.comp[a].data()), p + (size_t)a * b.size() * 2, b.size() * 16);
  return f;
}
void bvector_out(const BandVectorField& f, double* p) {
  for (int a = 0; a < f.band.d(); ++a)
    std::memcpy(p + (size_t)a * f.band.size() * 2, reinterpret_cast<const double*>(f.comp[a].data()),
                f.band.size() * 16);
}

using TV = TimeVaryingVelocity<BandVectorField>;

TV tv_in(const BandSpec& b, int param, int nt, const double* p) {
  const size_t stride = (size_t)b.d() * b.size() * 2;
  if (param == 0) return TV::stationary(bvector_in(b, p), nt);
  std::vector<BandVectorField> fs;
  for (int i = 0; i <= nt; ++i) fs.push_back(bvector_in(b, p + i * stride));
  return TV::nonstationary(std::move(fs));
}
void tv_out(const TV& v, double* p) {
  const BandSpec& b = v.node(0).band;
  const size_t stride = (size_t)b.d() * b.size() * 2;
  for (int i = 0; i < v.node_count(); ++i) bvector_out(v.node(i), p + i * stride);
}

template <class F>
int guard(F&& f, int* step = nullptr) {
  try {
    f();
    return 0;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    if (step) *step = e.step;
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefModel {
  BandSpec band;
  std::unique_ptr<Model<BandAlgebra>> model;
  std::unique_ptr<ForwardCache<BandAlgebra>> cache;
  int param = 0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { fftw_shim_set_threads(n); }

// ---- spectral.hpp -----------------------------------------------------------
int ref_embed(int d, const int* dims, const double* h, const int* band, int ncomp,
              const double* coeffs, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    BandSpec b = make_band(g, band);
    for (int c = 0; c < ncomp; ++c)
      scalar_out(embed(bscalar_in(b, coeffs + (size_t)c * b.size() * 2)), out + (size_t)c * g.size());
  });
}

int ref_project(int d, const int* dims, const double* h, const int* band, int ncomp,
                const double* field, double* coeffs) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    BandSpec b = make_band(g, band);
    for (int c = 0; c < ncomp; ++c)
      bscalar_out(project(scalar_in(g, field + (size_t)c * g.size()), b), coeffs + (size_t)c * b.size() * 2);
  });
}

// op: 0 star(s,s) 1 star(s,vec) 2 star_dot 3 band_jac_mul 4 band_jacT_mul
//     5 band_gradient(s) 6 band_divergence(vec) 7 sobolev(vec) 8 sobolev^-1(vec)
int ref_band_op(int op, int d, const int* dims, const double* h, const int* band, const double* a,
                const double* b_, double* out, double alpha, int s) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    BandSpec b = make_band(g, band);
    const size_t vs = (size_t)b.size() * 2;
    switch (op) {
      case 0: bscalar_out(star(bscalar_in(b, a), bscalar_in(b, b_)), out); break;
      case 1: bvector_out(star(bscalar_in(b, a), bvector_in(b, b_)), out); break;
      case 2: bscalar_out(star_dot(bvector_in(b, a), bvector_in(b, b_)), out); break;
      case 3: bvector_out(band_jac_mul(bvector_in(b, a), bvector_in(b, b_)), out); break;
      case 4: bvector_out(band_jacT_mul(bvector_in(b, a), bvector_in(b, b_)), out); break;
      case 5: bvector_out(band_gradient(bscalar_in(b, a)), out); break;
      case 6: bscalar_out(band_divergence(bvector_in(b, a)), out); break;
      case 7: bvector_out(SobolevOperator(alpha, s).apply(bvector_in(b, a), false), out); break;
      case 8: bvector_out(SobolevOperator(alpha, s).apply(bvector_in(b, a), true), out); break;
      default: throw Error("ref_band_op: bad op");
    }
    (void)vs;
  });
}

double ref_band_inner(int d, const int* dims, const double* h, const int* band, int ncomp,
                      const double* x, const double* y) {
  GridSpec g = make_grid(d, dims, h);
  BandSpec b = make_band(g, band);
  if (ncomp == 1) return band_inner(bscalar_in(b, x), bscalar_in(b, y));
  return band_inner(bvector_in(b, x), bvector_in(b, y));
}

int ref_spectral_gradient(int d, const int* dims, const double* h, const double* f, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    vector_out(spectral_gradient(scalar_in(g, f)), out);
  });
}

// ---- interp.hpp -------------------------------------------------------------
int ref_spline_coefficients(int d, const int* dims, const double* h, const double* f, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    scalar_out(spline_coefficients(scalar_in(g, f)), out);
  });
}

// kind 0 linear, 1 cubic, 2 nearest
int ref_warp(int d, const int* dims, const double* h, int ncomp, const double* f, const double* pts,
             int kind, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    VectorField P = vector_in(g, pts);
    for (int c = 0; c < ncomp; ++c) {
      ScalarField fc = scalar_in(g, f + (size_t)c * g.size());
      ScalarField r = kind == 2 ? warp_nearest(fc, P) : warp(fc, P, kind == 1 ? Interp::cubic : Interp::linear);
      scalar_out(r, out + (size_t)c * g.size());
    }
  });
}

// ---- transport.hpp ----------------------------------------------------------
// departure points of a band velocity (stationary), dir 0 fwd / 1 bwd
int ref_departure(int d, const int* dims, const double* h, const int* band, int nt, const double* v,
                  int dir, double* pts) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    BandSpec b = make_band(g, band);
    VelocityProvider<BandVectorField> prov(TV::stationary(bvector_in(b, v), nt), nt);
    vector_out(prov.departure(0, dir == 0 ? Direction::forward : Direction::backward), pts);
  });
}

int ref_advect_band(int d, const int* dims, const double* h, const int* band, int ncomp, const double* q,
                    const double* pts, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    BandSpec b = make_band(g, band);
    VectorField P = vector_in(g, pts);
    if (ncomp == 1)
      bscalar_out(advect_state(bscalar_in(b, q), P), out);
    else
      bvector_out(advect_state(bvector_in(b, q), P), out);
  });
}

double ref_cfl(int d, const int* dims, const double* h, const int* band, int nt, const double* v) {
  GridSpec g = make_grid(d, dims, h);
  BandSpec b = make_band(g, band);
  VelocityProvider<BandVectorField> prov(TV::stationary(bvector_in(b, v), nt), nt);
  return prov.cfl();
}

// ---- variants.hpp / optimizer.hpp ---------------------------------------------
void* ref_model_create(int d, const int* dims, const double* h, const int* band, const double* I0,
                       const double* I1, int variant, int nt, double sigma2, double alpha, int s,
                       int param) {
  void* out = nullptr;
  guard([&] {
    GridSpec g = make_grid(d, dims, h);
    auto m = std::make_unique<RefModel>();
    m->band = make_band(g, band);
    m->model = std::make_unique<Model<BandAlgebra>>(m->band, scalar_in(g, I0), scalar_in(g, I1));
    m->model->variant = static_cast<Variant>(variant);
    m->model->integrator = Integrator::sl;
    m->model->nt = nt;
    m->model->sigma2 = sigma2;
    m->model->lop = SobolevOperator(alpha, s);
    m->param = param;
    out = m.release();
  });
  return out;
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

// Model::integrator (variants.hpp:35,241): 0 sl, 1 rk4
int ref_model_set_integrator(void* h, int rk4) {
  return guard([&] { static_cast<RefModel*>(h)->model->integrator = rk4 ? Integrator::rk4 : Integrator::sl; });
}

// energies[4] = {E, E_reg, E_data, cfl}
int ref_model_forward(void* h, const double* v, int with_adjoint, double* energies, int* step) {
  auto* m = static_cast<RefModel*>(h);
  return guard(
      [&] {
        TV tv = tv_in(m->band, m->param, m->model->nt, v);
        m->cache = std::make_unique<ForwardCache<BandAlgebra>>(m->model->forward(tv, with_adjoint != 0));
        energies[0] = m->cache->energy;
        energies[1] = m->cache->energy_reg;
        energies[2] = m->cache->energy_data;
        energies[3] = m->cache->cfl;
      },
      step);
}

int ref_model_fields(void* h, double* m1, double* residual) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] {
    if (!m->cache) throw Error("no forward cache");
    if (m1) scalar_out(m->cache->m1, m1);
    if (residual) scalar_out(m->cache->residual, residual);
  });
}

// which: 0 u series, 1 rho series (nt+1 band vectors)
int ref_model_series(void* h, int which, double* out) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] {
    const auto& s = which == 0 ? m->cache->u : m->cache->rho;
    const size_t stride = (size_t)m->band.d() * m->band.size() * 2;
    for (int i = 0; i <= s.nt; ++i) bvector_out(s.node(i), out + i * stride);
  });
}

int ref_model_gradient(void* h, double* g) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] { tv_out(m->model->gradient(*m->cache), g); });
}

int ref_model_hessvec(void* h, const double* dv, double* out) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] {
    TV t = tv_in(m->band, m->param, m->model->nt, dv);
    tv_out(m->model->hessvec(*m->cache, t), out);
  });
}

int ref_model_precondition(void* h, const double* g, double* out) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] {
    TV t = tv_in(m->band, m->param, m->model->nt, g);
    tv_out(m->model->precondition(t), out);
  });
}

double ref_model_energy(void* h, const double* v) {
  auto* m = static_cast<RefModel*>(h);
  double e = 0.0;
  guard([&] { e = m->model->energy(tv_in(m->band, m->param, m->model->nt, v)); });
  return e;
}

// Iteration records: rec[k*10 + {0..9}] = iter, energy, energy_data, energy_reg,
// mse_rel, rel_grad, pcg_iters, pcg_fallback, epsilon, cfl ; pcg residuals in
// pcgres[k*8 + j] (-1 padded).  info[0..3] = n_records, stop reason,
// converged, iterations.
int ref_optimize(void* h, double* v_inout, int max_iter, int pcg_max_iter, double pcg_tol,
                 double grad_tol, double energy_tol, double step_tol, int cap, double* rec,
                 double* pcgres, int* info, double* wall_ms_out) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] {
    TV v0 = tv_in(m->band, m->param, m->model->nt, v_inout);
    OptimizeOptions opt;
    opt.max_iter = max_iter;
    opt.pcg_max_iter = pcg_max_iter;
    opt.pcg_tol = pcg_tol;
    opt.grad_tol = grad_tol;
    opt.energy_tol = energy_tol;
    opt.step_tol = step_tol;
    auto t0 = std::chrono::steady_clock::now();
    OptimizeResult<BandAlgebra> r = optimize(*m->model, v0, opt);
    if (wall_ms_out)
      *wall_ms_out = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    tv_out(r.v, v_inout);
    const int n = std::min<int>(cap, (int)r.history.size());
    for (int k = 0; k < n; ++k) {
      const auto& q = r.history[k];
      double* o = rec + k * 10;
      o[0] = q.iter; o[1] = q.energy; o[2] = q.energy_data; o[3] = q.energy_reg; o[4] = q.mse_rel;
      o[5] = q.rel_grad; o[6] = q.pcg_iters; o[7] = q.pcg_fallback; o[8] = q.epsilon; o[9] = q.cfl;
      for (int j = 0; j < 8; ++j) pcgres[k * 8 + j] = j < (int)q.pcg_residuals.size() ? q.pcg_residuals[j] : -1.0;
    }
    info[0] = (int)r.history.size();
    info[1] = (int)r.stop;
    info[2] = r.converged;
    info[3] = r.iterations;
  });
}

// ---- metrics.hpp ------------------------------------------------------------
// jac[4] = fwd min, fwd max, inv min, inv max ; disp_fwd/disp_inv optional
int ref_maps(void* h, const double* v, double* disp_fwd, double* disp_inv, double* jac) {
  auto* m = static_cast<RefModel*>(h);
  return guard([&] {
    TV tv = tv_in(m->band, m->param, m->model->nt, v);
    RegistrationMaps mp = compute_maps(*m->model, tv);
    if (disp_fwd) vector_out(mp.forward_disp, disp_fwd);
    if (disp_inv) vector_out(mp.inverse_disp, disp_inv);
    ValueRange a = value_range(map_jacobian_determinant(mp.forward_disp));
    ValueRange b = value_range(map_jacobian_determinant(mp.inverse_disp));
    jac[0] = a.min; jac[1] = a.max; jac[2] = b.min; jac[3] = b.max;
  });
}

int ref_jacobian_determinant(int d, const int* dims, const double* h, const double* disp, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    scalar_out(map_jacobian_determinant(vector_in(g, disp)), out);
  });
}

// ---- timing of the reference's own primitives (bench.py cpu_baseline) ---------------
// times[0] one full-grid complex DFT (fft_forward, fft.hpp:69-73)
// times[1] one scalar spline prefilter (spline_coefficients, interp.hpp:80-84)
// times[2] one scalar cubic gather at N points with a prebuilt sampler (warp, interp.hpp:191-200)
// times[3] one vector advect_state of a band field (transport.hpp:71-73), end to end
// mask selects which to run (bit i -> times[i]); unselected entries are left untouched.
int ref_time_ops(int d, const int* dims, const double* h, const int* band, int mask, double* times) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a) {
      return std::chrono::duration<double, std::milli>(clk::now() - a).count();
    };
    GridSpec g = make_grid(d, dims, h);
    BandSpec b = make_band(g, band);
    // smooth field and departure-like points x - 0.3 sin(.)
    ScalarField f(g);
    std::array<int, kMaxDim> idx{};
    for (std::size_t i = 0; i < g.size(); ++i) {
      g.unflatten(i, idx);
      double s = 0.0;
      for (int a = 0; a < g.d; ++a) s += std::sin(2.0 * M_PI * idx[a] / g.dims[a]);
      f.v[i] = s;
    }
    VectorField pts = identity_map(g);
    for (int a = 0; a < g.d; ++a)
      for (std::size_t i = 0; i < g.size(); ++i) pts.comp[a][i] -= 0.3 * std::sin(0.01 * (double)i + a);
    if (mask & 1) {
      std::vector<cplx> buf = fft_of(f);  // plan created here (not timed)
      auto t0 = clk::now();
      fft_forward(g, buf.data());
      times[0] = ms(t0);
    }
    if (mask & 2) {
      auto t0 = clk::now();
      ScalarField c = spline_coefficients(f);
      times[1] = ms(t0);
    }
    if (mask & 4) {
      ScalarSampler s(f, Interp::cubic);
      auto t0 = clk::now();
      ScalarField r = warp(s, pts);
      times[2] = ms(t0);
    }
    if (mask & 8) {
      BandVectorField q(b);
      for (int a = 0; a < g.d; ++a) q.comp[a] = project(f, b).c;
      auto t0 = clk::now();
      BandVectorField r = advect_state(q, pts);
      times[3] = ms(t0);
    }
  });
}

// ---- synth.hpp / io.hpp ---------------------------------------------------------
int ref_blob_pair(int d, const int* dims, const double* h, unsigned long long seed, double* src, double* tgt) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    ImagePair p = blob_pair(g, seed);
    scalar_out(p.source, src);
    scalar_out(p.target, tgt);
  });
}

int ref_two_disc_case(int d, const int* dims, const double* h, unsigned long long seed, double* src,
                      double* tgt, double* src_lab, double* tgt_lab) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    LabelCase c = two_disc_case(g, seed);
    scalar_out(c.source, src);
    scalar_out(c.target, tgt);
    scalar_out(c.source_labels, src_lab);
    scalar_out(c.target_labels, tgt_lab);
  });
}

// ---- metrics.hpp evaluation path: mse_rel, mean_dice, map_jacobian_determinant ------
int ref_evaluate(int d, const int* dims, const double* h, const double* warped, const double* target,
                 const double* source, const double* warped_labels, const double* target_labels,
                 const double* disp, double* mse, double* dice_mean, double* jac_minmax, double* det) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    if (warped && target && source)
      *mse = mse_rel(scalar_in(g, warped), scalar_in(g, target), scalar_in(g, source));
    if (warped_labels && target_labels)
      *dice_mean = mean_dice(scalar_in(g, warped_labels), scalar_in(g, target_labels));
    if (disp) {
      ScalarField j = map_jacobian_determinant(vector_in(g, disp));
      ValueRange r = value_range(j);
      jac_minmax[0] = r.min;
      jac_minmax[1] = r.max;
      if (det) scalar_out(j, det);
    }
  });
}

int ref_random_band_field(int d, const int* dims, const double* h, const int* band, unsigned long long seed,
                          double amplitude, double k0, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    bvector_out(random_band_field(make_band(g, band), seed, amplitude, k0), out);
  });
}

int ref_random_smooth_image(int d, const int* dims, const double* h, unsigned long long seed, double k0,
                            double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    scalar_out(random_smooth_image(g, seed, k0), out);
  });
}

int ref_random_smooth_field(int d, const int* dims, const double* h, unsigned long long seed,
                            double amplitude, double k0, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    vector_out(random_smooth_field(g, seed, amplitude, k0), out);
  });
}

int ref_rescale_unit(int d, const int* dims, const double* h, const double* f, double* out) {
  return guard([&] {
    GridSpec g = make_grid(d, dims, h);
    scalar_out(rescale_unit(scalar_in(g, f)), out);
  });
}

}  // extern "C"
