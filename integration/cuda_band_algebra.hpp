// CudaBandAlgebra: the reference's own Model / optimize templates (proj/include/lddmm,
// optimizer.hpp:86-262) over the B200 engine's C ABI (include/lddmm_cuda.h).
//
// This is the "operator level" drop-in of INTEGRATION.md §2, written as a maintainer
// of the reference would add it: an algebra whose Vec is a device velocity handle,
// plus explicit specialisations of Model<> and ForwardCache<> whose members call the
// ABI.  optimize<CudaBandAlgebra> / pcg_solve<CudaBandAlgebra> are the reference's
// templates, instantiated unchanged; they only touch (optimizer.hpp:86-262,
// variants.hpp:70-117):
//   Model::{source, target, forward, energy, gradient, hessvec, precondition},
//   ForwardCache::{energy, energy_data, energy_reg, cfl, m1, residual},
//   axpy / scaled / rep_inner / linf_norm / all_finite on Vec (found by ADL).
// Stationary parameterisation (the CLI default, lddmm_cli.cpp:29): one device buffer
// per TimeVaryingVelocity node.
#pragma once

#include <lddmm/optimizer.hpp>

#include <string>
#include <utility>

#include "lddmm_cuda.h"

namespace cudaalg {

// The context the Vec handles live in (one per process here, like the reference's
// single-threaded model).
inline lddmm_ctx*& context() {
  static lddmm_ctx* c = nullptr;
  return c;
}

inline void check(int rc, int step = -1) {
  if (rc == LDDMM_OK) return;
  const std::string msg = lddmm_last_error(context());
  if (rc == LDDMM_EDIVERGENCE) throw lddmm::DivergenceError(msg, step);  // core.hpp:32-38
  if (rc == LDDMM_ESHAPE) throw lddmm::ShapeError(msg);
  throw lddmm::Error(msg);
}

// BandVectorField on the device (fp64 band coefficients, reference DFT order).
struct DevVec {
  double* p = nullptr;
  DevVec() { check(lddmm_vel_alloc(context(), &p)); }  // zero (BandVectorField(dom))
  DevVec(const DevVec& o) : DevVec() { check(lddmm_vel_scale(context(), o.p, 1.0, p)); }
  DevVec(DevVec&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevVec& operator=(const DevVec& o) {
    if (this != &o) {
      if (!p) check(lddmm_vel_alloc(context(), &p));
      check(lddmm_vel_scale(context(), o.p, 1.0, p));
    }
    return *this;
  }
  DevVec& operator=(DevVec&& o) noexcept {
    std::swap(p, o.p);
    return *this;
  }
  ~DevVec() {
    if (p) lddmm_vel_free(context(), p);
  }
};

// the band-vector algebra of spectral.hpp:112-185 on the device
inline DevVec axpy(double a, const DevVec& x, const DevVec& y) {
  DevVec r;
  check(lddmm_vel_axpy(context(), a, x.p, y.p, r.p));
  return r;
}
inline DevVec scaled(const DevVec& x, double a) {
  DevVec r;
  check(lddmm_vel_scale(context(), x.p, a, r.p));
  return r;
}
inline double rep_inner(const DevVec& a, const DevVec& b) {  // band_inner (Parseval, h^3 / N)
  double s = 0.0;
  check(lddmm_vel_inner(context(), a.p, b.p, &s));
  return s;
}
inline double linf_norm(const DevVec& a) {
  double m = 0.0;
  check(lddmm_vel_linf(context(), a.p, &m));
  return m;
}
inline bool all_finite(const DevVec& a) {
  int ok = 0;
  check(lddmm_vel_all_finite(context(), a.p, &ok));
  return ok != 0;
}

struct CudaBandAlgebra {
  using Vec = DevVec;
  using Domain = lddmm::BandSpec;
};

}  // namespace cudaalg

namespace lddmm {

template <>
struct ForwardCache<cudaalg::CudaBandAlgebra> {
  bool with_adjoint = false;
  double cfl = 0.0;
  double energy = 0.0, energy_reg = 0.0, energy_data = 0.0;
  ScalarField m1;        // final warped image on the grid (host copy, as the reference keeps it)
  ScalarField residual;  // m1 - I1
};

// Model<BandAlgebra> (variants.hpp:229-548) whose operators run on the device; the
// engine context holds the single forward cache the driver reuses (gradient and the
// Hessian-vector products act on the last adjoint-enabled forward, as in optimize).
template <>
struct Model<cudaalg::CudaBandAlgebra> {
  using Vec = cudaalg::DevVec;
  using TV = TimeVaryingVelocity<Vec>;
  using Cache = ForwardCache<cudaalg::CudaBandAlgebra>;

  BandSpec dom;
  ScalarField source;  // I0
  ScalarField target;  // I1
  int nt = 5;

  Model(BandSpec d, ScalarField I0, ScalarField I1, int nt_)
      : dom(std::move(d)), source(std::move(I0)), target(std::move(I1)), nt(nt_) {
    cudaalg::check(lddmm_set_images(cudaalg::context(), source.v.data(), target.v.data()));
  }

  TV zero_velocity() const { return TV::stationary(Vec(), nt); }

  Cache forward(const TV& v, bool with_adjoint) const {
    lddmm_energies e{};
    int step = -1;
    cudaalg::check(lddmm_forward(cudaalg::context(), v.node(0).p, with_adjoint ? 1 : 0, &e, &step), step);
    Cache c;
    c.with_adjoint = with_adjoint;
    c.energy = e.energy;
    c.energy_reg = e.energy_reg;
    c.energy_data = e.energy_data;
    c.cfl = e.cfl;
    c.m1 = ScalarField(source.grid);
    c.residual = ScalarField(source.grid);
    cudaalg::check(lddmm_get_fields(cudaalg::context(), c.m1.v.data(), c.residual.v.data()));
    return c;
  }

  double energy(const TV& v) const {
    double E = 0.0;
    int step = -1;
    cudaalg::check(lddmm_energy(cudaalg::context(), v.node(0).p, &E, &step), step);
    return E;
  }

  TV gradient(const Cache& c) const {
    detail::require(c.with_adjoint, "gradient requires an adjoint-enabled forward cache");
    Vec g;
    cudaalg::check(lddmm_gradient(cudaalg::context(), g.p));
    return TV::stationary(std::move(g), nt);
  }

  TV hessvec(const Cache&, const TV& dv) const {
    Vec out;
    int step = -1;
    cudaalg::check(lddmm_hessvec(cudaalg::context(), dv.node(0).p, out.p, &step), step);
    return TV::stationary(std::move(out), nt);
  }

  TV precondition(const TV& g) const {
    Vec out;
    cudaalg::check(lddmm_precondition(cudaalg::context(), g.node(0).p, out.p));
    return TV::stationary(std::move(out), nt);
  }
};

}  // namespace lddmm
