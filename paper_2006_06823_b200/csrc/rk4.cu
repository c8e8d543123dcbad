// RK4 transport (transport.hpp:234-258) for the band representation: the rk4
// branches of the equation solvers (variants.hpp:444-547).  RK4 integrates the
// Eulerian right-hand side, so every stage is a handful of truncated products
// on the small product grid (★, star_dot, band_jac_mul, grad·v) — no full-grid
// gathers; time-dependent inputs are linear interpolations of nodes exactly as
// TimeVaryingVelocity::sample (core.hpp:303-315), VelocityProvider::div_at
// (transport.hpp:164-172) and sample_nodes (transport.hpp:44-54).
#include <cmath>

#include "engine.hpp"

namespace lddmm_b200 {

namespace {

// rk_ slots (band-vector sized)
enum { RK_K1 = 0, RK_K2, RK_K3, RK_K4, RK_TMP, RK_PING, RK_PONG, RK_VT, RK_DT, RK_S1, RK_S2, RK_P };

// node index / weight of a linear interpolation at u in [0, n] (transport.hpp:47-53):
// kind 0 -> node i, 1 -> node i + 1, 2 -> (1 - w) node i + w node i+1
struct Lerp {
  int i;
  double w;
  int kind;
};

Lerp lerp_at(double u, int n) {
  int i = (int)std::floor(u);
  if (i < 0) i = 0;
  if (i >= n) i = n - 1;
  const double w = u - i;
  if (w < 1e-14) return {i, w, 0};
  if (w > 1.0 - 1e-14) return {i, w, 1};
  return {i, w, 2};
}

}  // namespace

void Engine::enqueue_finite(const double2* p, long long n, int step) {
  launch_nonfinite_flag(n, p, part2_.p, slots_.p + 16 + step, stream_);
}

// TimeVaryingVelocity::sample(t) of the provider velocity (core.hpp:303-315)
const double2* Engine::rk_vel_at(const ProviderState& ps, double t, double2* scratch) {
  shape_require(t >= -1e-12 && t <= 1.0 + 1e-12, "sample: t outside [0,1]");
  if (prob_.stationary) return vnode(ps, 0);
  const Lerp l = lerp_at(t * prob_.nt, prob_.nt);
  if (l.kind == 0) return vnode(ps, l.i);
  if (l.kind == 1) return vnode(ps, l.i + 1);
  launch_axpby(vec_elems(), 1.0 - l.w, vnode(ps, l.i), l.w, vnode(ps, l.i + 1), scratch, stream_);
  return scratch;
}

// VelocityProvider::div_at(t) (transport.hpp:164-172)
const double2* Engine::rk_div_at(const ProviderState& ps, double t, double2* scratch) {
  if (prob_.stationary) return divnode(ps, 0);
  const double tc = std::min(std::max(t, 0.0), 1.0);
  const Lerp l = lerp_at(tc * prob_.nt, prob_.nt);
  if (l.kind == 0) return divnode(ps, l.i);
  if (l.kind == 1) return divnode(ps, l.i + 1);
  launch_axpby(kprod(), 1.0 - l.w, divnode(ps, l.i), l.w, divnode(ps, l.i + 1), scratch, stream_);
  return scratch;
}

// TimeVaryingVelocity::sample(t) of a velocity-shaped direction dv (core.hpp:303-315)
const double2* Engine::rk_tv_at(const double2* tv, double t, double2* scratch) {
  shape_require(t >= -1e-12 && t <= 1.0 + 1e-12, "sample: t outside [0,1]");
  if (prob_.stationary) return tv;
  const Lerp l = lerp_at(t * prob_.nt, prob_.nt);
  if (l.kind == 0) return tvnode(tv, l.i);
  if (l.kind == 1) return tvnode(tv, l.i + 1);
  launch_axpby(vec_elems(), 1.0 - l.w, tvnode(tv, l.i), l.w, tvnode(tv, l.i + 1), scratch, stream_);
  return scratch;
}

// sample_nodes(series, t) (transport.hpp:44-54); C double2 per node
const double2* Engine::rk_series_at(const double2* series, long long C, double t, double2* scratch) {
  const int nt = prob_.nt;
  const double tc = std::min(std::max(t, 0.0), 1.0);
  const Lerp l = lerp_at(tc * nt, nt);
  if (l.kind == 0) return series + l.i * C;
  if (l.kind == 1) return series + (l.i + 1) * C;
  launch_axpby(C, 1.0 - l.w, series + l.i * C, l.w, series + (l.i + 1) * C, scratch, stream_);
  return scratch;
}

// out = alpha * star_dot(grad q, w) + beta * add  (Alg::vdot(Alg::grad(q), w)); the i omega
// symbols of grad are applied in the small-grid embed prep
void Engine::graddot(const double2* q, const double2* w, double2* out, double alpha, const double2* add, double beta) {
  const long long K = kprod();
  PrepArgs pa{};
  pa.nf = 6;
  for (int b = 0; b < 3; ++b) pa.f[b] = PrepField{q, SYM_DERIV_X + b, 1.0};
  for (int b = 0; b < 3; ++b) pa.f[3 + b] = PrepField{w + b * K, SYM_NONE, 1.0};
  small_custom(pa, 3, out, 1, alpha, add, beta);
}

// rk4_integrate (transport.hpp:234-258).  series: nt+1 nodes of C double2 (or null:
// ping-pong, last node copied to `last`); init null -> zero.
void Engine::rk4_run(long long C, const double2* init, double2* series, double2* last, bool forward,
                     const RkRhs& rhs) {
  const int nt = prob_.nt;
  const double dt = forward ? 1.0 / nt : -1.0 / nt;
  int at = forward ? 0 : nt;
  auto node_ptr = [&](int i, int parity) -> double2* {
    return series ? series + i * C : rk(parity ? RK_PONG : RK_PING);
  };
  double2* q = node_ptr(at, 0);
  if (!init)
    LDDMM_CUDA(cudaMemsetAsync(q, 0, C * sizeof(double2), stream_));
  else if (init != q)
    LDDMM_CUDA(cudaMemcpyAsync(q, init, C * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  double2 *k1 = rk(RK_K1), *k2 = rk(RK_K2), *k3 = rk(RK_K3), *k4 = rk(RK_K4), *tmp = rk(RK_TMP);
  for (int s = 0; s < nt; ++s) {
    const double t = static_cast<double>(at) / nt;
    rhs(q, t, k1);
    launch_axpy(C, 0.5 * dt, k1, q, tmp, stream_);
    rhs(tmp, t + 0.5 * dt, k2);
    launch_axpy(C, 0.5 * dt, k2, q, tmp, stream_);
    rhs(tmp, t + 0.5 * dt, k3);
    launch_axpy(C, dt, k3, q, tmp, stream_);
    rhs(tmp, t + dt, k4);
    at += forward ? 1 : -1;
    double2* next = node_ptr(at, (s + 1) & 1);
    // next = dt/6 k1 + (dt/3 k2 + (dt/3 k3 + (dt/6 k4 + q)))
    launch_axpy(C, dt / 6.0, k4, q, tmp, stream_);
    launch_axpy(C, dt / 3.0, k3, tmp, next, stream_);
    launch_axpy(C, dt / 3.0, k2, next, tmp, stream_);
    launch_axpy(C, dt / 6.0, k1, tmp, next, stream_);
    enqueue_finite(next, C, s);
    q = next;
  }
  if (last) LDDMM_CUDA(cudaMemcpyAsync(last, q, C * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  finish_finite_checks(nt);
}

// D_t u = v: rhs = v(t) - jac(q, v(t))   (variants.hpp:474-477)
void Engine::rk4_displacement(ProviderState& ps, bool forward, double2* series, double2* last) {
  rk4_run(vec_elems(), nullptr, series, last, forward, [&](const double2* q, double t, double2* out) {
    const double2* vt = rk_vel_at(ps, t, rk(RK_VT));
    small_product(3, q, vt, out, -1.0, vt, 1.0);
  });
}

// D_t rho = -rho div v: rhs = -(div(t) * q + jac(q, v(t)))   (variants.hpp:503-506)
void Engine::rk4_vector_continuity_bwd(ProviderState& ps, const double2* q1, double2* series) {
  rk4_run(vec_elems(), q1, series, nullptr, false, [&](const double2* q, double t, double2* out) {
    const double2* vt = rk_vel_at(ps, t, rk(RK_VT));
    const double2* dvt = rk_div_at(ps, t, rk(RK_DT));
    small_product(3, q, vt, rk(RK_P), 1.0, nullptr, 0.0);
    small_product(1, dvt, q, out, -1.0, rk(RK_P), -1.0);
  });
}

// D_t du = dv - (Du) dv: rhs = -jac(q, v(t)) + (-jac(u(t), dv(t)) + dv(t))   (variants.hpp:541-545)
void Engine::rk4_incremental_displacement(ProviderState& ps, const double2* dv, double2* series) {
  const long long V = vec_elems();
  rk4_run(V, nullptr, series, nullptr, true, [&](const double2* q, double t, double2* out) {
    const double2* vt = rk_vel_at(ps, t, rk(RK_VT));
    const double2* dvt = rk_tv_at(dv, t, rk(RK_S1));
    const double2* ut = rk_series_at(u_.p, V, t, rk(RK_S2));
    small_product(3, ut, dvt, rk(RK_P), -1.0, dvt, 1.0);
    small_product(3, q, vt, out, -1.0, rk(RK_P), 1.0);
  });
}

// D_t m = 0: rhs = -grad(q) . v(t)   (variants.hpp:446-449)
void Engine::rk4_image_forward(ProviderState& ps, const double2* m0, double2* series, double2* last) {
  rk4_run(kprod(), m0, series, last, true, [&](const double2* q, double t, double2* out) {
    graddot(q, rk_vel_at(ps, t, rk(RK_VT)), out, -1.0, nullptr, 0.0);
  });
}

// D_t q = -q div v: rhs = -(q * div(t) + grad(q) . v(t))   (variants.hpp:459-462);
// Jacobian factor D_t U = div v - U div v: rhs = -grad(q) . v(t) + (-q * div(t) + div(t))
// (variants.hpp:490-494)
void Engine::rk4_scalar_continuity_bwd(ProviderState& ps, const double2* q1, double2* series, bool jf) {
  rk4_run(kprod(), q1, series, nullptr, false, [&](const double2* q, double t, double2* out) {
    const double2* vt = rk_vel_at(ps, t, rk(RK_VT));
    const double2* dvt = rk_div_at(ps, t, rk(RK_DT));
    if (jf) {
      small_product(0, q, dvt, rk(RK_P), -1.0, dvt, 1.0);
      graddot(q, vt, out, -1.0, rk(RK_P), 1.0);
    } else {
      graddot(q, vt, rk(RK_P), 1.0, nullptr, 0.0);
      small_product(0, q, dvt, out, -1.0, rk(RK_P), -1.0);
    }
  });
}

// D_t dm = -grad(m)(t) . dv(t): rhs = -(grad(m(t)) . dv(t) + grad(q) . v(t))   (variants.hpp:520-524);
// sample_nodes of the grad m series equals grad of the sampled m series (linear)
void Engine::rk4_incremental_image(ProviderState& ps, const double2* dv, double2* series) {
  const long long S = kprod();
  rk4_run(S, nullptr, series, nullptr, true, [&](const double2* q, double t, double2* out) {
    const double2* vt = rk_vel_at(ps, t, rk(RK_VT));
    const double2* dvt = rk_tv_at(dv, t, rk(RK_S1));
    const double2* mt = rk_series_at(m_ser_.p, S, t, rk(RK_S2));
    graddot(mt, dvt, rk(RK_P), 1.0, nullptr, 0.0);
    graddot(q, vt, out, -1.0, rk(RK_P), -1.0);
  });
}

}  // namespace lddmm_b200
