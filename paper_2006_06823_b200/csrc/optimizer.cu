// GN-Krylov host driver (restates optimizer.hpp:86-262 over the device model).
#include "optimizer.hpp"

#include <chrono>
#include <cmath>
#include <limits>

namespace lddmm_b200 {

namespace {

double now_ms() {
  using clock = std::chrono::steady_clock;
  return std::chrono::duration<double, std::milli>(clock::now().time_since_epoch()).count();
}

struct PcgInfo {
  int iters = 0;
  bool negative_curvature = false;
  std::vector<double> residuals;
};

struct Vec {
  double2* p;
};
struct Workspace {  // views of the engine's persistent optimizer workspace
  Vec g, rhs, dv, x, r, z, p, hp, trial;
  explicit Workspace(Engine& e)
      : g{e.opt_ws(0)}, rhs{e.opt_ws(1)}, dv{e.opt_ws(2)}, x{e.opt_ws(3)}, r{e.opt_ws(4)}, z{e.opt_ws(5)},
        p{e.opt_ws(6)}, hp{e.opt_ws(7)}, trial{e.opt_ws(8)} {}
};

// optimizer.hpp:86-120; x = 0, r = rhs, z = L^-1 r, p = z
void pcg_solve(Engine& e, Workspace& w, const double2* rhs, int max_iter, double tol, PcgInfo& info,
               OptimizeResult& res) {
  LDDMM_NVTX("pcg_solve");
  info = PcgInfo{};
  const long long n = e.vel_elems();
  e.tv_scaled(rhs, 0.0, w.x.p);
  LDDMM_CUDA(cudaMemcpyAsync(w.r.p, rhs, n * sizeof(double2), cudaMemcpyDeviceToDevice, e.stream()));
  e.precondition(w.r.p, w.z.p);
  double rz = e.tv_inner(w.r.p, w.z.p);
  if (!(rz > 0.0)) return;
  const double res0 = std::sqrt(rz);
  LDDMM_CUDA(cudaMemcpyAsync(w.p.p, w.z.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, e.stream()));
  for (int k = 0; k < max_iter; ++k) {
    e.hessvec(w.p.p, w.hp.p);
    ++res.hessvecs;
    const double php = e.tv_inner(w.p.p, w.hp.p);
    if (!(php > 0.0)) {
      info.negative_curvature = true;
      break;
    }
    const double alpha = rz / php;
    e.tv_axpy(alpha, w.p.p, w.x.p, w.x.p);
    e.tv_axpy(-alpha, w.hp.p, w.r.p, w.r.p);
    e.precondition(w.r.p, w.z.p);
    const double rz_next = std::max(e.tv_inner(w.r.p, w.z.p), 0.0);
    const double rel = std::sqrt(rz_next) / res0;
    info.residuals.push_back(rel);
    info.iters = k + 1;
    if (rel <= tol) break;
    e.tv_axpy(rz_next / rz, w.p.p, w.z.p, w.p.p);
    rz = rz_next;
  }
}

// optimizer.hpp:127-134: a transport blow-up rejects the trial
double trial_energy(Engine& e, const double2* v, OptimizeResult& res) {
  ++res.trials;
  try {
    const double en = e.energy(v);
    return std::isfinite(en) ? en : std::numeric_limits<double>::infinity();
  } catch (const EngineError& err) {
    if (err.status == 2) return std::numeric_limits<double>::infinity();
    throw;
  }
}

}  // namespace

OptimizeResult optimize(Engine& e, double2* v, const OptimizeOptions& opt) {
  OptimizeResult out;
  const long long n = e.vel_elems();
  Workspace w(e);
  const double mse_denom = e.mse_denominator();
  const double cellvol = e.problem().spacing[0] * e.problem().spacing[1] * e.problem().spacing[2];
  auto mse_rel = [&]() { return mse_denom > 0.0 ? e.residual_sumsq() * cellvol / mse_denom : 0.0; };

  Energies c = e.forward(v, true);
  ++out.forwards;
  e.gradient(w.g.p);
  const double g0 = e.tv_linf(w.g.p);

  IterationRecord first;
  first.iter = 0;
  first.energy = c.energy;
  first.energy_data = c.energy_data;
  first.energy_reg = c.energy_reg;
  first.mse_rel = mse_rel();
  first.rel_grad = g0 > 0.0 ? 1.0 : 0.0;
  first.cfl = c.cfl;
  out.history.push_back(first);
  out.final_energy = c.energy;

  if (g0 == 0.0) {
    out.stop = kZeroGradient;
    out.converged = true;
    out.rel_grad = 0.0;
    return out;
  }

  double e_prev = c.energy;
  for (int iter = 1; iter <= opt.max_iter; ++iter) {
    LDDMM_NVTX("GN iteration");
    const double t0 = now_ms();
    PcgInfo pcg;
    e.tv_scaled(w.g.p, -1.0, w.rhs.p);
    pcg_solve(e, w, w.rhs.p, opt.pcg_max_iter, opt.pcg_tol, pcg, out);
    LDDMM_CUDA(cudaMemcpyAsync(w.dv.p, w.x.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, e.stream()));
    double gd = e.tv_inner(w.g.p, w.dv.p);
    bool fallback = false;
    if (!(gd < 0.0)) {  // not a descent direction: preconditioned steepest descent
      e.precondition(w.rhs.p, w.dv.p);
      gd = e.tv_inner(w.g.p, w.dv.p);
      fallback = true;
    }

    double eps = 1.0;
    bool accepted = false;
    for (int trial = 0; trial < opt.armijo_max_trials; ++trial) {
      e.tv_axpy(eps, w.dv.p, v, w.trial.p);
      const double et = trial_energy(e, w.trial.p, out);
      if (et <= e_prev + opt.armijo_c * eps * gd) {
        accepted = true;
        break;
      }
      eps *= 0.5;
    }
    if (!accepted) {
      out.stop = kLineSearchFailure;
      out.converged = false;
      return out;
    }

    e.tv_axpy(eps, w.dv.p, v, v);
    c = e.forward(v, true);
    ++out.forwards;
    e.gradient(w.g.p);
    const double relg = e.tv_linf(w.g.p) / g0;
    out.iterations = iter;
    out.final_energy = c.energy;
    out.rel_grad = relg;

    IterationRecord rec;
    rec.iter = iter;
    rec.energy = c.energy;
    rec.energy_data = c.energy_data;
    rec.energy_reg = c.energy_reg;
    rec.mse_rel = mse_rel();
    rec.rel_grad = relg;
    rec.pcg_iters = pcg.iters;
    rec.pcg_fallback = fallback;
    rec.pcg_residuals = pcg.residuals;
    rec.epsilon = eps;
    rec.cfl = c.cfl;
    rec.wall_ms = now_ms() - t0;
    out.history.push_back(rec);

    const double step_norm = eps * e.tv_linf(w.dv.p);
    const double de = std::abs(e_prev - c.energy) / std::max(std::abs(e_prev), 1e-30);
    e_prev = c.energy;
    if (relg <= opt.grad_tol) {
      out.stop = kGradient;
      out.converged = true;
      return out;
    }
    if (de <= opt.energy_tol) {
      out.stop = kEnergyChange;
      out.converged = true;
      return out;
    }
    if (step_norm <= opt.step_tol) {
      out.stop = kStepSize;
      out.converged = true;
      return out;
    }
  }
  out.stop = kMaxIterations;
  out.converged = false;
  return out;
}

}  // namespace lddmm_b200
