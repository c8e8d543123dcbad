// Host-side Gauss-Newton-Krylov driver over the device model: a restatement of
// optimizer.hpp:18-262 (OptimizeOptions, StopReason, IterationRecord,
// pcg_solve, trial_energy, optimize) with identical control flow and branch
// order.  Velocities stay on the device; every inner product / norm is one
// device reduction returning a double.
#pragma once

#include <string>
#include <vector>

#include "engine.hpp"

namespace lddmm_b200 {

struct OptimizeOptions {  // optimizer.hpp:18-27
  int max_iter = 50;
  int pcg_max_iter = 5;
  double pcg_tol = 0.1;
  double grad_tol = 1e-2;
  double energy_tol = 1e-4;
  double step_tol = 1e-4;
  double armijo_c = 1e-4;
  int armijo_max_trials = 10;
};

enum StopReason { kGradient = 0, kEnergyChange, kStepSize, kZeroGradient, kMaxIterations, kLineSearchFailure };

struct IterationRecord {  // optimizer.hpp:50-61
  int iter = 0;
  double energy = 0, energy_data = 0, energy_reg = 0;
  double mse_rel = 0, rel_grad = 1;
  int pcg_iters = 0;
  bool pcg_fallback = false;
  double epsilon = 0, cfl = 0, wall_ms = 0;
  std::vector<double> pcg_residuals;
};

struct OptimizeResult {
  std::vector<IterationRecord> history;
  int stop = kMaxIterations;
  bool converged = false;
  int iterations = 0;
  double final_energy = 0, rel_grad = 1;
  int hessvecs = 0, trials = 0, forwards = 0;  // operation counts (bench bookkeeping)
};

// v: device velocity (engine.vel_elems() double2), updated in place with the result.
OptimizeResult optimize(Engine& e, double2* v, const OptimizeOptions& opt);

}  // namespace lddmm_b200
