// lddmm — command-line front end over the C ABI (include/lddmm_cuda.h).
//
// Drop-in for the reference driver (tools/lddmm_cli.cpp): same subcommands
// (register / evaluate / synth), option names, defaults, on-disk formats
// (io.hpp:1-209: little-endian float32 .raw + .json sidecar; report.json,
// convergence.csv, summary.txt) and exit codes (0 ok, 1 usage/input error,
// 2 transport divergence, lddmm_cli.cpp:340-358).  The registration, maps,
// warps, Jacobians and Dice counts run on the GPU through liblddmm_cuda.so;
// this file only parses arguments, reads/writes files and formats reports.
//
// Scope: the band representation on 2-D and 3-D grids, SL-RK2 or RK4 transport.
// --repr spatial exits with status 1 and says so.  `synth` generates 2-D and 3-D blobs/discs fixtures with
// the reference's seeded generators (synth.hpp:20-42,182-259) restated here.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/lddmm_cuda.h"

namespace {

using nlohmann::json;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Divergence : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// grids and fields (core.hpp:42-122, io.hpp:94-178)

struct Grid {
  int d = 0;
  std::array<int, 3> dims{1, 1, 1};
  std::array<double, 3> spacing{1.0, 1.0, 1.0};
  std::size_t size() const {
    std::size_t s = 1;
    for (int a = 0; a < d; ++a) s *= (std::size_t)dims[a];
    return s;
  }
  double extent(int a) const { return dims[a] * spacing[a]; }
  double min_spacing() const {
    double h = spacing[0];
    for (int a = 1; a < d; ++a) h = std::min(h, spacing[a]);
    return h;
  }
  double cell_volume() const {
    double v = 1.0;
    for (int a = 0; a < d; ++a) v *= spacing[a];
    return v;
  }
  void validate() const {
    if (d < 2 || d > 3) throw InputError("grid dimension must be 2 or 3");
    for (int a = 0; a < d; ++a) {
      if (dims[a] < 4 || dims[a] % 2 != 0) throw InputError("grid dims must be even and >= 4");
      if (!(spacing[a] > 0.0)) throw InputError("grid spacing must be positive");
    }
  }
  bool operator==(const Grid& o) const {
    if (d != o.d) return false;
    for (int a = 0; a < d; ++a)
      if (dims[a] != o.dims[a] || spacing[a] != o.spacing[a]) return false;
    return true;
  }
  void unflatten(std::size_t i, std::array<int, 3>& idx) const {
    for (int a = d - 1; a >= 0; --a) {
      idx[a] = (int)(i % (std::size_t)dims[a]);
      i /= (std::size_t)dims[a];
    }
  }
};

enum class Kind { scalar, vector, labels };

const char* kind_name(Kind k) {
  return k == Kind::vector ? "vector" : (k == Kind::labels ? "labels" : "scalar");
}

struct Field {
  Grid grid;
  Kind kind = Kind::scalar;
  int components = 1;
  std::vector<double> v;  // components * N, component-major
};

std::string strip_raw(const std::string& p) {
  const std::string suf = ".raw";
  if (p.size() > suf.size() && p.compare(p.size() - suf.size(), suf.size(), suf) == 0)
    return p.substr(0, p.size() - suf.size());
  return p;
}

void ensure_parent(const std::string& path) {
  std::filesystem::path p(path);
  if (p.has_parent_path() && !p.parent_path().empty()) std::filesystem::create_directories(p.parent_path());
}

std::string join_path(const std::string& dir, const std::string& name) {
  return (std::filesystem::path(dir) / name).string();
}

void write_json(const std::string& path, const json& j) {
  ensure_parent(path);
  std::ofstream f(path);
  if (!f) throw InputError("cannot open for writing: " + path);
  f << j.dump(2) << "\n";
}

// write_field (io.hpp:100-120): float32 payload + sidecar
void write_field(const std::string& path, const Field& fld) {
  const std::string base = strip_raw(path);
  std::vector<float> data(fld.v.size());
  for (std::size_t i = 0; i < fld.v.size(); ++i) data[i] = (float)fld.v[i];
  ensure_parent(base + ".raw");
  {
    std::ofstream f(base + ".raw", std::ios::binary);
    if (!f) throw InputError("cannot open for writing: " + base + ".raw");
    f.write(reinterpret_cast<const char*>(data.data()), (std::streamsize)(data.size() * sizeof(float)));
    if (!f) throw InputError("write failed: " + base + ".raw");
  }
  json j;
  j["dims"] = std::vector<int>(fld.grid.dims.begin(), fld.grid.dims.begin() + fld.grid.d);
  j["spacing"] = std::vector<double>(fld.grid.spacing.begin(), fld.grid.spacing.begin() + fld.grid.d);
  j["kind"] = kind_name(fld.kind);
  j["components"] = fld.components;
  write_json(base + ".json", j);
}

// load_field (io.hpp:130-164)
Field load_field(const std::string& path) {
  const std::string base = strip_raw(path);
  std::ifstream sf(base + ".json");
  if (!sf) throw InputError("cannot open sidecar: " + base + ".json");
  json j;
  try {
    sf >> j;
  } catch (const json::exception& e) {
    throw InputError("bad sidecar " + base + ".json: " + e.what());
  }
  Field out;
  try {
    std::vector<int> dims = j.at("dims").get<std::vector<int>>();
    std::vector<double> spacing = j.at("spacing").get<std::vector<double>>();
    if (dims.size() < 2 || dims.size() > 3) throw InputError("grid dimension must be 2 or 3");
    if (spacing.size() != dims.size()) throw InputError("dims/spacing size mismatch");
    out.grid.d = (int)dims.size();
    for (int a = 0; a < out.grid.d; ++a) {
      out.grid.dims[a] = dims[a];
      out.grid.spacing[a] = spacing[a];
    }
    out.grid.validate();
    const std::string kind = j.at("kind").get<std::string>();
    if (kind == "scalar") out.kind = Kind::scalar;
    else if (kind == "vector") out.kind = Kind::vector;
    else if (kind == "labels") out.kind = Kind::labels;
    else throw InputError("bad sidecar " + base + ".json: unknown kind \"" + kind + "\"");
    out.components = j.at("components").get<int>();
  } catch (const json::exception& e) {
    throw InputError("bad sidecar " + base + ".json: " + e.what());
  }
  const bool want_vector = out.kind == Kind::vector;
  if (out.components != (want_vector ? out.grid.d : 1))
    throw InputError("sidecar components inconsistent with kind for " + base);
  const std::size_t n = out.grid.size() * (std::size_t)out.components;
  std::ifstream f(base + ".raw", std::ios::binary | std::ios::ate);
  if (!f) throw InputError("cannot open: " + base + ".raw");
  const auto bytes = (std::size_t)f.tellg();
  if (bytes != n * sizeof(float))
    throw InputError("payload size mismatch for " + base + ".raw: got " + std::to_string(bytes) +
                     " bytes, sidecar implies " + std::to_string(n * sizeof(float)));
  f.seekg(0);
  std::vector<float> data(n);
  f.read(reinterpret_cast<char*>(data.data()), (std::streamsize)bytes);
  if (!f) throw InputError("read failed: " + base + ".raw");
  out.v.assign(data.begin(), data.end());
  return out;
}

Field load_scalar(const std::string& path) {
  Field f = load_field(path);
  if (f.kind == Kind::vector) throw InputError(path + ": expected a scalar or label field, got a vector field");
  return f;
}

Field load_vector(const std::string& path) {
  Field f = load_field(path);
  if (f.kind != Kind::vector) throw InputError(path + ": expected a vector field");
  return f;
}

// rescale_unit (io.hpp:166-178)
void rescale_unit(Field& f) {
  double lo = f.v.empty() ? 0.0 : f.v[0], hi = lo;
  for (double x : f.v) {
    lo = std::min(lo, x);
    hi = std::max(hi, x);
  }
  if (hi > lo) {
    const double s = 1.0 / (hi - lo);
    for (double& x : f.v) x = (x - lo) * s;
  } else {
    std::fill(f.v.begin(), f.v.end(), 0.0);
  }
}

// mse_rel (metrics.hpp:82-89): host fp64 in the reference's loop order
double mse_rel(const Field& warped, const Field& target, const Field& source) {
  const std::size_t n = target.v.size();
  double sn = 0.0, sd = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    const double a = -1.0 * target.v[i] + warped.v[i];
    sn += a * a;
  }
  for (std::size_t i = 0; i < n; ++i) {
    const double b = -1.0 * target.v[i] + source.v[i];
    sd += b * b;
  }
  const double cv = target.grid.cell_volume();
  const double d = sd * cv;
  if (d <= 0.0) return 0.0;
  return (sn * cv) / d;
}

// ---------------------------------------------------------------------------
// the GPU engine

const char* stop_name(int s) {
  static const char* names[] = {"gradient", "energy_change", "step_size", "zero_gradient", "max_iterations",
                                "line_search_failure"};
  return (s >= 0 && s < 6) ? names[s] : "unknown";
}

struct Ctx {
  lddmm_ctx* h = nullptr;
  explicit Ctx(const lddmm_problem& p) {
    const int rc = lddmm_create(&p, 0, &h);
    if (rc != LDDMM_OK) throw InputError(std::string("engine: ") + lddmm_last_error(nullptr));
  }
  ~Ctx() {
    if (h) lddmm_destroy(h);
  }
  void check(int rc, int step = -1) const {
    if (rc == LDDMM_OK) return;
    const std::string msg = lddmm_last_error(h);
    if (rc == LDDMM_EDIVERGENCE) throw Divergence(msg);
    if (rc == LDDMM_ESHAPE) throw InputError(msg);
    throw std::runtime_error(msg);
  }
};

void require_2d_or_3d(const Grid& g) {
  if (g.d != 2 && g.d != 3) throw InputError("grid dimension must be 2 or 3 (got d = " + std::to_string(g.d) + ")");
}

lddmm_problem problem_for(const Grid& g, int band, int nt, int variant, int param, double alpha, int s,
                          double sigma2) {
  lddmm_problem p{};
  p.d = g.d;  // 2-D grids run z-replicated inside the engine (lddmm_cuda.h)
  for (int a = 0; a < 3; ++a) {
    p.dims[a] = a < g.d ? g.dims[a] : 1;
    p.spacing[a] = a < g.d ? g.spacing[a] : 1.0;
    p.band[a] = a < g.d ? std::min(band, g.dims[a]) : 1;  // lddmm_cli.cpp:222-224
  }
  p.nt = nt;
  p.variant = variant;
  p.parameterization = param;
  p.alpha = alpha;
  p.s = s;
  p.sigma2 = sigma2;
  return p;
}

// ---------------------------------------------------------------------------
// options (lddmm_cli.cpp:21-52, 280-330)

struct RegOpts {
  std::string source, target, out;
  std::string source_labels, target_labels;
  std::string v0_path;
  std::string variant = "original";
  std::string integrator = "sl";
  std::string repr = "band";
  std::string param = "stationary";
  int band = 32;
  int nt = 0;
  double alpha = 0.0025;
  int s = 2;
  double sigma2 = 1.0;
  int max_iter = 50;
  int pcg_iter = 5;
  bool no_rescale = false;
};

struct EvalOpts {
  std::string source, target, warped, warped_labels, target_labels, displacement, out;
};

struct SynthOpts {
  std::string kind = "blobs";
  std::string out;
  int n = 64;
  int d = 2;
  double spacing = 1.0;
  std::uint64_t seed = 42;
};

int parse_variant(const std::string& s) {
  if (s == "original") return LDDMM_ORIGINAL;
  if (s == "state_equation") return LDDMM_STATE_EQUATION;
  if (s == "deformation_state_equation") return LDDMM_DEFORMATION_STATE_EQUATION;
  throw InputError("unknown variant: " + s);
}

// ---------------------------------------------------------------------------
// register (lddmm_cli.cpp:101-232)

std::string grid_to_string(const Grid& g) {
  std::ostringstream os;
  for (int a = 0; a < g.d; ++a) os << (a ? "x" : "") << g.dims[a];
  return os.str();
}

int do_register(const RegOpts& o) {
  Field I0 = load_scalar(o.source);
  Field I1 = load_scalar(o.target);
  if (!(I0.grid == I1.grid)) throw InputError("source and target must share one grid");
  if (!o.no_rescale) {
    rescale_unit(I0);
    rescale_unit(I1);
  }
  if (o.integrator != "sl" && o.integrator != "rk4")
    throw InputError("unknown integrator: " + o.integrator + " (expected sl or rk4)");
  const int nt = o.nt > 0 ? o.nt : (o.integrator == "rk4" ? 25 : 5);
  const int variant = parse_variant(o.variant);
  int param;
  if (o.param == "stationary") param = LDDMM_STATIONARY;
  else if (o.param == "nonstationary") param = LDDMM_NONSTATIONARY;
  else throw InputError("unknown parameterization: " + o.param);
  if (o.repr != "band" && o.repr != "bl" && o.repr != "spatial")
    throw InputError("unknown representation: " + o.repr + " (expected spatial or band)");
  if (o.repr == "spatial")
    throw InputError("--repr spatial is not part of the B200 engine (band representation only)");
  if (!(o.band >= 4 && o.band % 2 == 0)) throw InputError("--band must be even and >= 4");
  require_2d_or_3d(I0.grid);
  const Grid& g = I0.grid;
  const std::size_t N = g.size();

  lddmm_problem prob = problem_for(g, o.band, nt, variant, param, o.alpha, o.s, o.sigma2);
  prob.integrator = o.integrator == "rk4" ? LDDMM_RK4 : LDDMM_SL;
  Ctx ctx(prob);
  ctx.check(lddmm_set_images(ctx.h, I0.v.data(), I1.v.data()));
  double* v = nullptr;
  ctx.check(lddmm_vel_alloc(ctx.h, &v));
  struct VelFree {
    lddmm_ctx* h;
    double* v;
    ~VelFree() { lddmm_vel_free(h, v); }
  } vel_free{ctx.h, v};
  if (!o.v0_path.empty()) {
    Field w = load_vector(o.v0_path);
    if (!(w.grid == g)) throw InputError("--v0 grid does not match the images");
    ctx.check(lddmm_vel_from_spatial(ctx.h, w.v.data(), v));
  }
  lddmm_options opt;
  lddmm_default_options(&opt);
  opt.max_iter = o.max_iter;
  opt.pcg_max_iter = o.pcg_iter;
  std::vector<lddmm_iteration_record> hist((std::size_t)o.max_iter + 2);
  lddmm_result res{};
  const auto t0 = std::chrono::steady_clock::now();
  ctx.check(lddmm_optimize(ctx.h, v, &opt, hist.data(), (int)hist.size(), &res));
  const double wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  hist.resize((std::size_t)res.n_history);

  // compute_maps, warp(I0, forward_pts, cubic), Jacobian ranges (metrics.hpp:24-79)
  Field fwd{g, Kind::vector, g.d, std::vector<double>(g.d * N)};
  Field inv{g, Kind::vector, g.d, std::vector<double>(g.d * N)};
  double jac[4];
  ctx.check(lddmm_maps(ctx.h, v, fwd.v.data(), inv.v.data(), jac));
  Field warped{g, Kind::scalar, 1, std::vector<double>(N)};
  ctx.check(lddmm_warp(ctx.h, LDDMM_INTERP_CUBIC, I0.v.data(), 1, fwd.v.data(), warped.v.data()));

  write_field(join_path(o.out, "displacement_forward"), fwd);
  write_field(join_path(o.out, "displacement_inverse"), inv);
  write_field(join_path(o.out, "warped_source"), warped);
  const int nodes = param == LDDMM_STATIONARY ? 1 : nt + 1;
  for (int i = 0; i < nodes; ++i) {
    Field vel{g, Kind::vector, g.d, std::vector<double>(g.d * N)};
    ctx.check(lddmm_vel_to_spatial(ctx.h, v, i, vel.v.data()));
    if (param == LDDMM_STATIONARY) {
      write_field(join_path(o.out, "velocity"), vel);
    } else {
      char name[32];
      std::snprintf(name, sizeof(name), "velocity_%02d", i);
      write_field(join_path(o.out, name), vel);
    }
  }

  double dice_mean = -1.0;
  if (!o.source_labels.empty()) {
    Field labels = load_scalar(o.source_labels);
    if (!(labels.grid == g)) throw InputError("--source-labels grid mismatch");
    Field wl{g, Kind::labels, 1, std::vector<double>(N)};
    ctx.check(lddmm_warp(ctx.h, LDDMM_INTERP_NEAREST, labels.v.data(), 1, fwd.v.data(), wl.v.data()));
    write_field(join_path(o.out, "warped_labels"), wl);
    if (!o.target_labels.empty()) {
      Field tl = load_scalar(o.target_labels);
      if (!(tl.grid == g)) throw InputError("--target-labels grid mismatch");
      ctx.check(lddmm_mean_dice(ctx.h, wl.v.data(), tl.v.data(), &dice_mean));
    }
  }

  const double mse_initial = hist.front().mse_rel;
  const double mse_final = hist.back().mse_rel;
  json rep;
  rep["variant"] = o.variant;
  rep["integrator"] = o.integrator;
  rep["representation"] = o.repr;
  rep["parameterization"] = o.param;
  rep["nt"] = nt;
  rep["alpha"] = o.alpha;
  rep["s"] = o.s;
  rep["sigma2"] = o.sigma2;
  rep["dims"] = std::vector<int>(g.dims.begin(), g.dims.begin() + g.d);
  std::vector<int> bounds;
  for (int a = 0; a < g.d; ++a) bounds.push_back(std::min(o.band, g.dims[a]));
  rep["band"] = bounds;
  rep["rescaled_inputs"] = !o.no_rescale;
  rep["converged"] = res.converged != 0;
  rep["stop_reason"] = stop_name(res.stop_reason);
  rep["iterations"] = res.iterations;
  rep["final_energy"] = res.final_energy;
  rep["rel_grad"] = res.rel_grad;
  rep["mse_rel_initial"] = mse_initial;
  rep["mse_rel_final"] = mse_final;
  rep["cfl"] = hist.back().cfl;
  rep["jacobian_forward"] = {{"min", jac[0]}, {"max", jac[1]}};
  rep["jacobian_inverse"] = {{"min", jac[2]}, {"max", jac[3]}};
  if (dice_mean >= 0.0) rep["dice_mean"] = dice_mean;
  rep["wall_ms"] = wall_ms;
  write_json(join_path(o.out, "report.json"), rep);

  // write_convergence_csv (io.hpp:188-200)
  {
    const std::string path = join_path(o.out, "convergence.csv");
    ensure_parent(path);
    std::ofstream f(path);
    if (!f) throw InputError("cannot open for writing: " + path);
    f << "iter,energy,mse_rel,rel_grad,pcg_iters,epsilon,wall_ms\n";
    char buf[512];
    for (const auto& r : hist) {
      std::snprintf(buf, sizeof(buf), "%d,%.17g,%.17g,%.17g,%d,%.17g,%.17g\n", r.iter, r.energy, r.mse_rel,
                    r.rel_grad, r.pcg_iters, r.epsilon, r.wall_ms);
      f << buf;
    }
  }

  std::ostringstream sum;
  sum << "registration summary\n"
      << "  variant:        " << o.variant << "\n"
      << "  integrator:     " << o.integrator << " (nt=" << nt << ")\n"
      << "  representation: " << o.repr << "\n"
      << "  parameterization: " << o.param << "\n"
      << "  grid:           " << grid_to_string(g) << "\n"
      << "  iterations:     " << res.iterations << "\n"
      << "  stop reason:    " << stop_name(res.stop_reason) << "\n"
      << "  converged:      " << (res.converged ? "yes" : "no") << "\n"
      << "  energy:         " << hist.front().energy << " -> " << res.final_energy << "\n"
      << "  mse_rel:        " << mse_initial << " -> " << mse_final << "\n"
      << "  rel_grad:       " << res.rel_grad << "\n"
      << "  jacobian fwd:   [" << jac[0] << ", " << jac[1] << "]\n"
      << "  jacobian inv:   [" << jac[2] << ", " << jac[3] << "]\n";
  if (dice_mean >= 0.0) sum << "  dice mean:      " << dice_mean << "\n";
  sum << "  wall:           " << wall_ms << " ms\n";
  {
    const std::string path = join_path(o.out, "summary.txt");
    ensure_parent(path);
    std::ofstream f(path);
    if (!f) throw InputError("cannot open for writing: " + path);
    f << sum.str();
  }
  std::cout << sum.str();
  return 0;
}

// ---------------------------------------------------------------------------
// evaluate (lddmm_cli.cpp:236-262)

int do_evaluate(const EvalOpts& o) {
  Field src = load_scalar(o.source);
  Field tgt = load_scalar(o.target);
  if (!(src.grid == tgt.grid)) throw InputError("source and target must share one grid");
  Field warped = o.warped.empty() ? src : load_scalar(o.warped);
  if (!(warped.grid == tgt.grid)) throw InputError("--warped grid mismatch");
  json rep;
  rep["mse_rel"] = mse_rel(warped, tgt, src);
  const bool want_dice = !o.warped_labels.empty() && !o.target_labels.empty();
  if (want_dice || !o.displacement.empty()) {
    require_2d_or_3d(tgt.grid);
    // an engine context on this grid (the smallest band; only grid buffers are used)
    Ctx ctx(problem_for(tgt.grid, 4, 1, LDDMM_DEFORMATION_STATE_EQUATION, LDDMM_STATIONARY, 0.0025, 2, 1.0));
    if (want_dice) {
      Field wl = load_scalar(o.warped_labels);
      Field tl = load_scalar(o.target_labels);
      if (!(wl.grid == tl.grid) || !(wl.grid == tgt.grid)) throw InputError("label grids mismatch");
      double dm = 0.0;
      ctx.check(lddmm_mean_dice(ctx.h, wl.v.data(), tl.v.data(), &dm));
      rep["dice_mean"] = dm;
    }
    if (!o.displacement.empty()) {
      Field disp = load_vector(o.displacement);
      if (!(disp.grid == tgt.grid)) throw InputError("--displacement grid mismatch");
      double mm[2];
      ctx.check(lddmm_jacobian(ctx.h, disp.v.data(), nullptr, mm));
      rep["jacobian"] = {{"min", mm[0]}, {"max", mm[1]}};
    }
  }
  std::cout << rep.dump(2) << "\n";
  if (!o.out.empty()) write_json(o.out, rep);
  return 0;
}

// ---------------------------------------------------------------------------
// synth (lddmm_cli.cpp:264-296; generators of synth.hpp:20-259)

struct Rng {  // mt19937_64 + Box-Muller, synth.hpp:20-42
  std::mt19937_64 eng;
  explicit Rng(std::uint64_t seed) : eng(seed) {}
  double uniform() { return std::ldexp((double)eng(), -64); }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
};

double periodic_r2(const Grid& g, const std::array<int, 3>& idx, const std::array<double, 3>& c) {
  double r2 = 0.0;
  for (int a = 0; a < g.d; ++a) {
    const double L = g.extent(a);
    double dx = idx[a] * g.spacing[a] - c[a];
    dx -= L * std::round(dx / L);
    r2 += dx * dx;
  }
  return r2;
}

void add_gaussian(Field& f, const std::array<double, 3>& c, double sigma, double amp) {
  std::array<int, 3> idx{};
  const double inv = 1.0 / (2.0 * sigma * sigma);
  for (std::size_t i = 0; i < f.v.size(); ++i) {
    f.grid.unflatten(i, idx);
    f.v[i] += amp * std::exp(-periodic_r2(f.grid, idx, c) * inv);
  }
}

void add_tanh_disc(Field& f, const std::array<double, 3>& c, double radius, double edge, double amp) {
  std::array<int, 3> idx{};
  for (std::size_t i = 0; i < f.v.size(); ++i) {
    f.grid.unflatten(i, idx);
    const double r = std::sqrt(periodic_r2(f.grid, idx, c));
    f.v[i] += amp * 0.5 * (1.0 - std::tanh((r - radius) / edge));
  }
}

void paint_disc_label(Field& f, const std::array<double, 3>& c, double radius, double label) {
  std::array<int, 3> idx{};
  for (std::size_t i = 0; i < f.v.size(); ++i) {
    f.grid.unflatten(i, idx);
    if (periodic_r2(f.grid, idx, c) <= radius * radius) f.v[i] = label;
  }
}

int do_synth(const SynthOpts& o) {
  if (o.d != 2 && o.d != 3) throw InputError("--d must be 2 or 3");
  Grid g;
  g.d = o.d;
  for (int a = 0; a < o.d; ++a) {
    g.dims[a] = o.n;
    g.spacing[a] = o.spacing;
  }
  g.validate();
  auto blank = [&](Kind k) { return Field{g, k, 1, std::vector<double>(g.size(), 0.0)}; };
  if (o.kind == "blobs") {  // blob_pair (synth.hpp:190-211)
    Rng rng(o.seed);
    Field s = blank(Kind::scalar), t = blank(Kind::scalar);
    const int n_blobs = 2 + (int)(rng.uniform() * 2.0);
    for (int k = 0; k < n_blobs; ++k) {
      std::array<double, 3> c{};
      for (int a = 0; a < g.d; ++a) c[a] = rng.uniform(0.3, 0.7) * g.extent(a);
      const double sigma = rng.uniform(0.09, 0.14) * g.extent(0);
      const double amp = rng.uniform(0.6, 1.0);
      add_gaussian(s, c, sigma, amp);
      std::array<double, 3> ct = c;
      for (int a = 0; a < g.d; ++a) ct[a] += rng.uniform(-0.05, 0.05) * g.extent(a);
      const double sigma_t = sigma * rng.uniform(0.88, 1.12);
      add_gaussian(t, ct, sigma_t, amp);
    }
    rescale_unit(s);
    rescale_unit(t);
    write_field(join_path(o.out, "source"), s);
    write_field(join_path(o.out, "target"), t);
  } else if (o.kind == "discs") {  // two_disc_case (synth.hpp:222-257)
    Rng rng(o.seed);
    Field s = blank(Kind::scalar), t = blank(Kind::scalar);
    Field sl = blank(Kind::labels), tl = blank(Kind::labels);
    const double L = g.extent(0);
    const double edge = 1.5 * g.min_spacing();
    std::array<double, 3> c1{}, c2{};
    c1[0] = (0.34 + rng.uniform(-0.03, 0.03)) * L;
    c1[1] = (0.50 + rng.uniform(-0.03, 0.03)) * g.extent(1);
    c2[0] = (0.66 + rng.uniform(-0.03, 0.03)) * L;
    c2[1] = (0.50 + rng.uniform(-0.03, 0.03)) * g.extent(1);
    const double r1 = rng.uniform(0.11, 0.13) * L;
    const double r2 = rng.uniform(0.08, 0.10) * L;
    std::array<double, 3> t1 = c1, t2 = c2;
    t1[0] += rng.uniform(0.04, 0.08) * L;
    t1[1] += rng.uniform(-0.06, 0.06) * g.extent(1);
    t2[0] -= rng.uniform(0.04, 0.08) * L;
    t2[1] += rng.uniform(-0.06, 0.06) * g.extent(1);
    const double rt1 = r1 * rng.uniform(1.05, 1.2);
    const double rt2 = r2 * rng.uniform(0.8, 0.95);
    add_tanh_disc(s, c1, r1, edge, 1.0);
    add_tanh_disc(s, c2, r2, edge, 0.6);
    add_tanh_disc(t, t1, rt1, edge, 1.0);
    add_tanh_disc(t, t2, rt2, edge, 0.6);
    rescale_unit(s);
    rescale_unit(t);
    paint_disc_label(sl, c1, r1, 1.0);
    paint_disc_label(sl, c2, r2, 2.0);
    paint_disc_label(tl, t1, rt1, 1.0);
    paint_disc_label(tl, t2, rt2, 2.0);
    write_field(join_path(o.out, "source"), s);
    write_field(join_path(o.out, "target"), t);
    write_field(join_path(o.out, "source_labels"), sl);
    write_field(join_path(o.out, "target_labels"), tl);
  } else if (o.kind == "rotation") {
    throw InputError("synth --kind rotation transports with the spatial SL integrator, which is not part of the "
                     "B200 engine");
  } else {
    throw InputError("unknown synth kind: " + o.kind + " (expected blobs, discs, or rotation)");
  }
  std::cout << "wrote " << o.kind << " fixtures to " << o.out << "\n";
  return 0;
}

// ---------------------------------------------------------------------------
// argument parsing (the CLI11 surface of lddmm_cli.cpp:280-330)

struct Opt {
  std::string name;
  std::string help;
  bool flag = false;
  bool required = false;
  std::function<void(const std::string&)> set;
};

template <class T>
std::function<void(const std::string&)> setter(T& dst) {
  return [&dst](const std::string& s) {
    std::istringstream is(s);
    T v{};
    is >> v;
    if (is.fail() || !is.eof()) throw UsageError("invalid value '" + s + "'");
    dst = v;
  };
}
template <>
std::function<void(const std::string&)> setter<std::string>(std::string& dst) {
  return [&dst](const std::string& s) { dst = s; };
}

void usage(std::ostream& os) {
  os << "diffeomorphic image registration on periodic grids (B200 engine)\n"
        "Usage: lddmm SUBCOMMAND [OPTIONS]\n\n"
        "Subcommands:\n"
        "  register   register a source image onto a target\n"
        "  evaluate   compute metrics on existing fields\n"
        "  synth      generate synthetic test fixtures\n";
}

void sub_usage(std::ostream& os, const std::string& sub, const std::vector<Opt>& opts) {
  os << "Usage: lddmm " << sub << " [OPTIONS]\n\nOptions:\n  -h,--help  print this help\n";
  for (const auto& o : opts)
    os << "  --" << o.name << (o.flag ? "" : " VALUE") << (o.required ? " REQUIRED" : "") << "  " << o.help << "\n";
}

// returns false when --help was printed
bool parse(int argc, char** argv, const std::string& sub, std::vector<Opt>& opts) {
  std::map<std::string, bool> seen;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "-h" || a == "--help") {
      sub_usage(std::cout, sub, opts);
      return false;
    }
    if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
    std::string name = a.substr(2), value;
    bool has_value = false;
    const auto eq = name.find('=');
    if (eq != std::string::npos) {
      value = name.substr(eq + 1);
      name = name.substr(0, eq);
      has_value = true;
    }
    auto it = std::find_if(opts.begin(), opts.end(), [&](const Opt& o) { return o.name == name; });
    if (it == opts.end()) throw UsageError("unknown option: --" + name);
    if (it->flag) {
      if (has_value) throw UsageError("--" + name + " takes no value");
      it->set("1");
    } else {
      if (!has_value) {
        if (i + 1 >= argc) throw UsageError("--" + name + " requires a value");
        value = argv[++i];
      }
      it->set(value);
    }
    seen[name] = true;
  }
  for (const auto& o : opts)
    if (o.required && !seen.count(o.name)) throw UsageError("--" + o.name + " is required");
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return 1;
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    usage(std::cout);
    return 0;
  }
  RegOpts reg;
  EvalOpts ev;
  SynthOpts sy;
  bool no_rescale = false;
  std::vector<Opt> opts;
  if (sub == "register") {
    opts = {
        {"source", "source image (.raw with .json sidecar)", false, true, setter(reg.source)},
        {"target", "target image", false, true, setter(reg.target)},
        {"out", "output directory", false, true, setter(reg.out)},
        {"variant", "original | state_equation | deformation_state_equation", false, false, setter(reg.variant)},
        {"integrator", "sl | rk4", false, false, setter(reg.integrator)},
        {"repr", "band | spatial (velocity representation)", false, false, setter(reg.repr)},
        {"param", "stationary | nonstationary", false, false, setter(reg.param)},
        {"band", "retained modes per axis for --repr band", false, false, setter(reg.band)},
        {"nt", "time steps (default: 5 for sl, 25 for rk4)", false, false, setter(reg.nt)},
        {"alpha", "regularizer strength", false, false, setter(reg.alpha)},
        {"s", "regularizer exponent", false, false, setter(reg.s)},
        {"sigma2", "data-term weight 1/sigma2", false, false, setter(reg.sigma2)},
        {"max-iter", "outer iteration cap", false, false, setter(reg.max_iter)},
        {"pcg-iter", "inner PCG iteration cap", false, false, setter(reg.pcg_iter)},
        {"v0", "warm-start velocity (spatial vector field)", false, false, setter(reg.v0_path)},
        {"source-labels", "labels to carry through the map", false, false, setter(reg.source_labels)},
        {"target-labels", "reference labels for Dice", false, false, setter(reg.target_labels)},
        {"no-rescale", "skip min-max rescaling of inputs", true, false,
         [&](const std::string&) { no_rescale = true; }},
    };
  } else if (sub == "evaluate") {
    opts = {
        {"source", "source image", false, true, setter(ev.source)},
        {"target", "target image", false, true, setter(ev.target)},
        {"warped", "warped source (defaults to the source)", false, false, setter(ev.warped)},
        {"warped-labels", "warped label field", false, false, setter(ev.warped_labels)},
        {"target-labels", "reference label field", false, false, setter(ev.target_labels)},
        {"displacement", "displacement field for Jacobian range", false, false, setter(ev.displacement)},
        {"out", "also write the report to this path", false, false, setter(ev.out)},
    };
  } else if (sub == "synth") {
    opts = {
        {"kind", "blobs | discs | rotation", false, false, setter(sy.kind)},
        {"out", "output directory", false, true, setter(sy.out)},
        {"n", "grid points per axis", false, false, setter(sy.n)},
        {"d", "dimension (2 or 3)", false, false, setter(sy.d)},
        {"spacing", "grid spacing", false, false, setter(sy.spacing)},
        {"seed", "random seed", false, false, setter(sy.seed)},
    };
  } else {
    std::cerr << "error: unknown subcommand: " << sub << "\n";
    usage(std::cerr);
    return 1;
  }
  try {
    if (!parse(argc, argv, sub, opts)) return 0;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    sub_usage(std::cerr, sub, opts);
    return 1;
  }
  reg.no_rescale = no_rescale;
  try {
    if (sub == "register") return do_register(reg);
    if (sub == "evaluate") return do_evaluate(ev);
    return do_synth(sy);
  } catch (const Divergence& de) {
    std::cerr << "error: transport diverged: " << de.what() << "\n";
    return 2;
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return 1;
  }
}
