// Runs the REFERENCE's optimize<Alg> (optimizer.hpp:143-262, unmodified header) over
// Model<CudaBandAlgebra> (cuda_band_algebra.hpp: every operator on the B200 engine),
// and, on the same context and images, the engine's own C++ driver (lddmm_optimize).
// Prints both GN-Krylov histories as JSON for tests/test_gpu_dropin.py.
//
//   dropin_optimize <dims x y z> <band x y z> <nt> <sigma2> <max_iter> <I0.f64> <I1.f64>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "cuda_band_algebra.hpp"

static std::vector<double> read_f64(const char* path, size_t n) {
  std::vector<double> v(n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(n * sizeof(double)));
  if (!f) {
    std::fprintf(stderr, "cannot read %zu doubles from %s\n", n, path);
    std::exit(1);
  }
  return v;
}

static void print_record(const char* sep, int iter, double E, double Ed, double Er, double mse, double relg, int pcg,
                         int fb, double eps, double cfl) {
  std::printf("%s{\"iter\": %d, \"energy\": %.17g, \"energy_data\": %.17g, \"energy_reg\": %.17g, "
              "\"mse_rel\": %.17g, \"rel_grad\": %.17g, \"pcg_iters\": %d, \"pcg_fallback\": %d, "
              "\"epsilon\": %.17g, \"cfl\": %.17g}",
              sep, iter, E, Ed, Er, mse, relg, pcg, fb, eps, cfl);
}

int main(int argc, char** argv) {
  if (argc != 14) {
    std::fprintf(stderr, "usage: %s nx ny nz kx ky kz nt sigma2 max_iter I0.f64 I1.f64 v_ref.f64 v_drv.f64\n",
                 argv[0]);
    return 1;
  }
  std::vector<int> n = {std::atoi(argv[1]), std::atoi(argv[2]), std::atoi(argv[3])};
  std::vector<int> k = {std::atoi(argv[4]), std::atoi(argv[5]), std::atoi(argv[6])};
  const int nt = std::atoi(argv[7]);
  const double sigma2 = std::atof(argv[8]);
  const int max_iter = std::atoi(argv[9]);
  lddmm::GridSpec g(n, {1.0, 1.0, 1.0});
  lddmm::BandSpec band(g, std::array<int, lddmm::kMaxDim>{k[0], k[1], k[2]});
  lddmm::ScalarField I0(g, read_f64(argv[10], g.size())), I1(g, read_f64(argv[11], g.size()));

  lddmm_problem p{};
  p.d = 3;
  for (int a = 0; a < 3; ++a) {
    p.dims[a] = n[a];
    p.spacing[a] = 1.0;
    p.band[a] = k[a];
  }
  p.nt = nt;
  p.variant = LDDMM_DEFORMATION_STATE_EQUATION;
  p.parameterization = LDDMM_STATIONARY;
  p.alpha = 0.0025;  // SobolevOperator{} defaults (spectral.hpp:518-525)
  p.s = 2;
  p.sigma2 = sigma2;
  p.integrator = LDDMM_SL;
  if (lddmm_create(&p, 0, &cudaalg::context()) != LDDMM_OK) {
    std::fprintf(stderr, "lddmm_create: %s\n", lddmm_last_error(nullptr));
    return 1;
  }

  lddmm::OptimizeOptions opt;  // reference defaults
  opt.max_iter = max_iter;
  opt.pcg_max_iter = 5;
  std::printf("{\"reference_optimize\": {\"history\": [");
  {
    lddmm::Model<cudaalg::CudaBandAlgebra> model(band, I0, I1, nt);
    auto r = lddmm::optimize(model, model.zero_velocity(), opt);  // the reference's template
    const char* sep = "";
    for (const auto& h : r.history) {
      print_record(sep, h.iter, h.energy, h.energy_data, h.energy_reg, h.mse_rel, h.rel_grad, h.pcg_iters,
                   h.pcg_fallback ? 1 : 0, h.epsilon, h.cfl);
      sep = ", ";
    }
    std::printf("], \"stop\": \"%s\", \"iterations\": %d}", lddmm::to_string(r.stop), r.iterations);
    std::vector<double> vh(lddmm_velocity_doubles(cudaalg::context()));
    cudaalg::check(lddmm_vel_download(cudaalg::context(), r.v.node(0).p, vh.data()));
    std::ofstream(argv[12], std::ios::binary).write(reinterpret_cast<const char*>(vh.data()),
                                                   (std::streamsize)(vh.size() * sizeof(double)));
  }
  {
    lddmm_options o;
    lddmm_default_options(&o);
    o.max_iter = max_iter;
    o.pcg_max_iter = 5;
    std::vector<lddmm_iteration_record> hist(max_iter + 2);
    lddmm_result res{};
    double* v = nullptr;
    cudaalg::check(lddmm_vel_alloc(cudaalg::context(), &v));
    cudaalg::check(lddmm_set_images(cudaalg::context(), I0.v.data(), I1.v.data()));
    cudaalg::check(lddmm_optimize(cudaalg::context(), v, &o, hist.data(), (int)hist.size(), &res));
    std::printf(", \"engine_driver\": {\"history\": [");
    const char* sep = "";
    for (int i = 0; i < res.n_history && i < (int)hist.size(); ++i) {
      const auto& h = hist[i];
      print_record(sep, h.iter, h.energy, h.energy_data, h.energy_reg, h.mse_rel, h.rel_grad, h.pcg_iters,
                   h.pcg_fallback, h.epsilon, h.cfl);
      sep = ", ";
    }
    const char* names[] = {"gradient", "energy_change", "step_size", "zero_gradient", "max_iterations",
                           "line_search_failure"};
    std::printf("], \"stop\": \"%s\", \"iterations\": %d}}\n", names[res.stop_reason], res.iterations);
    std::vector<double> vh(lddmm_velocity_doubles(cudaalg::context()));
    cudaalg::check(lddmm_vel_download(cudaalg::context(), v, vh.data()));
    std::ofstream(argv[13], std::ios::binary).write(reinterpret_cast<const char*>(vh.data()),
                                                   (std::streamsize)(vh.size() * sizeof(double)));
    lddmm_vel_free(cudaalg::context(), v);
  }
  lddmm_destroy(cudaalg::context());
  return 0;
}
