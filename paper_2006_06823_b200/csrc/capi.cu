// extern "C" implementation of include/lddmm_cuda.h over Engine / optimize.
#include <algorithm>
#include <cstring>
#include <unordered_set>
#include <vector>
#include <memory>
#include <string>

#include "../../include/lddmm_cuda.h"
#include "engine.hpp"
#include "optimizer.hpp"

using namespace lddmm_b200;

struct lddmm_ctx {
  std::unique_ptr<Engine> eng;
  std::string err;
  // d = 2: the engine runs the 3-D problem (Nx, Ny, zr) (Problem::zrep); the ABI keeps
  // the reference's 2-D layouts and converts at the boundary (grid fields: replicate
  // along z / take the z = 0 slice; vectors: 2 components; band vectors: the kz = 0
  // plane scaled by zr, components x, y)
  int d = 3;
  int zr = 1;
};

namespace {

thread_local std::string g_create_err;

// Binds the context's device for the duration of an ABI call and restores the
// caller's current device afterwards (contexts on different GPUs in one process).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (dev < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class F>
int guard(lddmm_ctx* ctx, F&& f, int* step = nullptr) {
  try {
    DeviceScope dev(ctx && ctx->eng ? ctx->eng->device() : -1);
    f();
    return LDDMM_OK;
  } catch (const EngineError& e) {
    if (ctx) ctx->err = e.what();
    if (step && e.status == LDDMM_EDIVERGENCE) *step = e.step;
    return e.status;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return LDDMM_ECUDA;
  }
}

inline double2* D2(double* p) { return reinterpret_cast<double2*>(p); }
inline const double2* D2(const double* p) { return reinterpret_cast<const double2*>(p); }

// ---- 2-D <-> internal 3-D layout conversions (lddmm_ctx::d == 2) -------------------

constexpr int kZRep2D = 4;  // z replicas of a 2-D problem (even, >= 4, a multiple of 4)

long long n2d(const lddmm_ctx* ctx) {
  const Problem& p = ctx->eng->problem();
  return (long long)p.dims[0] * p.dims[1];
}

// host grid components: 2-D [nc][Nx*Ny] -> 3-D [nc3][Nx*Ny*zr] (z-constant; components
// nc .. nc3-1 zero)
std::vector<double> grid_to3(const lddmm_ctx* ctx, const double* src, int nc, int nc3) {
  const long long n2 = n2d(ctx), n3 = n2 * ctx->zr;
  std::vector<double> out((size_t)nc3 * n3, 0.0);
  for (int c = 0; c < nc; ++c)
    for (long long i = 0; i < n2; ++i)
      for (int z = 0; z < ctx->zr; ++z) out[(size_t)c * n3 + i * ctx->zr + z] = src[(size_t)c * n2 + i];
  return out;
}

// host 3-D [nc3][n3] -> 2-D [nc][n2] (the z = 0 slice of the first nc components)
void grid_to2(const lddmm_ctx* ctx, const double* src, int nc, double* dst) {
  const long long n2 = n2d(ctx), n3 = n2 * ctx->zr;
  for (int c = 0; c < nc; ++c)
    for (long long i = 0; i < n2; ++i) dst[(size_t)c * n2 + i] = src[(size_t)c * n3 + i * ctx->zr];
}

// band vectors: 2-D [nodes][2][Kx][Ky] complex <-> 3-D [nodes][3][Kx][Ky][Kz]
void band_to3(const lddmm_ctx* ctx, const double* src, int nodes, double* dst) {
  const Problem& p = ctx->eng->problem();
  const long long kxy = (long long)p.band[0] * p.band[1], kz = p.band[2];
  const long long v2 = 2 * kxy, v3 = 3 * kxy * kz;
  std::memset(dst, 0, (size_t)nodes * v3 * 2 * sizeof(double));
  for (int nd = 0; nd < nodes; ++nd)
    for (int c = 0; c < 2; ++c)
      for (long long k = 0; k < kxy; ++k) {
        const double* s = src + 2 * (nd * v2 + c * kxy + k);
        double* o = dst + 2 * (nd * v3 + (c * kxy + k) * kz);  // kz = 0 entry
        o[0] = ctx->zr * s[0];
        o[1] = ctx->zr * s[1];
      }
}

void band_to2(const lddmm_ctx* ctx, const double* src, int nodes, double* dst) {
  const Problem& p = ctx->eng->problem();
  const long long kxy = (long long)p.band[0] * p.band[1], kz = p.band[2];
  const long long v2 = 2 * kxy, v3 = 3 * kxy * kz;
  for (int nd = 0; nd < nodes; ++nd)
    for (int c = 0; c < 2; ++c)
      for (long long k = 0; k < kxy; ++k) {
        const double* s = src + 2 * (nd * v3 + (c * kxy + k) * kz);
        double* o = dst + 2 * (nd * v2 + c * kxy + k);
        o[0] = s[0] / ctx->zr;
        o[1] = s[1] / ctx->zr;
      }
}

int vel_nodes(const lddmm_ctx* ctx) { return (int)(ctx->eng->vel_elems() / ctx->eng->vec_elems()); }

__global__ void replicate_z_kernel(const float* __restrict__ src, long long n2, int zr, float* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2 * zr;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i / zr];
}

OptimizeOptions to_opts(const lddmm_options* o) {
  OptimizeOptions r;
  if (!o) return r;
  r.max_iter = o->max_iter;
  r.pcg_max_iter = o->pcg_max_iter;
  r.pcg_tol = o->pcg_tol;
  r.grad_tol = o->grad_tol;
  r.energy_tol = o->energy_tol;
  r.step_tol = o->step_tol;
  r.armijo_c = o->armijo_c;
  r.armijo_max_trials = o->armijo_max_trials;
  return r;
}

void fill_result(const OptimizeResult& r, lddmm_iteration_record* hist, int cap, lddmm_result* res) {
  if (hist) {
    const int n = std::min<int>(cap, (int)r.history.size());
    for (int k = 0; k < n; ++k) {
      const IterationRecord& q = r.history[k];
      lddmm_iteration_record& o = hist[k];
      std::memset(&o, 0, sizeof(o));
      o.iter = q.iter;
      o.energy = q.energy;
      o.energy_data = q.energy_data;
      o.energy_reg = q.energy_reg;
      o.mse_rel = q.mse_rel;
      o.rel_grad = q.rel_grad;
      o.pcg_iters = q.pcg_iters;
      o.pcg_fallback = q.pcg_fallback ? 1 : 0;
      o.epsilon = q.epsilon;
      o.cfl = q.cfl;
      o.wall_ms = q.wall_ms;
      o.n_pcg_residuals = std::min<int>(16, (int)q.pcg_residuals.size());
      for (int j = 0; j < o.n_pcg_residuals; ++j) o.pcg_residuals[j] = q.pcg_residuals[j];
    }
  }
  if (res) {
    res->stop_reason = r.stop;
    res->converged = r.converged ? 1 : 0;
    res->iterations = r.iterations;
    res->n_history = (int)r.history.size();
    res->final_energy = r.final_energy;
    res->rel_grad = r.rel_grad;
    res->hessvecs = r.hessvecs;
    res->trials = r.trials;
    res->forwards = r.forwards;
  }
}

}  // namespace

extern "C" {

void lddmm_default_options(lddmm_options* o) {
  OptimizeOptions d;
  o->max_iter = d.max_iter;
  o->pcg_max_iter = d.pcg_max_iter;
  o->pcg_tol = d.pcg_tol;
  o->grad_tol = d.grad_tol;
  o->energy_tol = d.energy_tol;
  o->step_tol = d.step_tol;
  o->armijo_c = d.armijo_c;
  o->armijo_max_trials = d.armijo_max_trials;
}

int lddmm_create(const lddmm_problem* p, int device, lddmm_ctx** out) {
  *out = nullptr;
  auto ctx = std::make_unique<lddmm_ctx>();
  int caller_dev = -1;
  if (cudaGetDevice(&caller_dev) != cudaSuccess) caller_dev = -1;
  DeviceScope restore(caller_dev);  // the Engine constructor binds `device`
  const int rc = guard(ctx.get(), [&] {
    shape_require(p != nullptr, "null problem");
    shape_require(p->d == 3 || p->d == 2, "grid dimension must be 2 or 3 (core.hpp:49-52)");
    Problem q;
    for (int a = 0; a < 3; ++a) {
      q.dims[a] = p->dims[a];
      q.spacing[a] = p->spacing[a];
      q.band[a] = p->band[a];
    }
    if (p->d == 2) {
      // z replicated kZRep2D times at spacing 1 / kZRep2D (Problem::zrep)
      q.dims[2] = kZRep2D;
      q.spacing[2] = 1.0 / kZRep2D;
      q.band[2] = kZRep2D;
      q.d = 2;
      q.zrep = kZRep2D;
      ctx->d = 2;
      ctx->zr = kZRep2D;
    }
    q.nt = p->nt;
    q.variant = p->variant;
    q.stationary = p->parameterization == LDDMM_STATIONARY ? 1 : 0;
    q.alpha = p->alpha;
    q.s = p->s;
    q.sigma2 = p->sigma2;
    shape_require(p->integrator == LDDMM_SL || p->integrator == LDDMM_RK4, "unknown integrator");
    q.rk4 = p->integrator == LDDMM_RK4 ? 1 : 0;
    ctx->eng = std::make_unique<Engine>(q, device);
  });
  if (rc != LDDMM_OK) {
    g_create_err = ctx->err;
    return rc;
  }
  *out = ctx.release();
  return LDDMM_OK;
}

void lddmm_destroy(lddmm_ctx* ctx) {
  if (!ctx) return;
  DeviceScope dev(ctx->eng ? ctx->eng->device() : -1);
  delete ctx;
}

const char* lddmm_last_error(const lddmm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int lddmm_sync(lddmm_ctx* ctx) {
  return guard(ctx, [&] { ctx->eng->sync(); });
}

long long lddmm_launch_count(void) { return launch_counter(); }

void* lddmm_stream(lddmm_ctx* ctx) { return (void*)ctx->eng->stream(); }

int lddmm_gather_timing(lddmm_ctx* ctx, int mode) {
  return guard(ctx, [&] { ctx->eng->set_gather_timing(mode); });
}

int lddmm_gather_stats(lddmm_ctx* ctx, double* ms, long long* launches, double* bytes) {
  return guard(ctx, [&] { ctx->eng->gather_stats(ms, launches, bytes); });
}

int lddmm_dft_stats(lddmm_ctx* ctx, double* ms, long long* launches, double* flops) {
  return guard(ctx, [&] { ctx->eng->timing_stats(1, ms, launches, flops); });
}

int lddmm_set_images(lddmm_ctx* ctx, const double* I0, const double* I1) {
  return guard(ctx, [&] {
    if (ctx->d == 2) {
      const std::vector<double> a = grid_to3(ctx, I0, 1, 1), b = grid_to3(ctx, I1, 1, 1);
      ctx->eng->set_images_host(a.data(), b.data());
    } else {
      ctx->eng->set_images_host(I0, I1);
    }
  });
}

int lddmm_set_images_dev_f32(lddmm_ctx* ctx, const float* I0, const float* I1) {
  return guard(ctx, [&] {
    if (ctx->d == 2) {
      Engine& e = *ctx->eng;
      const long long n2 = n2d(ctx);
      DevBuf<float> a(n2 * ctx->zr), b(n2 * ctx->zr);
      replicate_z_kernel<<<grid_for(n2 * ctx->zr, 256), 256, 0, e.stream()>>>(I0, n2, ctx->zr, a.p);
      LDDMM_LAUNCH_CHECK();
      replicate_z_kernel<<<grid_for(n2 * ctx->zr, 256), 256, 0, e.stream()>>>(I1, n2, ctx->zr, b.p);
      LDDMM_LAUNCH_CHECK();
      e.set_images_device_f32(a.p, b.p);
      e.sync();
    } else {
      ctx->eng->set_images_device_f32(I0, I1);
    }
  });
}

long long lddmm_velocity_doubles(const lddmm_ctx* ctx) {
  if (ctx->d == 2) {
    const Problem& p = ctx->eng->problem();
    return 2LL * vel_nodes(ctx) * 2 * p.band[0] * p.band[1];
  }
  return 2 * ctx->eng->vel_elems();
}

int lddmm_vel_alloc(lddmm_ctx* ctx, double** v) {
  return guard(ctx, [&] {
    const size_t bytes = ctx->eng->vel_elems() * sizeof(double2);
    LDDMM_CUDA(cudaMalloc(v, bytes));
    LDDMM_CUDA(cudaMemsetAsync(*v, 0, bytes, ctx->eng->stream()));
    ctx->eng->sync();
  });
}

int lddmm_vel_free(lddmm_ctx* ctx, double* v) {
  return guard(ctx, [&] { LDDMM_CUDA(cudaFree(v)); });
}

int lddmm_vel_upload(lddmm_ctx* ctx, double* dv, const double* hv) {
  return guard(ctx, [&] {
    const size_t bytes = ctx->eng->vel_elems() * sizeof(double2);
    if (ctx->d == 2) {
      std::vector<double> t(2 * ctx->eng->vel_elems());
      band_to3(ctx, hv, vel_nodes(ctx), t.data());
      LDDMM_CUDA(cudaMemcpyAsync(dv, t.data(), bytes, cudaMemcpyHostToDevice, ctx->eng->stream()));
      ctx->eng->sync();
      return;
    }
    LDDMM_CUDA(cudaMemcpyAsync(dv, hv, bytes, cudaMemcpyHostToDevice, ctx->eng->stream()));
    ctx->eng->sync();
  });
}

int lddmm_vel_download(lddmm_ctx* ctx, const double* dv, double* hv) {
  return guard(ctx, [&] {
    const size_t bytes = ctx->eng->vel_elems() * sizeof(double2);
    if (ctx->d == 2) {
      std::vector<double> t(2 * ctx->eng->vel_elems());
      LDDMM_CUDA(cudaMemcpyAsync(t.data(), dv, bytes, cudaMemcpyDeviceToHost, ctx->eng->stream()));
      ctx->eng->sync();
      band_to2(ctx, t.data(), vel_nodes(ctx), hv);
      return;
    }
    LDDMM_CUDA(cudaMemcpyAsync(hv, dv, bytes, cudaMemcpyDeviceToHost, ctx->eng->stream()));
    ctx->eng->sync();
  });
}

int lddmm_vel_axpy(lddmm_ctx* ctx, double a, const double* x, const double* y, double* out) {
  return guard(ctx, [&] { ctx->eng->tv_axpy(a, D2(x), D2(y), D2(out)); });
}
int lddmm_vel_scale(lddmm_ctx* ctx, const double* x, double a, double* out) {
  return guard(ctx, [&] { ctx->eng->tv_scaled(D2(x), a, D2(out)); });
}
int lddmm_vel_inner(lddmm_ctx* ctx, const double* x, const double* y, double* out) {
  return guard(ctx, [&] { *out = ctx->eng->tv_inner(D2(x), D2(y)); });
}
int lddmm_vel_linf(lddmm_ctx* ctx, const double* x, double* out) {
  return guard(ctx, [&] { *out = ctx->eng->tv_linf(D2(x)); });
}
int lddmm_vel_all_finite(lddmm_ctx* ctx, const double* x, int* out) {
  return guard(ctx, [&] { *out = ctx->eng->tv_all_finite(D2(x)) ? 1 : 0; });
}

int lddmm_forward(lddmm_ctx* ctx, const double* v, int with_adjoint, lddmm_energies* out, int* step) {
  return guard(
      ctx,
      [&] {
        Energies e = ctx->eng->forward(D2(v), with_adjoint != 0);
        if (out) *out = lddmm_energies{e.energy, e.energy_reg, e.energy_data, e.cfl};
      },
      step);
}

int lddmm_energy(lddmm_ctx* ctx, const double* v, double* energy, int* step) {
  return guard(ctx, [&] { *energy = ctx->eng->energy(D2(v)); }, step);
}

int lddmm_gradient(lddmm_ctx* ctx, double* out) {
  return guard(ctx, [&] {
    ctx->eng->gradient(D2(out));
    ctx->eng->sync();
  });
}

int lddmm_hessvec(lddmm_ctx* ctx, const double* dv, double* out, int* step) {
  return guard(
      ctx,
      [&] {
        ctx->eng->hessvec(D2(dv), D2(out));
        ctx->eng->sync();
      },
      step);
}

int lddmm_precondition(lddmm_ctx* ctx, const double* in, double* out) {
  return guard(ctx, [&] {
    ctx->eng->precondition(D2(in), D2(out));
    ctx->eng->sync();
  });
}

// device fp32 grid components -> host fp64 in the ABI layout (2-D: the z = 0 slice)
static void fetch_grid(lddmm_ctx* ctx, const float* dev, int nc, double* host) {
  Engine& e = *ctx->eng;
  const long long N = e.npts();
  DevBuf<double> tmp(nc * N);
  launch_f32_to_f64(nc * N, dev, tmp.p, e.stream());
  if (ctx->d == 2) {
    std::vector<double> t(nc * N);
    LDDMM_CUDA(cudaMemcpyAsync(t.data(), tmp.p, nc * N * sizeof(double), cudaMemcpyDeviceToHost, e.stream()));
    e.sync();
    grid_to2(ctx, t.data(), nc, host);
    return;
  }
  LDDMM_CUDA(cudaMemcpyAsync(host, tmp.p, nc * N * sizeof(double), cudaMemcpyDeviceToHost, e.stream()));
  e.sync();
}

int lddmm_get_fields(lddmm_ctx* ctx, double* m1, double* res) {
  return guard(ctx, [&] {
    if (m1) fetch_grid(ctx, ctx->eng->m1(), 1, m1);
    if (res) fetch_grid(ctx, ctx->eng->residual(), 1, res);
  });
}

int lddmm_get_grid(lddmm_ctx* ctx, int which, double* host_out) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts();
    const float* src = e.grid_field(which);
    shape_require(src != nullptr, "lddmm_get_grid: unknown field");
    (void)N;
    fetch_grid(ctx, src, 1, host_out);
  });
}

int lddmm_get_series(lddmm_ctx* ctx, int which, double* host_out) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long n = (e.problem().nt + 1) * e.vec_elems();
    DevBuf<double2> tmp(n);
    e.series(which, tmp.p);
    if (ctx->d == 2) {
      std::vector<double> t(2 * n);
      LDDMM_CUDA(cudaMemcpy(t.data(), tmp.p, n * sizeof(double2), cudaMemcpyDeviceToHost));
      band_to2(ctx, t.data(), e.problem().nt + 1, host_out);
      return;
    }
    LDDMM_CUDA(cudaMemcpy(host_out, tmp.p, n * sizeof(double2), cudaMemcpyDeviceToHost));
  });
}

int lddmm_optimize(lddmm_ctx* ctx, double* v, const lddmm_options* opt, lddmm_iteration_record* hist, int cap,
                   lddmm_result* res) {
  return guard(ctx, [&] {
    OptimizeResult r = optimize(*ctx->eng, D2(v), to_opts(opt));
    ctx->eng->sync();
    fill_result(r, hist, cap, res);
  });
}

int lddmm_register(lddmm_ctx* ctx, const double* I0, const double* I1, const lddmm_options* opt, double* host_v,
                   lddmm_iteration_record* hist, int cap, lddmm_result* res) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    if (ctx->d == 2) {
      const std::vector<double> a = grid_to3(ctx, I0, 1, 1), b = grid_to3(ctx, I1, 1, 1);
      e.set_images_host(a.data(), b.data());
    } else {
      e.set_images_host(I0, I1);
    }
    double2* v = e.register_velocity();
    LDDMM_CUDA(cudaMemsetAsync(v, 0, e.vel_elems() * sizeof(double2), e.stream()));
    OptimizeResult r = optimize(e, v, to_opts(opt));
    if (host_v && ctx->d == 2) {
      std::vector<double> t(2 * e.vel_elems());
      LDDMM_CUDA(cudaMemcpyAsync(t.data(), v, e.vel_elems() * sizeof(double2), cudaMemcpyDeviceToHost, e.stream()));
      e.sync();
      band_to2(ctx, t.data(), vel_nodes(ctx), host_v);
    } else if (host_v) {
      LDDMM_CUDA(cudaMemcpyAsync(host_v, v, e.vel_elems() * sizeof(double2), cudaMemcpyDeviceToHost, e.stream()));
    }
    e.sync();
    fill_result(r, hist, cap, res);
  });
}

int lddmm_maps(lddmm_ctx* ctx, const double* v, double* hf, double* hi, double jac[4]) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts();
    DevBuf<float> f(3 * N), i(3 * N);
    e.maps(D2(v), f.p, i.p, jac);
    const int nc = ctx->d;  // 2-D: the x, y displacement components
    if (hf) fetch_grid(ctx, f.p, nc, hf);
    if (hi) fetch_grid(ctx, i.p, nc, hi);
  });
}

int lddmm_op_embed(lddmm_ctx* ctx, const double* band, int ncomp, float* grid, int prefilter) {
  return guard(ctx, [&] {
    ctx->eng->embed(D2(band), ncomp, grid, prefilter != 0);
    ctx->eng->sync();
  });
}

int lddmm_op_project(lddmm_ctx* ctx, const float* grid, int ncomp, double* band) {
  return guard(ctx, [&] {
    ctx->eng->project(grid, ncomp, D2(band));
    ctx->eng->sync();
  });
}

int lddmm_op_advect(lddmm_ctx* ctx, const double* band, int ncomp, const float* dep, double* out) {
  return guard(ctx, [&] {
    ctx->eng->advect(D2(band), ncomp, dep, D2(out));
    ctx->eng->sync();
  });
}

int lddmm_op_departure(lddmm_ctx* ctx, const double* v, float* df, float* db, double* cfl) {
  return guard(ctx, [&] { ctx->eng->departure(D2(v), df, db, cfl); });
}

int lddmm_op_band(lddmm_ctx* ctx, int op, const double* a, const double* b, double* out) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    switch (op) {
      case 0: e.star_ss(D2(a), D2(b), D2(out), 1.0); break;
      case 1: e.star_sv(D2(a), D2(b), D2(out), 1.0); break;
      case 2: e.star_dot(D2(a), D2(b), D2(out), 1.0); break;
      case 3: e.jac_mul(D2(a), D2(b), D2(out), 1.0, false); break;
      case 4: e.jac_mul(D2(a), D2(b), D2(out), 1.0, true); break;
      case 5: e.band_divergence(D2(a), D2(out)); break;
      default: throw EngineError(1, "lddmm_op_band: unknown op");
    }
    e.sync();
  });
}

int lddmm_op_gather(lddmm_ctx* ctx, int impl, const float* coef, int ncomp, const float* dep, float* out) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    int N[3] = {e.problem().dims[0], e.problem().dims[1], e.problem().dims[2]};
    if (impl == 4) {
      shape_require(launch_gather_pipe(coef, ncomp, dep, out, N, make_float3(1.f, 1.f, 1.f), e.stream()),
                    "lddmm_op_gather: impl 4 (pipelined gather) does not support this grid");
    } else if (impl == 0)
      launch_gather_cubic(coef, ncomp, dep, out, N, e.stream());
    else if (impl == 3)
      launch_gather_scaled(coef, ncomp, dep, 1.f, 1.f, 1.f, out, N, e.stream(), false);
    else if (impl == 1)
      launch_gather_cubic_tiled(coef, ncomp, dep, out, N, e.stream());
    else
      launch_gather_cubic_global(coef, ncomp, dep, out, N, e.stream());
    e.sync();
  });
}

int lddmm_op_warp(lddmm_ctx* ctx, const float* field, int ncomp, const float* disp, float* out) {
  return guard(ctx, [&] {
    ctx->eng->warp_grid(field, ncomp, disp, out);
    ctx->eng->sync();
  });
}

}  // extern "C"

// ---- evaluation path --------------------------------------------------------------

namespace {

// distinct nonzero label values in ascending order (metrics.hpp:120-126: std::set)
std::vector<float> label_inventory(const float* host, long long n) {
  std::unordered_set<float> seen;
  for (long long i = 0; i < n; ++i)
    if (host[i] != 0.0f) seen.insert(host[i]);
  std::vector<float> v(seen.begin(), seen.end());
  std::sort(v.begin(), v.end());
  return v;
}

// mean_dice (metrics.hpp:97-131) from device counts; same per-label ratio and
// ascending-label summation order as the reference
double mean_dice_dev(Engine& e, const float* a, const float* b) {
  const long long N = e.npts();
  std::vector<float> hb(N);
  LDDMM_CUDA(cudaMemcpyAsync(hb.data(), b, N * sizeof(float), cudaMemcpyDeviceToHost, e.stream()));
  e.sync();
  std::vector<float> labels = label_inventory(hb.data(), N);
  const bool empty = labels.empty();
  if (empty) labels.push_back(1.0f);  // dice(warped, target, 1.0) (metrics.hpp:128)
  const int nl = (int)labels.size();
  DevBuf<float> dl(nl);
  DevBuf<unsigned long long> dc(3 * nl);
  LDDMM_CUDA(cudaMemcpyAsync(dl.p, labels.data(), nl * sizeof(float), cudaMemcpyHostToDevice, e.stream()));
  e.dice_counts(a, b, dl.p, nl, dc.p);
  std::vector<unsigned long long> c(3 * nl);
  LDDMM_CUDA(cudaMemcpyAsync(c.data(), dc.p, 3 * nl * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             e.stream()));
  e.sync();
  double s = 0.0;
  for (int l = 0; l < nl; ++l) {
    const unsigned long long na = c[3 * l], nb = c[3 * l + 1], nab = c[3 * l + 2];
    const double dsc = na + nb == 0 ? 1.0 : 2.0 * (double)nab / (double)(na + nb);
    if (empty) return dsc;
    s += dsc;
  }
  return s / (double)nl;
}

void upload_f32(Engine& e, const double* host, long long n, float* dev) {
  DevBuf<double> t(n);
  LDDMM_CUDA(cudaMemcpyAsync(t.p, host, n * sizeof(double), cudaMemcpyHostToDevice, e.stream()));
  launch_f64_to_f32(n, t.p, dev, e.stream());
  e.sync();
}


}  // namespace

extern "C" {

int lddmm_op_warp_nearest(lddmm_ctx* ctx, const float* field, int ncomp, const float* disp, float* out) {
  return guard(ctx, [&] {
    shape_require(ncomp >= 1, "warp_nearest: ncomp >= 1");
    ctx->eng->warp_nearest(field, ncomp, disp, out);
    ctx->eng->sync();
  });
}

int lddmm_op_jacobian(lddmm_ctx* ctx, const float* disp, float* det, double minmax[2]) {
  return guard(ctx, [&] { ctx->eng->jacobian_grid(disp, det, minmax); });
}

int lddmm_op_mean_dice(lddmm_ctx* ctx, const float* a, const float* b, double* out) {
  return guard(ctx, [&] { *out = mean_dice_dev(*ctx->eng, a, b); });
}

int lddmm_warp(lddmm_ctx* ctx, int kind, const double* field, int ncomp, const double* disp, double* out) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts();
    shape_require(kind == LDDMM_INTERP_CUBIC || kind == LDDMM_INTERP_NEAREST,
                  "lddmm_warp: kind must be LDDMM_INTERP_CUBIC or LDDMM_INTERP_NEAREST");
    shape_require(ncomp >= 1 && ncomp <= 6, "lddmm_warp: 1..6 components");
    DevBuf<float> f(ncomp * N), d(3 * N), o(ncomp * N);
    if (ctx->d == 2) {
      const std::vector<double> f3 = grid_to3(ctx, field, ncomp, ncomp), d3 = grid_to3(ctx, disp, 2, 3);
      upload_f32(e, f3.data(), ncomp * N, f.p);
      upload_f32(e, d3.data(), 3 * N, d.p);
    } else {
      upload_f32(e, field, ncomp * N, f.p);
      upload_f32(e, disp, 3 * N, d.p);
    }
    if (kind == LDDMM_INTERP_CUBIC)
      e.warp_grid(f.p, ncomp, d.p, o.p);
    else
      e.warp_nearest(f.p, ncomp, d.p, o.p);
    fetch_grid(ctx, o.p, ncomp, out);
  });
}

int lddmm_jacobian(lddmm_ctx* ctx, const double* disp, double* det, double minmax[2]) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts();
    DevBuf<float> d(3 * N);
    if (ctx->d == 2) {
      const std::vector<double> d3 = grid_to3(ctx, disp, 2, 3);
      upload_f32(e, d3.data(), 3 * N, d.p);
    } else {
      upload_f32(e, disp, 3 * N, d.p);
    }
    DevBuf<float> o(det ? N : 1);
    e.jacobian_grid(d.p, det ? o.p : nullptr, minmax);
    if (det) fetch_grid(ctx, o.p, 1, det);
  });
}

int lddmm_mean_dice(lddmm_ctx* ctx, const double* a, const double* b, double* out) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts();
    DevBuf<float> da(N), db(N);
    if (ctx->d == 2) {
      // Dice of the z-replicated labels = Dice of the 2-D labels (every count times zr)
      const std::vector<double> a3 = grid_to3(ctx, a, 1, 1), b3 = grid_to3(ctx, b, 1, 1);
      upload_f32(e, a3.data(), N, da.p);
      upload_f32(e, b3.data(), N, db.p);
    } else {
      upload_f32(e, a, N, da.p);
      upload_f32(e, b, N, db.p);
    }
    *out = mean_dice_dev(e, da.p, db.p);
  });
}

int lddmm_vel_from_spatial(lddmm_ctx* ctx, const double* host_vec, double* v) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts(), V = e.vec_elems();
    DevBuf<float> g(3 * N);
    if (ctx->d == 2) {
      const std::vector<double> g3 = grid_to3(ctx, host_vec, 2, 3);
      upload_f32(e, g3.data(), 3 * N, g.p);
    } else {
      upload_f32(e, host_vec, 3 * N, g.p);
    }
    e.project(g.p, 3, D2(v));
    const int nodes = (int)(e.vel_elems() / V);
    for (int i = 1; i < nodes; ++i)
      LDDMM_CUDA(cudaMemcpyAsync(D2(v) + i * V, D2(v), V * sizeof(double2), cudaMemcpyDeviceToDevice, e.stream()));
    e.sync();
  });
}

int lddmm_vel_to_spatial(lddmm_ctx* ctx, const double* v, int node, double* host_vec) {
  return guard(ctx, [&] {
    Engine& e = *ctx->eng;
    const long long N = e.npts(), V = e.vec_elems();
    const int nodes = (int)(e.vel_elems() / V);
    shape_require(node >= 0 && node < nodes, "lddmm_vel_to_spatial: node out of range");
    DevBuf<float> g(3 * N);
    e.embed(D2(v) + node * V, 3, g.p, false);
    fetch_grid(ctx, g.p, ctx->d, host_vec);
  });
}

}  // extern "C"
