// The `original` and `state_equation` variants on the device (variants.hpp:373-422,
// 444-527, gradient 291-309, hessvec 313-344), band-limited, SL, stationary.
// The deformation-state variant lives in engine.cu.
//
//   original : m transported forward as a band scalar (D_t m = 0), scalar adjoint
//              lambda backward (D_t q = -q div v), node term lambda * grad m
//   state    : u forward, m_i = pi(I0 o (x - iota u_i)), nu backward, Jacobian factor
//              U backward (D_t U = div v - U div v), lambda_i = pi(J_i (lambda1 o psi_i)),
//              node term lambda_i * grad m_i
//
// grad m_i is never materialised: the i*omega symbols are applied in the embed
// prep of the small product grid.
#include <algorithm>
#include <vector>

#include "engine.hpp"

namespace lddmm_b200 {

namespace {
std::vector<double> trap_w(int nt) {  // variants.hpp:40-46
  std::vector<double> w(nt + 1, 1.0 / nt);
  w.front() *= 0.5;
  w.back() *= 0.5;
  return w;
}
}  // namespace

void Engine::ensure_variant_buffers() {
  const long long S = kprod(), V = vec_elems(), N = npts();
  const int nt = prob_.nt;
  if (prob_.variant == 2) return;
  if (!m_ser_.p) {
    m_ser_.alloc((nt + 1) * S);
    lam_ser_.alloc((nt + 1) * S);
    dm_ser_.alloc((nt + 1) * S);
    if (prob_.variant == 0 && trial_reuse_ok()) trial_mser_.alloc((nt + 1) * S);
  }
  if (prob_.variant == 1 && !nu_ser_.p) {
    nu_ser_.alloc((nt + 1) * V);
    bigU_ser_.alloc((nt + 1) * S);
    jac_f_.alloc((nt + 1) * N);
    psi_f_.alloc((nt + 1) * 3 * N);
    fgI0coef_.alloc(3 * N);
    lcoef_.alloc(N);
  }
}

// D_t u = v forward (from 0 at t = 0) or backward (from 0 at t = 1), variants.hpp:468-472
void Engine::solve_displacement(ProviderState& ps, bool forward, double2* series) {
  if (prob_.rk4) {
    rk4_displacement(ps, forward, series, nullptr);
    return;
  }
  const long long V = vec_elems(), K = kprod();
  const int nt = prob_.nt;
  const double sdt = forward ? 1.0 / nt : -1.0 / nt;
  double2* F = bt(0);
  if (prob_.stationary) advect(ps.v.p, 3, forward ? ps.dep_fwd.p : ps.dep_bwd.p, F);
  LDDMM_CUDA(cudaMemsetAsync(series + (forward ? 0 : nt) * V, 0, V * sizeof(double2), stream_));
  for (int s = 0; s < nt; ++s) {
    const int from = forward ? s : nt - s, to = forward ? s + 1 : nt - s - 1;
    const int step = forward ? s : nt - s - 1;
    const float* dep = forward ? depf(ps, step) : depb(ps, step);
    double2* tmp = bt(1);
    if (prob_.stationary) {
      if (s == 0) {
        launch_scale(V, 0.5 * sdt, ps.v.p, tmp, stream_);
      } else {
        const double2* q = series + from * V;
        const double2* in[3] = {q, q + K, q + 2 * K};
        FinField outs[3];
        for (int c = 0; c < 3; ++c) outs[c] = FinField{tmp + c * K, 1.0, ps.v.p + c * K, 0.5 * sdt};
        advect_multi(in, 3, dep, outs);
      }
      launch_axpy(V, 0.5 * sdt, F, tmp, series + to * V, stream_);
    } else {
      launch_axpy(V, 0.5 * sdt, vnode(ps, from), series + from * V, tmp, stream_);
      const double2* in[3] = {tmp, tmp + K, tmp + 2 * K};
      FinField outs[3];
      for (int c = 0; c < 3; ++c)
        outs[c] = FinField{series + to * V + c * K, 1.0, vnode(ps, to) + c * K, 0.5 * sdt};
      advect_multi(in, 3, dep, outs);
    }
    enqueue_finite_check(series + to * V, s);
  }
  finish_finite_checks(nt);
}

// D_t m = 0 forward from m0 (variants.hpp:444-446): m_{s+1} = advect(m_s)
void Engine::solve_image_forward(ProviderState& ps, const double2* m0, double2* series, bool keep_all,
                                 double2* last) {
  if (prob_.rk4) {
    rk4_image_forward(ps, m0, keep_all ? series : nullptr, last);
    return;
  }
  const long long S = kprod();
  const int nt = prob_.nt;
  const double2* prev = m0;
  if (keep_all && series != m0)
    LDDMM_CUDA(cudaMemcpyAsync(series, m0, S * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  for (int s = 0; s < nt; ++s) {
    double2* dst = keep_all ? series + (s + 1) * S : tmp_u_.p + ((s + 1) & 1) * S;
    const double2* in[1] = {prev};
    FinField outs[1] = {FinField{dst, 1.0, nullptr, 0.0}};
    advect_multi(in, 1, depf(ps, s), outs);
    // the finite check reads a vector-sized block; scalars use their own length
    launch_nonfinite_flag(S, dst, part2_.p, slots_.p + 16 + s, stream_);
    prev = dst;
  }
  if (last) LDDMM_CUDA(cudaMemcpyAsync(last, prev, S * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  finish_finite_checks(nt);
}

// Backward SL with source src(q) = -(q * div v) [+ div v for the Jacobian factor]
// (variants.hpp:454-457 scalar continuity, 482-489 jacobian factor)
void Engine::solve_scalar_continuity_bwd(ProviderState& ps, const double2* q1, double2* series, bool jf) {
  if (prob_.rk4) {
    rk4_scalar_continuity_bwd(ps, q1, series, jf);
    return;
  }
  const long long S = kprod();
  const int nt = prob_.nt;
  const double sdt = -1.0 / nt;
  if (q1)
    LDDMM_CUDA(cudaMemcpyAsync(series + nt * S, q1, S * sizeof(double2), cudaMemcpyDeviceToDevice, stream_));
  else
    LDDMM_CUDA(cudaMemsetAsync(series + nt * S, 0, S * sizeof(double2), stream_));
  for (int s = 0; s < nt; ++s) {
    const int from = nt - s, to = nt - s - 1;
    const double2* q = series + from * S;
    double2 *sf = bt(0), *A = bt(1), *F = bt(2), *qs = bt(3), *ft = bt(4), *tmp = bt(5);
    small_product(0, q, divnode(ps, from), sf, -1.0, jf ? divnode(ps, from) : nullptr, 1.0);  // src(q_from)
    const double2* in[2] = {q, sf};
    FinField outs[2] = {FinField{A, 1.0, nullptr, 0.0}, FinField{F, 1.0, nullptr, 0.0}};
    advect_multi(in, 2, depb(ps, to), outs);
    launch_axpy(S, sdt, F, A, qs, stream_);
    small_product(0, qs, divnode(ps, to), ft, -1.0, jf ? divnode(ps, to) : nullptr, 1.0);  // src(q*)
    launch_axpy(S, 0.5 * sdt, ft, A, tmp, stream_);
    launch_axpy(S, 0.5 * sdt, F, tmp, series + to * S, stream_);
    launch_nonfinite_flag(S, series + to * S, part2_.p, slots_.p + 16 + s, stream_);
  }
  finish_finite_checks(nt);
}

// generic truncated product on the small grid with a caller-built prep list
void Engine::small_custom(const PrepArgs& pa, int prodop, double2* out, int nout, double alpha, const double2* add,
                          double beta) {
  const long long M = small_.npts(), K = kprod();
  embed_fields(small_, pa, sgrid_.p, sD_.p, sE1_.p, sE2_.p);
  const long long off = prodop == 3 ? 3 * M : (prodop == 0 || prodop == 1 ? 9 * M : M);
  launch_products(prodop, M, sgrid_.p, sgrid_.p + off, sacc_.p, 1.f, true, stream_);
  FinArgs fa{};
  fa.nf = nout;
  for (int c = 0; c < nout; ++c)
    fa.f[c] = FinField{out + c * K, alpha * small_ratio_, add ? add + c * K : nullptr, beta};
  project_fields(small_, sacc_.p, fa, sG1_.p, sG2_.p, sG3_.p);
}

// D_t dm = -grad(m_i) . dv, forward from 0 (variants.hpp:512-519), merged advect
void Engine::solve_incremental_image(ProviderState& ps, const double2* dv, double2* series) {
  if (prob_.rk4) {
    rk4_incremental_image(ps, dv, series);
    return;
  }
  const long long S = kprod(), K = kprod();
  const int nt = prob_.nt;
  const double dt = 1.0 / nt;
  double2* src = src_.p;  // (nt+1) scalars
  for (int i = 0; i <= nt; ++i) {
    PrepArgs pa{};
    pa.nf = 6;
    for (int a = 0; a < 3; ++a) pa.f[a] = PrepField{m_ser_.p + i * S, SYM_DERIV_X + a, 1.0};
    for (int c = 0; c < 3; ++c) pa.f[3 + c] = PrepField{tvnode(dv, i) + c * K, SYM_NONE, 1.0};
    small_custom(pa, 3, src + i * S, 1, -1.0, nullptr, 0.0);  // -star_dot(grad m_i, dv_i)
  }
  LDDMM_CUDA(cudaMemsetAsync(series, 0, S * sizeof(double2), stream_));
  for (int s = 0; s < nt; ++s) {
    double2* in = bt(0);
    launch_axpy(S, 0.5 * dt, src + s * S, series + s * S, in, stream_);
    const double2* ins[1] = {in};
    FinField outs[1] = {FinField{series + (s + 1) * S, 1.0, src + (s + 1) * S, 0.5 * dt}};
    advect_multi(ins, 1, depf(ps, s), outs);
    launch_nonfinite_flag(S, series + (s + 1) * S, part2_.p, slots_.p + 16 + s, stream_);
  }
  finish_finite_checks(nt);
}

// out = L like + sum_i w_i star(Lam_i, grad M_i)   (variants.hpp:298-301,357-362; linear assembly)
void Engine::assemble_star_grad(const double2* Lam, const double2* Mser, const double2* like, double2* out) {
  const long long S = kprod(), V = vec_elems(), M = small_.npts(), K = kprod();
  const int nt = prob_.nt;
  const auto w = trap_w(nt);
  if (!prob_.stationary) {  // out_i = L like_i + star(Lam_i, grad M_i)  (variants.hpp:364-368)
    for (int i = 0; i <= nt; ++i) {
      PrepArgs pa{};
      pa.nf = 4;
      pa.f[0] = PrepField{Lam + i * S, SYM_NONE, 1.0};
      for (int a = 0; a < 3; ++a) pa.f[1 + a] = PrepField{Mser + i * S, SYM_DERIV_X + a, 1.0};
      double2* tmp = bt(7);
      small_custom(pa, 2, tmp, 3, 1.0, nullptr, 0.0);
      double2* lv = bt(8);
      launch_sobolev(like + i * V, lv, 3, full_.K, full_.omega_unit, prob_.alpha, prob_.s, false, stream_);
      launch_axpy(V, 1.0, lv, tmp, out + i * V, stream_);
    }
    return;
  }
  for (int i = 0; i <= nt; ++i) {
    PrepArgs pa{};
    pa.nf = 4;
    pa.f[0] = PrepField{Lam + i * S, SYM_NONE, 1.0};
    for (int a = 0; a < 3; ++a) pa.f[1 + a] = PrepField{Mser + i * S, SYM_DERIV_X + a, 1.0};
    embed_fields(small_, pa, sgrid_.p, sD_.p, sE1_.p, sE2_.p);
    launch_products(2, M, sgrid_.p, sgrid_.p + M, sacc_.p, (float)w[i], i == 0, stream_);
  }
  double2* tmp = bt(7);
  FinArgs fa{};
  fa.nf = 3;
  for (int c = 0; c < 3; ++c) fa.f[c] = FinField{tmp + c * K, small_ratio_, nullptr, 0.0};
  project_fields(small_, sacc_.p, fa, sG1_.p, sG2_.p, sG3_.p);
  double2* lv = bt(8);
  launch_sobolev(like, lv, 3, full_.K, full_.omega_unit, prob_.alpha, prob_.s, false, stream_);
  launch_axpy(V, 1.0, lv, tmp, out, stream_);
}

// spline coefficients of a grid field (ScalarSampler, interp.hpp:94-96), fp64 recursion
void Engine::grid_spline(const float* f, float* coef) {
  const long long N = npts();
  launch_f32_to_f64(N, f, f64c_.p, stream_);
  launch_prefilter3d(f64c_.p, full_.N, stream_);
  launch_f64_to_f32(N, f64c_.p, coef, stream_);
}

// lambda_i = pi(J_i (lam1 o psi_i)), i = 0..nt (variants.hpp:413-420, 329-333)
void Engine::lambda_nodes_state(const float* lam1, double2* out_series) {
  const long long N = npts(), S = kprod();
  const int nt = prob_.nt;
  grid_spline(lam1, lcoef_.p);
  for (int i = 0; i <= nt; ++i) {
    launch_warp_by_displacement(lcoef_.p, 1, psi_f_.p + i * 3 * N, h_, gridB_.p, full_.N, stream_,
                                pullback_large_);
    launch_mul_f32(N, jac_f_.p + i * N, gridB_.p, gridB_.p, stream_);
    project(gridB_.p, 1, out_series + i * S);
  }
}

// forward_original (variants.hpp:373-384); returns sum(res^2)
double Engine::forward_original(bool with_adjoint, const double2* v, bool have_m) {
  const long long N = npts(), S = kprod();
  const int nt = prob_.nt;
  (void)v;
  if (!have_m) solve_image_forward(prov_, m0_.p, m_ser_.p, true, nullptr);  // else adopted from the trial
  embed(m_ser_.p + nt * S, 1, m1_.p, false);
  const int g = launch_residual(N, m1_.p, I1_.p, res_.p, part_.p, stream_);
  const double ss = reduce(g, 0);
  if (with_adjoint) {
    launch_affine_f32(N, res_.p, (float)(-2.0 / prob_.sigma2), 0.f, gridB_.p, stream_);
    double2* lam1 = bt(10);
    project(gridB_.p, 1, lam1);
    solve_scalar_continuity_bwd(prov_, lam1, lam_ser_.p, false);
  }
  return ss;
}

double Engine::energy_original(const double2* v) {
  const long long N = npts(), S = kprod();
  trial_valid_ = false;  // set again only when this trial completes
  provider_build(v, trial_prov_, false);
  const double2* last;
  if (trial_reuse_ok()) {
    // keep the whole image series for a forward at the same velocity (see forward())
    solve_image_forward(trial_prov_, m0_.p, trial_mser_.p, true, nullptr);
    last = trial_mser_.p + prob_.nt * S;
  } else {
    solve_image_forward(trial_prov_, m0_.p, nullptr, false, bt(11));
    last = bt(11);
  }
  embed(last, 1, trial_m1_.p, false);
  const int g = launch_residual(N, trial_m1_.p, I1_.p, trial_res_.p, part_.p, stream_);
  const double ss = reduce(g, 0);
  if (trial_reuse_ok()) trial_valid_ = true;
  return reg_energy(v) + ss * cell_volume_ / prob_.sigma2;
}

// forward_state (variants.hpp:386-422); returns sum(res^2)
double Engine::forward_state(bool with_adjoint, bool have_u) {
  const long long N = npts(), S = kprod(), V = vec_elems();
  const int nt = prob_.nt;
  if (!have_u) solve_displacement_fwd(prov_, u_.p, true, nullptr);  // else adopted from the trial
  double ss = 0.0;
  warp_m1(u_.p + nt * V, m1_.p, res_.p, false, &ss);
  if (!with_adjoint) return ss;
  // grad_src_warped from the band-filtered gradient (variants.hpp:176-178,421); ugrid_ = iota(u(1))
  launch_warp_by_displacement(fgI0coef_.p, 3, ugrid_.p, h_, m1_.p + N, full_.N, stream_, pullback_large_);
  // image reconstructions m_i = pi(I0 o (x - iota(u_i)))
  for (int i = 0; i <= nt; ++i) {
    embed(u_.p + i * V, 3, ugrid_.p, false);
    launch_warp_by_displacement(I0coef_.p, 1, ugrid_.p, h_, gridB_.p, full_.N, stream_, pullback_large_);
    project(gridB_.p, 1, m_ser_.p + i * S);
  }
  solve_displacement(prov_, false, nu_ser_.p);
  solve_scalar_continuity_bwd(prov_, nullptr, bigU_ser_.p, true);
  for (int i = 0; i <= nt; ++i) {
    embed(bigU_ser_.p + i * S, 1, jac_f_.p + i * N, false);
    launch_affine_f32(N, jac_f_.p + i * N, -1.f, 1.f, jac_f_.p + i * N, stream_);  // J = -iota(U) + 1
    embed(nu_ser_.p + i * V, 3, psi_f_.p + i * 3 * N, false);
  }
  launch_affine_f32(N, res_.p, (float)(-2.0 / prob_.sigma2), 0.f, gridB_.p, stream_);  // lambda1
  lambda_nodes_state(gridB_.p, lam_ser_.p);
  return ss;
}

void Engine::hessvec_original(const double2* dv, double2* out) {
  const long long S = kprod();
  const int nt = prob_.nt;
  solve_incremental_image(prov_, dv, dm_ser_.p);
  double2* dlam1 = bt(10);
  launch_scale(S, -2.0 / prob_.sigma2, dm_ser_.p + nt * S, dlam1, stream_);
  solve_scalar_continuity_bwd(prov_, dlam1, dseries_.p, false);
  assemble_star_grad(dseries_.p, m_ser_.p, dv, out);
}

void Engine::hessvec_state(const double2* dv, double2* out) {
  const long long N = npts(), V = vec_elems();
  const int nt = prob_.nt;
  solve_incremental_displacement(prov_, dv, dseries_.p);
  embed(dseries_.p + nt * V, 3, ugrid_.p, false);  // du1
  launch_dlam1(N, m1_.p + N, ugrid_.p, -2.0 / prob_.sigma2, gridB_.p, stream_);
  lambda_nodes_state(gridB_.p, dm_ser_.p);
  assemble_star_grad(dm_ser_.p, m_ser_.p, dv, out);
}

}  // namespace lddmm_b200
