"""2-D registrations on the device (GridSpec d = 2, core.hpp:49-52): the engine runs a 2-D
problem as a 3-D one with the z axis replicated (Problem::zrep) and the C ABI keeps the
reference's 2-D layouts.  Parity against the reference's own 2-D acceptance workloads
(proj/tests/acceptance.cpp), run once by the unmodified reference
(tools/ref_2d_golden.py -> tests/golden/accept2d_ref.npz):

* gates 4-6 (run_blob, acceptance.cpp:173-195): the 10 blob pairs on 64^2, band 16,
  deformation-state, SL nt = 5 and RK4 nt = 25; GN / PCG / step lengths / stop identical
  and the SURVEY.md §8(c) tolerances for seeds 1, 2; final mse_rel and the min inverse-map
  Jacobian for all 20 runs;
* gate 8 (check_label_overlap, acceptance.cpp:308-345): the two-disc cases, three
  variants, SL nt = 5: Dice of the warped labels and the gate verdict.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "accept2d_ref.npz")
VARIANTS = ["original", "state_equation", "deformation_state_equation"]
DIMS, SP, BAND = (64, 64), (1.0, 1.0), (16, 16)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def relerr(x, r):
    return abs(x - r) / abs(r) if r != 0 else abs(x)


def gold():
    if not os.path.exists(GOLD):
        pytest.skip("accept2d_ref.npz not generated (tools/ref_2d_golden.py)")
    return np.load(GOLD)


def model(L, src, tgt, variant, nt, sigma2, integrator="sl"):
    return L.Model(L.BandSpec(L.GridSpec(DIMS, SP), BAND), src, tgt, variant, nt, sigma2, integrator=integrator)


@pytest.mark.parametrize("seed", [1, 2])
def test_2d_blob_registration_matches_reference(cuda, seed):
    from oracle import ref
    from paper_2006_06823_b200 import lddmm as L
    z = gold()
    s, t = ref.blob_pair(DIMS, SP, seed)
    m = model(L, s, t, "deformation_state_equation", 5, 0.01)
    res = L.optimize(m, None, L.OptimizeOptions(max_iter=15, pcg_max_iter=5))
    hist = z[f"blob{seed}_history"]
    assert len(res.history) == hist.shape[0]
    worst = 0.0
    for r, row in zip(res.history, hist):
        assert r.pcg_iters == int(row[6]) and r.pcg_fallback == bool(row[7]) and r.epsilon == row[8]
        worst = max(worst, relerr(r.energy, row[1]))
        assert abs(r.mse_rel - row[4]) <= 1e-5
        assert abs(r.cfl - row[9]) <= 1e-6 * max(1.0, row[9])
    ev = rel(res.v.numpy(), z[f"blob{seed}_v"])
    _, _, jac = L.compute_maps(m, res.v)
    ej = float(np.max(np.abs(jac - z[f"blob{seed}_jac"])))
    print(f"2-D blob {seed}: GN {res.iterations}, max rel E {worst:.1e}, velocity {ev:.1e}, Jacobian {ej:.1e}")
    assert worst <= 1e-5 and ev <= 1e-4 and ej <= 1e-4


def test_2d_acceptance_gates_4_to_6(cuda):
    """The blob suite on the device: per run the reference's final mse_rel (1e-4), its
    convergence flag and iteration count, and the min inverse-map Jacobian (1e-3); the
    gates themselves: mean |mse_rel gap SL - RK4| <= 0.05 (gate 4), min det > 0 (gate 6)."""
    from oracle import ref
    from paper_2006_06823_b200 import lddmm as L
    z = gold()
    blob = z["blob"]
    got = {}
    for row in blob:
        seed, integ = int(row[0]), "sl" if row[1] == 0 else "rk4"
        s, t = ref.blob_pair(DIMS, SP, seed)
        m = model(L, s, t, "deformation_state_equation", 5 if integ == "sl" else 25, 0.01, integ)
        res = L.optimize(m, None, L.OptimizeOptions(max_iter=15, pcg_max_iter=5))
        _, _, jac = L.compute_maps(m, res.v)
        got[(seed, integ)] = (res.history[-1].mse_rel, res.converged, res.iterations, jac[2])
        assert abs(res.history[-1].mse_rel - row[2]) <= 1e-4, (seed, integ)
        assert res.converged == bool(row[3]) and res.iterations == int(row[4]), (seed, integ)
        assert abs(jac[2] - row[5]) <= 1e-3, (seed, integ)
    gap = np.mean([abs(got[(k, "sl")][0] - got[(k, "rk4")][0]) for k in range(1, 11)])
    min_det = min(v[3] for v in got.values() if v[1])
    print(f"2-D gates 4-6 on the device: mean |mse gap| {gap:.4f} (gate <= 0.05), min det {min_det:.3f} (gate > 0)")
    assert gap <= 0.05 and min_det > 0.0


def test_2d_acceptance_gate_8_dice(cuda):
    """Two-disc label overlap: per case and variant the Dice of the nearest-neighbour-warped
    source labels within 5e-3 of the reference's, and the same gate verdict (deformation
    gain >= 0.15 over the initial Dice and the variant ordering)."""
    from oracle import ref
    from paper_2006_06823_b200 import lddmm as L
    z = gold()
    g8 = z["gate8"]
    dice = np.zeros((10, 3))
    init = np.zeros(10)
    for row in g8:
        seed, vi = int(row[0]), int(row[1])
        src, tgt, sl, tl = ref.two_disc_case(DIMS, SP, seed)
        m = model(L, src, tgt, VARIANTS[vi], 5, 0.05)
        res = L.optimize(m, None, L.OptimizeOptions(max_iter=30, pcg_max_iter=5, grad_tol=1e-3))
        fwd, _, _ = L.compute_maps(m, res.v)
        warped = L.warp(m.ctx, sl, fwd, "nearest")
        dice[seed - 1, vi] = L.mean_dice(m.ctx, warped, tl)
        init[seed - 1] = row[3]
        assert abs(dice[seed - 1, vi] - row[2]) <= 5e-3, (seed, VARIANTS[vi], dice[seed - 1, vi], row[2])
    ref_dice = np.zeros((10, 3))
    for row in g8:
        ref_dice[int(row[0]) - 1, int(row[1])] = row[2]
    mean, rmean = dice.mean(0), ref_dice.mean(0)
    verdict = lambda d: (d[2] - init.mean() >= 0.15) and d[2] >= d[0] and d[2] >= d[1]  # noqa: E731
    print(f"2-D gate 8: device mean Dice {np.round(mean, 4)} vs reference {np.round(rmean, 4)}; "
          f"initial {init.mean():.4f}; gate {'PASS' if verdict(mean) else 'FAIL'} "
          f"(reference {'PASS' if verdict(rmean) else 'FAIL'})")
    assert verdict(mean) == verdict(rmean)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("integrator", ["sl", "rk4"])
def test_2d_model_ops_match_reference(cuda, variant, integrator):
    """forward (energies, cfl), gradient and one Hessian-vector product of a 2-D model
    against the reference library itself on the same inputs (32 x 40 grid, band 8 x 12)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2006_06823_b200 import lddmm as L
    dims, band, nt = (32, 40), (8, 12), 4
    s, t = ref.blob_pair(dims, (1.0, 1.0), 3)
    rm = ref.RefModel(s, t, dims, (1.0, 1.0), band, variant, nt, 0.05, integrator=integrator)
    v = ref.random_band_field(dims, (1.0, 1.0), band, 11, 1.2, 2.0)[None]
    dv = ref.random_band_field(dims, (1.0, 1.0), band, 12, 0.5, 2.0)[None]
    want_e = rm.forward(v, True)
    want_g = rm.gradient()
    want_h = rm.hessvec(dv)
    m = L.Model(L.BandSpec(L.GridSpec(dims, (1.0, 1.0)), band), s, t, variant, nt, 0.05, integrator=integrator)
    e = m.forward(m.velocity(v), True)
    g = m.gradient().numpy()
    h = m.hessvec(m.velocity(dv)).numpy()
    for k in ("energy", "energy_reg", "energy_data"):
        assert relerr(e[k], want_e[k]) <= 1e-5, (k, e[k], want_e[k])
    assert abs(e["cfl"] - want_e["cfl"]) <= 1e-6 * max(1.0, want_e["cfl"])
    assert rel(g, want_g) <= 1e-4 and rel(h, want_h) <= 1e-4, (rel(g, want_g), rel(h, want_h))
