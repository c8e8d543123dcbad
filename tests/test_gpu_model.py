"""GPU parity of the deformation-state model and the GN-Krylov driver against the
CPU oracle (oracle/lddmm_np.py, pinned to the reference in tests/test_oracle.py).

Mirrors test_variants.cpp (forward/gradient/hessvec, Hessian symmetry and
linearity) and test_optimizer.cpp (descent, stop rules) at sizes the oracle
finishes in seconds.  Tolerances: energies rel 1e-5, band vectors
rel-L2 1e-4, GN/PCG iteration counts and stop reason identical.
"""
import os

import numpy as np
import pytest

from oracle import lddmm_np as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def smooth_pair(dims, seed):
    from paper_2006_06823_b200 import phantoms
    rng = np.random.default_rng(seed)
    c = tuple(n / 2 for n in dims)
    s = phantoms.tanh_ellipsoid(dims, c, tuple(0.3 * n for n in dims), edge=2.5)
    u = phantoms.smooth_displacement(dims, seed, amplitude=1.5, kmax=1, nmodes=3)
    t = phantoms.tanh_ellipsoid(dims, c, tuple(0.3 * n for n in dims), edge=2.5, disp=u)
    s = s + 0.05 * rng.standard_normal(dims) * 0
    return phantoms.rescale_unit(s), phantoms.rescale_unit(t)


def rand_band(b, seed, amp):
    g = b.grid
    rng = np.random.default_rng(seed)
    c = O.project(rng.standard_normal((3,) + g.dims), b)
    k2 = sum(w * w for w in np.meshgrid(*[b.signed_freq(a).astype(float) for a in range(3)], indexing="ij"))
    c = c * np.exp(-0.3 * k2)
    return c * (amp / np.max(np.abs(O.embed(c, b))))


SETUPS = [
    dict(dims=(16, 12, 14), band=(8, 8, 6), nt=3, sigma2=0.5),
    dict(dims=(20, 20, 20), band=(8, 8, 8), nt=4, sigma2=0.05),
]


VARIANTS = ["deformation_state_equation", "original", "state_equation"]


def build(setup, variant="deformation_state_equation"):
    from paper_2006_06823_b200 import lddmm as L
    dims, band = setup["dims"], setup["band"]
    I0, I1 = smooth_pair(dims, 3)
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, band)
    om = O.Model(b, I0, I1, variant, setup["nt"], setup["sigma2"])
    gm = L.Model(L.BandSpec(L.GridSpec(dims), band), I0, I1, variant, setup["nt"], setup["sigma2"])
    return b, om, gm, I0, I1


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("setup", SETUPS)
def test_forward_gradient_hessvec(cuda, setup, variant):
    """Model::forward / gradient / hessvec / precondition for the three variants (variants.hpp:262-353)."""
    b, om, gm, I0, I1 = build(setup, variant)
    v = rand_band(b, 21, 1.2)
    dv = rand_band(b, 22, 1.0)
    c = om.forward(v, True)
    e = gm.forward(gm.velocity(v), True)
    assert abs(e["energy"] - c.energy) <= 1e-5 * abs(c.energy)
    assert abs(e["energy_data"] - c.energy_data) <= 1e-5 * abs(c.energy_data)
    assert abs(e["energy_reg"] - c.energy_reg) <= 1e-9 * abs(c.energy_reg)
    assert abs(e["cfl"] - c.cfl) <= 1e-5 * c.cfl
    m1, res = gm.fields()
    assert np.max(np.abs(m1 - c.m1)) < 1e-5
    if variant != "original":
        u = gm.series("u")
        assert rel(u, np.stack(c.u)) < 1e-5
    if variant == "deformation_state_equation":
        rho = gm.series("rho")
        assert rel(rho, np.stack(c.rho)) < 1e-4
    g_gpu = gm.gradient().numpy()[0]
    assert rel(g_gpu, om.gradient(c)) < 1e-4
    hv = gm.hessvec(gm.velocity(dv)).numpy()[0]
    assert rel(hv, om.hessvec(c, dv)) < 1e-4
    pc = gm.precondition(gm.velocity(dv)).numpy()[0]
    assert rel(pc, om.precondition(dv)) < 1e-13
    # energy() leaves the cache alone (the Armijo trials of optimizer.hpp:201-208)
    e2 = gm.energy(gm.velocity(dv * 0.3))
    assert abs(e2 - om.energy(dv * 0.3)) <= 1e-5 * abs(e2)
    hv2 = gm.hessvec(gm.velocity(dv)).numpy()[0]
    assert rel(hv2, hv) < 1e-12


def test_hessian_symmetry_linearity(cuda):
    """test_variants.cpp:105-155 — <a, H b> = <H a, b> to O(dt^2); H linear."""
    b, om, gm, I0, I1 = build(SETUPS[1])
    v = rand_band(b, 31, 1.0)
    a = rand_band(b, 32, 1.0)
    bb = rand_band(b, 33, 1.0)
    gm.forward(gm.velocity(v), True)
    va, vb = gm.velocity(a), gm.velocity(bb)
    ha, hb = gm.hessvec(va), gm.hessvec(vb)
    s1, s2 = gm.tv_inner(va, hb), gm.tv_inner(ha, vb)
    assert abs(s1 - s2) <= 0.05 * max(abs(s1), abs(s2))
    hab = gm.hessvec(gm.velocity(2.0 * a + bb)).numpy()
    assert rel(hab, 2.0 * ha.numpy() + hb.numpy()) < 1e-5


@pytest.mark.parametrize("variant,fixed_work", [(v, f) for v in VARIANTS for f in (False, True)])
def test_optimize_matches_oracle(cuda, variant, fixed_work):
    """optimize (optimizer.hpp:143-262): same GN iterations, PCG iterations, step lengths and
    stop reason; energies per iteration within 1e-5 relative (config-3 style: every variant)."""
    from paper_2006_06823_b200 import lddmm as L
    setup = SETUPS[1]
    b, om, gm, I0, I1 = build(setup, variant)
    kw = dict(max_iter=4)
    if fixed_work:
        kw.update(grad_tol=0.0, energy_tol=0.0, step_tol=0.0, pcg_tol=0.0, max_iter=3)
    ref = O.optimize(om, om.zero_velocity(), O.Options(**kw))
    res = L.optimize(gm, None, L.OptimizeOptions(**kw))
    assert res.stop == ref["stop"]
    assert res.iterations == ref["iterations"]
    assert len(res.history) == len(ref["history"])
    for r, q in zip(res.history, ref["history"]):
        assert r.pcg_iters == q["pcg_iters"]
        assert r.pcg_fallback == q["pcg_fallback"]
        assert r.epsilon == q["epsilon"]
        assert abs(r.energy - q["energy"]) <= 1e-5 * abs(q["energy"])
        assert abs(r.mse_rel - q["mse_rel"]) <= 1e-5
    assert rel(res.v.numpy()[0], ref["v"]) < 1e-4


def test_maps_and_jacobian(cuda):
    """compute_maps + map_jacobian_determinant ranges (metrics.hpp:24-79)."""
    from paper_2006_06823_b200 import lddmm as L
    b, om, gm, I0, I1 = build(SETUPS[0])
    v = rand_band(b, 41, 1.5)
    f, i, jac = L.compute_maps(gm, gm.velocity(v))
    wf, wi = O.compute_maps(om, v)
    assert rel(f, wf) < 1e-4 and rel(i, wi) < 1e-4
    jf = O.map_jacobian_determinant(wf, b.grid)
    ji = O.map_jacobian_determinant(wi, b.grid)
    assert np.allclose(jac, [jf.min(), jf.max(), ji.min(), ji.max()], atol=1e-4)


def test_divergence_reported(cuda):
    """A blown-up velocity raises DivergenceError with a step index (transport.hpp:225-228)."""
    from paper_2006_06823_b200 import lddmm as L
    b, om, gm, I0, I1 = build(SETUPS[0])
    v = rand_band(b, 51, 1.0)
    v[0, 1, 1, 1] = np.nan
    with pytest.raises(L.DivergenceError):
        gm.forward(gm.velocity(v), True)


@pytest.mark.parametrize("variant", VARIANTS)
def test_nonstationary_model_and_optimize(cuda, variant):
    """Nonstationary parameterization on the device vs the oracle: forward / gradient /
    hessvec and a short optimize with identical GN/PCG path (core.hpp:290-316,
    transport.hpp:120-187, variants.hpp:364-368)."""
    from paper_2006_06823_b200 import lddmm as L
    setup = SETUPS[0]
    dims, band, nt = setup["dims"], setup["band"], setup["nt"]
    I0, I1 = smooth_pair(dims, 3)
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, band)
    om = O.Model(b, I0, I1, variant, nt, setup["sigma2"], stationary=False)
    gm = L.Model(L.BandSpec(L.GridSpec(dims), band), I0, I1, variant, nt, setup["sigma2"],
                 parameterization="nonstationary")
    v = [rand_band(b, 90 + i, 1.0) for i in range(nt + 1)]
    dv = [rand_band(b, 95 + i, 1.0) for i in range(nt + 1)]
    c = om.forward(v, True)
    e = gm.forward(gm.velocity(np.stack(v)), True)
    assert abs(e["energy"] - c.energy) <= 1e-5 * abs(c.energy)
    assert abs(e["cfl"] - c.cfl) <= 1e-5 * c.cfl
    assert rel(gm.gradient().numpy(), np.stack(om.gradient(c))) < 1e-4
    assert rel(gm.hessvec(gm.velocity(np.stack(dv))).numpy(), np.stack(om.hessvec(c, dv))) < 1e-4
    ref = O.optimize(om, om.zero_velocity(), O.Options(max_iter=3))
    res = L.optimize(gm, None, L.OptimizeOptions(max_iter=3))
    assert res.stop == ref["stop"] and res.iterations == ref["iterations"]
    for r, q in zip(res.history, ref["history"]):
        assert r.pcg_iters == q["pcg_iters"] and r.epsilon == q["epsilon"]
        assert abs(r.energy - q["energy"]) <= 1e-5 * abs(q["energy"])
    assert rel(res.v.numpy(), np.stack(ref["v"])) < 1e-4


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("tag", ["s", "n"])
def test_rk4_matches_reference(cuda, variant, tag):
    """RK4 integrator on the device (transport.hpp:234-258, rk4 branches of
    variants.hpp:444-547) against the reference's own outputs (tests/golden/model_rk4.npz):
    forward energies, gradient, hessvec (stationary and nonstationary), a short optimize
    with identical GN/PCG path, and the endpoint maps."""
    from paper_2006_06823_b200 import lddmm as L
    z = np.load(os.path.join(GOLD, "model_rk4.npz"))
    dims = tuple(int(x) for x in z["dims"])
    band, nt = tuple(int(x) for x in z["band"]), int(z["nt"])
    st = tag == "s"
    gm = L.Model(L.BandSpec(L.GridSpec(dims), band), z["I0"], z["I1"], variant, nt, float(z["sigma2"]),
                 parameterization="stationary" if st else "nonstationary", integrator="rk4")
    v = z["v"] if st else z["vn"]
    dv = z["dv"] if st else z["dvn"]
    e = gm.forward(gm.velocity(v), True)
    ref = z[f"{variant}_{tag}_energy"]
    assert abs(e["energy"] - ref[0]) <= 1e-5 * abs(ref[0])
    assert abs(e["energy_reg"] - ref[1]) <= 1e-9 * abs(ref[1])
    assert abs(e["cfl"] - ref[3]) <= 1e-5 * ref[3]
    assert rel(gm.gradient().numpy(), z[f"{variant}_{tag}_gradient"]) < 1e-4
    assert rel(gm.hessvec(gm.velocity(dv)).numpy(), z[f"{variant}_{tag}_hessvec"]) < 1e-4
    if st:
        res = L.optimize(gm, None, L.OptimizeOptions(max_iter=3))
        hist = z[f"{variant}_opt_history"]
        assert L.STOP_REASONS.index(res.stop) == int(z[f"{variant}_opt_stop"])
        assert len(res.history) == hist.shape[0]
        for r, row in zip(res.history, hist):
            assert r.pcg_iters == int(row[2]) and r.epsilon == row[3]
            assert abs(r.energy - row[1]) <= 1e-5 * abs(row[1])
        assert rel(res.v.numpy(), z[f"{variant}_opt_v"]) < 1e-4
    if st and variant == "deformation_state_equation":
        f, i, jac = L.compute_maps(gm, gm.velocity(v))
        assert rel(f, z["maps_fwd"]) < 1e-4 and rel(i, z["maps_inv"]) < 1e-4
        assert np.allclose(jac, z["maps_jac"], atol=1e-4)


def test_rk4_needs_two_steps(cuda):
    """rk4_integrate rejects nt < 2 (transport.hpp:236) — ShapeError at context creation."""
    from paper_2006_06823_b200 import lddmm as L
    with pytest.raises(L.ShapeError):
        L.Context(L.BandSpec(L.GridSpec((8, 8, 8)), (4, 4, 4)), nt=1, integrator="rk4")
