"""Known-answer tests of the reference, run on the device.

The reference's unit tests pin this path with analytic or self-consistency
checks rather than stored vectors; these are their band-representation, 3-D
counterparts through the C ABI:

- gradient vs central finite differences of the energy, every variant x
  integrator x parameterisation (test_variants.cpp:48-74, test_helpers.hpp:68-98);
- zero velocity: m1 is the source, E_reg = 0, E = |res|^2 / sigma2
  (test_variants.cpp:89-103);
- curvature positive at zero velocity (test_variants.cpp:105-155);
- departure points of a constant flow move exactly one step upstream
  (test_transport.cpp:62-79);
- band advect by a constant shift equals the analytic phase shift
  (test_transport.cpp:170-181);
- SL and RK4 agree with a fine RK4 reference (test_transport.cpp:148-168);
- descent reduces energy and mismatch; iteration cap (test_optimizer.cpp:117-143,197-207).

fp32 grid fields set the floor of the finite-difference check: the step is 1e-3
(the reference uses 1e-4 in fp64) and the tolerance the reference's 1e-3.
"""
import os

import numpy as np
import pytest

from oracle import lddmm_np as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DIMS, BAND, NT = (16, 12, 14), (8, 8, 6), 3


def images(seed=41):
    z = np.load(os.path.join(GOLD, "model.npz"))
    return z["I0"], z["I1"]


def rand_band(b, seed, amp, nodes=None):
    g = b.grid
    rng = np.random.default_rng(seed)

    def one():
        c = O.project(rng.standard_normal((3,) + g.dims), b)
        k2 = sum(w * w for w in np.meshgrid(*[b.signed_freq(a).astype(float) for a in range(3)], indexing="ij"))
        c = c * np.exp(-0.3 * k2)
        return c * (amp / np.max(np.abs(O.embed(c, b))))
    return one() if nodes is None else np.stack([one() for _ in range(nodes)])


def model(variant, integrator, param, sigma2=0.5, nt=NT):
    from paper_2006_06823_b200 import lddmm as L
    I0, I1 = images()
    return L.Model(L.BandSpec(L.GridSpec(DIMS), BAND), I0, I1, variant, nt, sigma2, parameterization=param,
                   integrator=integrator)


VARIANTS = ["deformation_state_equation", "original", "state_equation"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("integrator", ["sl", "rk4"])
@pytest.mark.parametrize("param", ["stationary", "nonstationary"])
def test_gradient_matches_finite_differences(cuda, variant, integrator, param):
    m = model(variant, integrator, param)
    b = O.Band(O.Grid(DIMS, (1.0, 1.0, 1.0)), BAND)
    nodes = None if param == "stationary" else NT + 1
    v = m.velocity(rand_band(b, 901, 0.4, nodes))
    m.forward(v, True)
    g = m.gradient()
    gn = np.sqrt(m.tv_inner(g, g))
    eps, worst = 1e-3, 0.0
    for k in range(3):
        w = m.velocity(rand_band(b, 4321 + 7919 * (k + 1), 1.0, nodes))
        pred = m.tv_inner(g, w)
        ep = m.energy(m.velocity(v.numpy() + eps * w.numpy()))
        em = m.energy(m.velocity(v.numpy() - eps * w.numpy()))
        fd = (ep - em) / (2 * eps)
        worst = max(worst, abs(pred - fd) / max(gn * np.sqrt(m.tv_inner(w, w)), 1e-12))
    assert worst < 1e-3


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("integrator", ["sl", "rk4"])
def test_zero_velocity_transports_the_source(cuda, variant, integrator):
    m = model(variant, integrator, "stationary")
    I0, I1 = images()
    e = m.forward(m.zero_velocity(), False)
    m1, res = m.fields()
    if variant == "original":  # the image state is the band scalar pi(I0) (variants.hpp:374)
        b = O.Band(O.Grid(DIMS, (1.0, 1.0, 1.0)), BAND)
        I0 = O.embed(O.project(I0, b), b)
    assert np.max(np.abs(m1 - I0)) < 1e-5
    assert np.max(np.abs(res - (I0 - I1))) < 1e-5
    assert e["energy_reg"] == 0.0
    assert abs(e["energy"] - float(np.sum(res * res)) / 0.5) <= 1e-6 * e["energy"]


@pytest.mark.parametrize("variant", VARIANTS)
def test_curvature_positive_at_zero_velocity(cuda, variant):
    m = model(variant, "sl", "stationary")
    b = O.Band(O.Grid(DIMS, (1.0, 1.0, 1.0)), BAND)
    m.forward(m.zero_velocity(), True)
    for seed in (5, 6, 7):
        dv = m.velocity(rand_band(b, seed, 1.0))
        assert m.tv_inner(dv, m.hessvec(dv)) > 0.0


def test_constant_flow_departure(cuda):
    from paper_2006_06823_b200 import lddmm as L
    h = (0.5, 0.5, 0.5)
    nt = 4
    ctx = L.Context(L.BandSpec(L.GridSpec((16, 16, 16), h), (8, 8, 8)), nt=nt)
    vel = np.array([0.9, -0.4, 0.3])
    v = np.zeros((3, 8, 8, 8), dtype=np.complex128)
    v[:, 0, 0, 0] = vel * 16 ** 3  # the DC coefficient of a constant field (embed divides by N)
    ops = L.Ops(ctx)
    df, db, cfl = ops.departure(v)
    dt = 1.0 / nt
    for a in range(3):
        assert np.max(np.abs(df[a].cpu().numpy() - (-dt * vel[a] / h[a]))) < 1e-6
        assert np.max(np.abs(db[a].cpu().numpy() - (dt * vel[a] / h[a]))) < 1e-6
    assert abs(cfl - 0.9 * dt / 0.5) < 1e-7  # max |iota(v)| taken over the fp32 grid


def test_band_advect_matches_phase_shift(cuda):
    from paper_2006_06823_b200 import lddmm as L
    import torch
    g = O.Grid((32, 32, 32), (1.0, 1.0, 1.0))
    b = O.Band(g, (8, 8, 8))
    ctx = L.Context(L.BandSpec(L.GridSpec(g.dims), b.bounds))
    rng = np.random.default_rng(61)
    q = O.project(rng.standard_normal(g.dims), b)
    k2 = sum(w * w for w in np.meshgrid(*[b.signed_freq(a).astype(float) for a in range(3)], indexing="ij"))
    q = q * np.exp(-k2 / 1.5 ** 2)
    shift = np.array([1.3, -0.6, 0.45])
    dep = torch.tensor(np.broadcast_to(-shift[:, None, None, None], (3,) + g.dims).copy(), dtype=torch.float32,
                       device="cuda")
    adv = L.Ops.to_complex(L.Ops(ctx).advect(q[None], 1, dep))
    om = np.meshgrid(*[2 * np.pi * b.signed_freq(a) / g.dims[a] for a in range(3)], indexing="ij")
    want = O.embed(q * np.exp(-1j * sum(o * s for o, s in zip(om, shift))), b)
    got = O.embed(adv[0], b)
    assert np.max(np.abs(got - want)) < 2e-3 * max(1.0, np.max(np.abs(O.embed(q, b))))


def test_sl_and_rk4_track_a_fine_rk4_reference(cuda):
    """The image transported by SL (nt = 10) and RK4 (nt = 20) against RK4 with nt = 320."""
    from paper_2006_06823_b200 import lddmm as L
    b = O.Band(O.Grid(DIMS, (1.0, 1.0, 1.0)), BAND)
    v = rand_band(b, 31, 1.2)
    out = {}
    for integ, nt in (("rk4", 320), ("sl", 10), ("rk4", 20)):
        m = model("original", integ, "stationary", nt=nt)
        m.forward(m.velocity(v), False)
        out[(integ, nt)] = m.fields()[0]
    ref = out[("rk4", 320)]
    # the reference's 2-D spatial bounds are 5e-4 (SL, nt = 10) and 1e-7 (RK4, fp64); here
    # 3-D, band-limited, |v| = 1.2 voxels, fp32 grids: measured 7.6e-4 and 6e-8
    assert np.max(np.abs(out[("sl", 10)] - ref)) < 1e-3
    assert np.max(np.abs(out[("rk4", 20)] - ref)) < 1e-6


def test_descent_and_iteration_cap(cuda):
    from paper_2006_06823_b200 import lddmm as L
    z = np.load(os.path.join(GOLD, "synth.npz"))
    s, t = z["blobs3_source"], z["blobs3_target"]
    b = L.BandSpec(L.GridSpec((16, 16, 16)), (8, 8, 8))
    m = L.Model(b, s, t, "deformation_state_equation", 5, 0.01)
    res = L.optimize(m, None, L.OptimizeOptions(max_iter=10))
    h = res.history
    assert len(h) >= 2 and abs(h[0].mse_rel - 1.0) < 1e-6
    assert all(h[i].energy <= h[i - 1].energy + 1e-12 for i in range(1, len(h)))
    assert h[-1].mse_rel < 0.6 and res.final_energy < h[0].energy
    assert res.iterations >= 1 and h[1].pcg_iters >= 1 and not h[1].pcg_fallback and h[1].epsilon > 0
    cap = L.optimize(m, None, L.OptimizeOptions(max_iter=1, grad_tol=0.0, energy_tol=0.0, step_tol=0.0))
    assert cap.stop == "max_iterations" and not cap.converged and cap.iterations == 1
