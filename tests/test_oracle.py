"""Pins the CPU oracle (oracle/lddmm_np.py, a numpy restatement of the reference)
to golden fixtures produced by the REFERENCE ITSELF (tests/golden/make_golden.py
running the unmodified reference headers), plus the reference's own analytic
known-answer tests that apply to this path.  CPU only."""
import os

import numpy as np
import pytest

from oracle import lddmm_np as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def grid_band(z):
    g = O.Grid(tuple(int(x) for x in z["dims"]), tuple(float(x) for x in z["spacing"]))
    return g, O.Band(g, tuple(int(x) for x in z["band"]))


def test_spectral_golden():
    """embed/project/star/jac/jacT/grad/div/Sobolev/band_inner (spectral.hpp:170-573)."""
    z = load("spectral")
    g, b = grid_band(z)
    u, w, s, t, f = z["u"], z["w"], z["s"], z["t"], z["f"]
    assert rel(O.embed(u, b), z["embed_u"]) < 1e-12
    assert rel(O.project(f, b), z["project_f"]) < 1e-12
    assert rel(O.star(s[0], t[0], b), z["star_ss"][0]) < 1e-12
    assert rel(O.star(s[0], u, b), z["star_sv"]) < 1e-12
    assert rel(O.star_dot(u, w, b), z["star_dot"][0]) < 1e-12
    assert rel(O.band_jac_mul(u, w, b), z["jac"]) < 1e-12
    assert rel(O.band_jacT_mul(u, w, b), z["jacT"]) < 1e-12
    assert rel(O.band_gradient(s[0], b), z["grad"]) < 1e-14
    assert rel(O.band_divergence(u, b), z["div"][0]) < 1e-14
    lop = O.Sobolev(0.0025, 2)
    assert rel(lop.apply(u, b), z["sobolev"]) < 1e-14
    assert rel(lop.apply(u, b, True), z["sobolev_inv"]) < 1e-14
    assert abs(O.band_inner(u, w, b) - float(z["inner_uw"])) <= 1e-12 * abs(float(z["inner_uw"]))
    assert rel(O.spectral_gradient(f[0], g), z["sgrad_f0"]) < 1e-12


def test_interp_golden():
    """prefilter and cubic / linear / nearest warps (interp.hpp:23-225)."""
    z = load("interp")
    g = O.Grid(tuple(int(x) for x in z["dims"]), tuple(float(x) for x in z["spacing"]))
    assert rel(O.spline_coefficients(z["f"]), z["coef"]) < 1e-13
    assert rel(O.warp(z["f"], z["pts"], g, "cubic"), z["cubic"][0]) < 1e-13
    assert rel(O.warp(z["f"], z["pts"], g, "linear"), z["linear"][0]) < 1e-13
    assert np.array_equal(O.warp_nearest(z["f"], z["pts"], g), z["nearest"][0])


def test_transport_golden():
    """sl_departure + advect_state + cfl (transport.hpp:67-194)."""
    z = load("transport")
    g, b = grid_band(z)
    nt = int(z["nt"])
    prov = O.Provider(z["v"], nt, b)
    assert np.max(np.abs(prov.departure(0, "forward") - z["Xf"])) < 1e-12
    assert np.max(np.abs(prov.departure(0, "backward") - z["Xb"])) < 1e-12
    assert rel(O.advect_band(z["q"], z["Xf"], b), z["adv_f"]) < 1e-12
    assert rel(O.advect_band(z["q"], z["Xb"], b), z["adv_b"]) < 1e-12
    assert abs(prov.cfl() - float(z["cfl"])) < 1e-14


@pytest.mark.parametrize("variant", ["deformation_state_equation", "original", "state_equation"])
def test_model_golden(variant):
    """Model::forward/gradient/hessvec/precondition for all three variants (variants.hpp:262-353)."""
    z = load("model")
    dims = tuple(int(x) for x in z["dims"])
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, tuple(int(x) for x in z["band"]))
    m = O.Model(b, z["I0"], z["I1"], variant, int(z["nt"]), float(z["sigma2"]))
    v, dv = z["v"][0], z["dv"][0]
    c = m.forward(v, True)
    e = z[f"{variant}_energy"]
    assert np.allclose([c.energy, c.energy_reg, c.energy_data, c.cfl], e, rtol=1e-12, atol=0)
    assert np.max(np.abs(c.m1 - z[f"{variant}_m1"])) < 1e-12
    assert rel(m.gradient(c), z[f"{variant}_gradient"][0]) < 1e-11
    assert rel(m.hessvec(c, dv), z[f"{variant}_hessvec"][0]) < 1e-11
    assert rel(m.precondition(dv), z[f"{variant}_precondition"][0]) < 1e-14
    if variant != "original":
        assert rel(np.stack(c.u), z[f"{variant}_u"]) < 1e-11
    if variant == "deformation_state_equation":
        assert rel(np.stack(c.rho), z[f"{variant}_rho"]) < 1e-11
        fwd, inv = O.compute_maps(m, v)
        assert rel(fwd, z["maps_fwd"]) < 1e-12 and rel(inv, z["maps_inv"]) < 1e-12
        jf = O.map_jacobian_determinant(fwd, g)
        ji = O.map_jacobian_determinant(inv, g)
        assert np.allclose([jf.min(), jf.max(), ji.min(), ji.max()], z["maps_jac"], rtol=1e-12)


@pytest.mark.parametrize("tag", ["parity", "fixed"])
def test_optimize_golden(tag):
    """optimize: identical history (GN/PCG counts, epsilon, stop) and energies (optimizer.hpp:143-262)."""
    z = load("optimize")
    dims = tuple(int(x) for x in z["dims"])
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, tuple(int(x) for x in z["band"]))
    m = O.Model(b, z["I0"], z["I1"], "deformation_state_equation", int(z["nt"]), float(z["sigma2"]))
    kw = dict(max_iter=6) if tag == "parity" else dict(max_iter=3, grad_tol=0.0, energy_tol=0.0, step_tol=0.0,
                                                      pcg_tol=0.0)
    r = O.optimize(m, m.zero_velocity(), O.Options(**kw))
    hist = z[f"{tag}_history"]
    assert O.STOP.index(r["stop"]) == int(z[f"{tag}_stop"])
    assert r["iterations"] == int(z[f"{tag}_iterations"])
    assert len(r["history"]) == hist.shape[0]
    for q, row in zip(r["history"], hist):
        assert q["pcg_iters"] == int(row[6]) and q["epsilon"] == row[8]
        assert np.allclose([q["energy"], q["energy_data"], q["energy_reg"], q["mse_rel"], q["rel_grad"]],
                           row[[1, 2, 3, 4, 5]], rtol=1e-9, atol=1e-14)
    assert rel(r["v"], z[f"{tag}_v"]) < 1e-8


def test_prefilter_symbol_kat():
    """The periodic cubic prefilter equals division by B(k) = prod (4 + 2 cos(2 pi k / N)) / 6 —
    the identity the CUDA engine folds into its embed (interp.hpp:23-63)."""
    rng = np.random.default_rng(0)
    f = rng.standard_normal((10, 12, 8))
    F = np.fft.fftn(f)
    Bs = [(4 + 2 * np.cos(2 * np.pi * np.arange(n) / n)) / 6 for n in f.shape]
    B = Bs[0][:, None, None] * Bs[1][None, :, None] * Bs[2][None, None, :]
    want = np.fft.ifftn(F / B).real
    assert np.max(np.abs(O.spline_coefficients(f) - want)) < 1e-12


def test_small_grid_product_kat():
    """star on an M grid with M >= 3K/2 - 2 equals the parent-grid product times M/N — the
    engine's small-product-grid lever, checked on the oracle in fp64."""
    g = O.Grid((24, 20, 22), (1.0, 1.0, 1.0))
    b = O.Band(g, (8, 8, 8))
    rng = np.random.default_rng(1)
    a = O.project(rng.standard_normal(g.dims), b)
    c = O.project(rng.standard_normal(g.dims), b)
    gm = O.Grid((10, 10, 10), (2.4, 2.0, 2.2))
    bm = O.Band(gm, (8, 8, 8))
    small = O.project(O.embed(a, bm) * O.embed(c, bm), bm) * (gm.size / g.size)
    assert rel(small, O.star(a, c, b)) < 1e-12


def test_unit_kats():
    """Analytic KATs of the reference (test_spectral.cpp:102-126, test_core.cpp, test_interp.cpp:109-121)."""
    g = O.Grid((16, 12, 10), (1.0, 0.5, 2.0))
    b = O.Band(g, (8, 8, 6))
    x = O.identity_map(g)
    L = [n * h for n, h in zip(g.dims, g.spacing)]
    f = np.sin(2 * np.pi * 2 * x[0] / L[0]) + np.cos(2 * np.pi * 1 * x[1] / L[1])
    c = O.project(f, b)
    assert np.max(np.abs(O.embed(c, b) - f)) < 1e-12  # band contains both modes
    dfx = O.embed(O.band_derivative(c, b, 0), b)
    assert np.max(np.abs(dfx - 2 * np.pi * 2 / L[0] * np.cos(2 * np.pi * 2 * x[0] / L[0]))) < 1e-12
    w = O.trapezoid_weights(5)
    assert abs(w.sum() - 1.0) < 1e-15 and w[0] == w[-1] == 0.1
    # cubic interpolation reproduces node values exactly
    rng = np.random.default_rng(2)
    h = rng.standard_normal(g.dims)
    assert np.max(np.abs(O.warp(h, x, g, "cubic") - h)) < 1e-12


@pytest.mark.parametrize("variant", ["deformation_state_equation", "original", "state_equation"])
def test_model_nonstationary_golden(variant):
    """Nonstationary parameterization: per-node providers, departures per step, per-node
    assembly and trapezoid-weighted inner products (core.hpp:290-316, transport.hpp:120-187,
    variants.hpp:94-103,280-287,364-368)."""
    z = load("model_ns")
    dims = tuple(int(x) for x in z["dims"])
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, tuple(int(x) for x in z["band"]))
    nt = int(z["nt"])
    m = O.Model(b, z["I0"], z["I1"], variant, nt, float(z["sigma2"]), stationary=False)
    v, dv = list(z["v"]), list(z["dv"])
    c = m.forward(v, True)
    assert np.allclose([c.energy, c.energy_reg, c.energy_data, c.cfl], z[f"{variant}_energy"], rtol=1e-12)
    assert rel(np.stack(m.gradient(c)), z[f"{variant}_gradient"]) < 1e-11
    assert rel(np.stack(m.hessvec(c, dv)), z[f"{variant}_hessvec"]) < 1e-11
    r = O.optimize(m, m.zero_velocity(), O.Options(max_iter=3))
    hist = z[f"{variant}_opt_history"]
    assert O.STOP.index(r["stop"]) == int(z[f"{variant}_opt_stop"])
    assert len(r["history"]) == hist.shape[0]
    for q, row in zip(r["history"], hist):
        assert q["pcg_iters"] == int(row[2]) and q["epsilon"] == row[3]
        assert abs(q["energy"] - row[1]) <= 1e-9 * abs(row[1])


def test_evaluation_golden():
    """Evaluation path: warp_nearest, mean_dice, mse_rel, map_jacobian_determinant
    (interp.hpp:213-225, metrics.hpp:40-131) against the reference's own outputs."""
    z = load("evaluation")
    g = O.Grid(tuple(int(x) for x in z["dims"]), tuple(float(x) for x in z["spacing"]))
    x = O.identity_map(g)
    wl = O.warp_nearest(z["source_labels"], x - z["disp"], g)
    assert np.array_equal(wl, z["warped_labels"])
    assert O.mean_dice(wl, z["target_labels"]) == float(z["dice_mean"])
    assert abs(O.mse_rel(z["warped_source"], z["target"], z["source"], g) - float(z["mse_rel"])) < 1e-13
    det = O.map_jacobian_determinant(z["disp"], g)
    assert np.max(np.abs(det - z["det"])) < 1e-12
    assert np.allclose([det.min(), det.max()], z["jac"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("variant", ["deformation_state_equation", "original", "state_equation"])
@pytest.mark.parametrize("tag", ["s", "n"])
def test_model_rk4_golden(variant, tag):
    """RK4 integrator (transport.hpp:234-258, the rk4 branches of variants.hpp:444-547),
    band representation, stationary (s) and nonstationary (n), against the reference."""
    z = load("model_rk4")
    dims = tuple(int(x) for x in z["dims"])
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, tuple(int(x) for x in z["band"]))
    nt = int(z["nt"])
    st = tag == "s"
    m = O.Model(b, z["I0"], z["I1"], variant, nt, float(z["sigma2"]), stationary=st, integrator="rk4")
    v = z["v"][0] if st else list(z["vn"])
    dv = z["dv"][0] if st else list(z["dvn"])
    c = m.forward(v, True)
    assert np.allclose([c.energy, c.energy_reg, c.energy_data, c.cfl], z[f"{variant}_{tag}_energy"], rtol=1e-12)
    gr = m.gradient(c)
    hv = m.hessvec(c, dv)
    gw, hw = z[f"{variant}_{tag}_gradient"], z[f"{variant}_{tag}_hessvec"]
    assert rel(gr if st else np.stack(gr), gw[0] if st else gw) < 1e-11
    assert rel(hv if st else np.stack(hv), hw[0] if st else hw) < 1e-11
    if st:
        r = O.optimize(m, m.zero_velocity(), O.Options(max_iter=3))
        hist = z[f"{variant}_opt_history"]
        assert O.STOP.index(r["stop"]) == int(z[f"{variant}_opt_stop"])
        assert len(r["history"]) == hist.shape[0]
        for q, row in zip(r["history"], hist):
            assert q["pcg_iters"] == int(row[2]) and q["epsilon"] == row[3]
            assert abs(q["energy"] - row[1]) <= 1e-9 * abs(row[1])
        assert rel(r["v"], z[f"{variant}_opt_v"][0]) < 1e-8
    if st and variant == "deformation_state_equation":
        fwd, inv = O.compute_maps(m, v)
        assert rel(fwd, z["maps_fwd"]) < 1e-12 and rel(inv, z["maps_inv"]) < 1e-12
