"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers (/root/reference/proj/include, compiled by
oracle/Makefile into oracle/_ref/libref_lddmm.so with our FFTW3-API shim) on
small seeded inputs and stores inputs + outputs as compressed .npz.  The
fixtures pin the numpy restatement (oracle/lddmm_np.py) in tests/test_oracle.py
and are the CPU-side golden vectors for the GPU parity tests.  The reference
has no stored golden vectors of its own; every input here comes
from the reference's own deterministic generators (synth.hpp) where one exists.

    python tests/golden/make_golden.py      # needs /root/reference (this container)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

DIMS = (16, 12, 14)
H = (1.0, 0.8, 1.25)
BAND = (8, 8, 6)


def spectral():
    g = dict(dims=np.array(DIMS), spacing=np.array(H), band=np.array(BAND))
    u = ref.random_band_field(DIMS, H, BAND, 11, 1.0, 2.0)
    w = ref.random_band_field(DIMS, H, BAND, 12, 1.0, 2.0)
    s = ref.random_band_field(DIMS, H, BAND, 13, 1.0, 2.0)[:1]
    t = ref.random_band_field(DIMS, H, BAND, 14, 1.0, 2.0)[:1]
    f = ref.random_smooth_field(DIMS, H, 15, 1.0, 3.0)
    g.update(u=u, w=w, s=s, t=t, f=f,
             embed_u=ref.embed(u, DIMS, H, BAND), project_f=ref.project(f, DIMS, H, BAND),
             star_ss=ref.band_op("star_ss", s, t, DIMS, H, BAND),
             star_sv=ref.band_op("star_sv", s, u, DIMS, H, BAND),
             star_dot=ref.band_op("star_dot", u, w, DIMS, H, BAND),
             jac=ref.band_op("jac", u, w, DIMS, H, BAND), jacT=ref.band_op("jacT", u, w, DIMS, H, BAND),
             grad=ref.band_op("grad", s, None, DIMS, H, BAND), div=ref.band_op("div", u, None, DIMS, H, BAND),
             sobolev=ref.band_op("sobolev", u, None, DIMS, H, BAND, 0.0025, 2),
             sobolev_inv=ref.band_op("sobolev_inv", u, None, DIMS, H, BAND, 0.0025, 2),
             inner_uw=ref.band_inner(u, w, DIMS, H, BAND),
             sgrad_f0=ref.spectral_gradient(f[0], DIMS, H))
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), **g)


def interp():
    f = ref.random_smooth_field(DIMS, H, 21, 1.0, 4.0)[0]
    disp = ref.random_smooth_field(DIMS, H, 22, 2.5, 2.0)
    x = np.stack(np.meshgrid(*[np.arange(n) * h for n, h in zip(DIMS, H)], indexing="ij"))
    pts = x - disp
    np.savez_compressed(os.path.join(HERE, "interp.npz"), dims=np.array(DIMS), spacing=np.array(H), f=f, pts=pts,
                        coef=ref.spline_coefficients(f, DIMS, H), cubic=ref.warp(f, pts, DIMS, H, "cubic"),
                        linear=ref.warp(f, pts, DIMS, H, "linear"), nearest=ref.warp(f, pts, DIMS, H, "nearest"))


def transport():
    nt = 4
    v = ref.random_band_field(DIMS, H, BAND, 31, 2.0, 2.0)
    q = ref.random_band_field(DIMS, H, BAND, 32, 1.0, 2.0)
    Xf = ref.departure(v, DIMS, H, BAND, nt, "forward")
    Xb = ref.departure(v, DIMS, H, BAND, nt, "backward")
    np.savez_compressed(os.path.join(HERE, "transport.npz"), dims=np.array(DIMS), spacing=np.array(H),
                        band=np.array(BAND), nt=nt, v=v, q=q, Xf=Xf, Xb=Xb,
                        adv_f=ref.advect_band(q, Xf, DIMS, H, BAND), adv_b=ref.advect_band(q, Xb, DIMS, H, BAND),
                        cfl=ref.cfl(v, DIMS, H, BAND, nt))


def model():
    dims, h, band, nt = (16, 12, 14), (1.0, 1.0, 1.0), (8, 8, 6), 3
    I0 = ref.random_smooth_image(dims, h, 41, 1.0)
    I1 = ref.random_smooth_image(dims, h, 42, 1.0)
    v = ref.random_band_field(dims, h, band, 43, 1.2, 2.0)[None]
    dv = ref.random_band_field(dims, h, band, 44, 1.0, 2.0)[None]
    out = dict(dims=np.array(dims), band=np.array(band), nt=nt, sigma2=0.5, I0=I0, I1=I1, v=v, dv=dv)
    for var in ("deformation_state_equation", "original", "state_equation"):
        m = ref.RefModel(I0, I1, dims, h, band, var, nt, 0.5)
        e = m.forward(v, True)
        m1, res = m.fields()
        out[f"{var}_energy"] = np.array([e["energy"], e["energy_reg"], e["energy_data"], e["cfl"]])
        out[f"{var}_m1"] = m1
        out[f"{var}_gradient"] = m.gradient()
        out[f"{var}_hessvec"] = m.hessvec(dv)
        out[f"{var}_precondition"] = m.precondition(dv)
        if var != "original":
            out[f"{var}_u"] = m.series("u")
        if var == "deformation_state_equation":
            out[f"{var}_rho"] = m.series("rho")
            fwd, inv, jac = m.maps(v)
            out["maps_fwd"], out["maps_inv"], out["maps_jac"] = fwd, inv, jac
    np.savez_compressed(os.path.join(HERE, "model.npz"), **out)


def optimize():
    """test_optimizer.cpp:117-143 style: def-state SL band descent on a smooth 3-D pair."""
    dims, h, band, nt = (16, 16, 16), (1.0, 1.0, 1.0), (8, 8, 8), 4
    I0 = ref.random_smooth_image(dims, h, 51, 1.0)
    I1 = ref.random_smooth_image(dims, h, 52, 1.0)
    out = dict(dims=np.array(dims), band=np.array(band), nt=nt, sigma2=0.05, I0=I0, I1=I1)
    for tag, kw in (("parity", dict(max_iter=6)),
                    ("fixed", dict(max_iter=3, grad_tol=0.0, energy_tol=0.0, step_tol=0.0, pcg_tol=0.0))):
        m = ref.RefModel(I0, I1, dims, h, band, "deformation_state_equation", nt, 0.05)
        r = m.optimize(None, **kw)
        hist = np.array([[q.iter, q.energy, q.energy_data, q.energy_reg, q.mse_rel, q.rel_grad, q.pcg_iters,
                          q.pcg_fallback, q.epsilon, q.cfl] for q in r["history"]])
        out[f"{tag}_history"] = hist
        out[f"{tag}_v"] = r["v"]
        out[f"{tag}_stop"] = ref.STOP_REASONS.index(r["stop"])
        out[f"{tag}_iterations"] = r["iterations"]
    np.savez_compressed(os.path.join(HERE, "optimize.npz"), **out)


def model_nonstationary():
    """Nonstationary parameterization (core.hpp:290-316; transport.hpp:120-131,176-187;
    variants.hpp:364-368): forward/gradient/hessvec of the three variants + a short optimize."""
    dims, h, band, nt = (16, 12, 14), (1.0, 1.0, 1.0), (8, 8, 6), 3
    I0 = ref.random_smooth_image(dims, h, 61, 1.0)
    I1 = ref.random_smooth_image(dims, h, 62, 1.0)
    v = np.stack([ref.random_band_field(dims, h, band, 63 + i, 1.0, 2.0) for i in range(nt + 1)])
    dv = np.stack([ref.random_band_field(dims, h, band, 73 + i, 1.0, 2.0) for i in range(nt + 1)])
    out = dict(dims=np.array(dims), band=np.array(band), nt=nt, sigma2=0.5, I0=I0, I1=I1, v=v, dv=dv)
    for var in ("deformation_state_equation", "original", "state_equation"):
        m = ref.RefModel(I0, I1, dims, h, band, var, nt, 0.5, param="nonstationary")
        e = m.forward(v, True)
        out[f"{var}_energy"] = np.array([e["energy"], e["energy_reg"], e["energy_data"], e["cfl"]])
        out[f"{var}_gradient"] = m.gradient()
        out[f"{var}_hessvec"] = m.hessvec(dv)
        r = m.optimize(None, max_iter=3)
        out[f"{var}_opt_history"] = np.array([[q.iter, q.energy, q.pcg_iters, q.epsilon] for q in r["history"]])
        out[f"{var}_opt_stop"] = ref.STOP_REASONS.index(r["stop"])
    np.savez_compressed(os.path.join(HERE, "model_ns.npz"), **out)


def synth():
    """blob_pair / two_disc_case (synth.hpp:182-259) in 2-D and 3-D: fixtures for the CLI's
    `synth` subcommand (lddmm_cli.cpp:264-296)."""
    out = {}
    for d in (2, 3):
        dims, h = (16,) * d, (1.0,) * d
        s, t = ref.blob_pair(dims, h, 3)
        out[f"blobs{d}_source"], out[f"blobs{d}_target"] = s, t
        s, t, sl, tl = ref.two_disc_case(dims, h, 5)
        out[f"discs{d}_source"], out[f"discs{d}_target"] = s, t
        out[f"discs{d}_source_labels"], out[f"discs{d}_target_labels"] = sl, tl
    np.savez_compressed(os.path.join(HERE, "synth.npz"), **out)


def evaluation():
    """Evaluation path (metrics.hpp:40-131, interp.hpp:213-225): nearest-warped labels, Dice,
    mse_rel and the Jacobian range of a displacement, on the 3-D disc case."""
    dims, h = (16, 12, 14), (1.0, 1.0, 1.0)
    s, t, sl, tl = ref.two_disc_case(dims, h, 7)
    disp = ref.random_smooth_field(dims, h, 81, 1.0, 2.0)
    x = np.stack(np.meshgrid(*[np.arange(n) * hh for n, hh in zip(dims, h)], indexing="ij"))
    wl = ref.warp(sl, x - disp, dims, h, "nearest")[0]
    ws = ref.warp(s, x - disp, dims, h, "cubic")[0]
    e = ref.evaluate(dims, h, warped=ws, target=t, source=s, warped_labels=wl, target_labels=tl, disp=disp)
    np.savez_compressed(os.path.join(HERE, "evaluation.npz"), dims=np.array(dims), spacing=np.array(h), source=s,
                        target=t, source_labels=sl, target_labels=tl, disp=disp, warped_labels=wl,
                        warped_source=ws, mse_rel=e["mse_rel"], dice_mean=e["dice_mean"], jac=e["jac"],
                        det=e["det"])


def cli_register():
    """What `lddmm register` must reproduce on the 3-D disc case (cli_smoke.sh analog):
    synth --kind discs --d 3 --n 32 --seed 5, then register --variant
    deformation_state_equation --band 16 --sigma2 0.01 --max-iter 4 with labels
    (lddmm_cli.cpp:101-232).  Inputs are the float32 payloads the CLI reads."""
    dims, h, band, nt = (32, 32, 32), (1.0, 1.0, 1.0), (16, 16, 16), 5
    s, t, sl, tl = (x.astype(np.float32).astype(np.float64) for x in ref.two_disc_case(dims, h, 5))
    m = ref.RefModel(s, t, dims, h, band, "deformation_state_equation", nt, 0.01)
    r = m.optimize(None, max_iter=4, pcg_max_iter=5)
    hist = np.array([[q.iter, q.energy, q.energy_data, q.energy_reg, q.mse_rel, q.rel_grad, q.pcg_iters,
                      q.pcg_fallback, q.epsilon, q.cfl] for q in r["history"]])
    fwd, inv, jac = m.maps(r["v"])
    x = np.stack(np.meshgrid(*[np.arange(n) * hh for n, hh in zip(dims, h)], indexing="ij"))
    wl = ref.warp(sl, x - fwd, dims, h, "nearest")[0]
    e = ref.evaluate(dims, h, warped_labels=wl, target_labels=tl)
    np.savez_compressed(os.path.join(HERE, "cli_register.npz"), history=hist, stop=ref.STOP_REASONS.index(r["stop"]),
                        iterations=r["iterations"], jac=jac, dice_mean=e["dice_mean"], v=r["v"])


def model_rk4():
    """RK4 integrator (transport.hpp:234-258; variants.hpp:444-547 rk4 branches), band
    representation, all three variants, stationary and nonstationary (§8f row 4)."""
    dims, h, band, nt = (16, 12, 14), (1.0, 1.0, 1.0), (8, 8, 6), 4
    I0 = ref.random_smooth_image(dims, h, 91, 1.0)
    I1 = ref.random_smooth_image(dims, h, 92, 1.0)
    v = ref.random_band_field(dims, h, band, 93, 1.0, 2.0)[None]
    dv = ref.random_band_field(dims, h, band, 94, 1.0, 2.0)[None]
    vn = np.stack([ref.random_band_field(dims, h, band, 95 + i, 1.0, 2.0) for i in range(nt + 1)])
    dvn = np.stack([ref.random_band_field(dims, h, band, 105 + i, 1.0, 2.0) for i in range(nt + 1)])
    out = dict(dims=np.array(dims), band=np.array(band), nt=nt, sigma2=0.5, I0=I0, I1=I1, v=v, dv=dv, vn=vn, dvn=dvn)
    for var in ("deformation_state_equation", "original", "state_equation"):
        for tag, param, vv, dd in (("s", "stationary", v, dv), ("n", "nonstationary", vn, dvn)):
            m = ref.RefModel(I0, I1, dims, h, band, var, nt, 0.5, param=param, integrator="rk4")
            e = m.forward(vv, True)
            out[f"{var}_{tag}_energy"] = np.array([e["energy"], e["energy_reg"], e["energy_data"], e["cfl"]])
            out[f"{var}_{tag}_gradient"] = m.gradient()
            out[f"{var}_{tag}_hessvec"] = m.hessvec(dd)
        m = ref.RefModel(I0, I1, dims, h, band, var, nt, 0.5, integrator="rk4")
        r = m.optimize(None, max_iter=3)
        out[f"{var}_opt_history"] = np.array([[q.iter, q.energy, q.pcg_iters, q.epsilon] for q in r["history"]])
        out[f"{var}_opt_stop"] = ref.STOP_REASONS.index(r["stop"])
        out[f"{var}_opt_v"] = r["v"]
    m = ref.RefModel(I0, I1, dims, h, band, "deformation_state_equation", nt, 0.5, integrator="rk4")
    fwd, inv, jac = m.maps(v)
    out["maps_fwd"], out["maps_inv"], out["maps_jac"] = fwd, inv, jac
    np.savez_compressed(os.path.join(HERE, "model_rk4.npz"), **out)


def gate8():
    """Acceptance gate 8 analog in 3-D (acceptance.cpp:307-343): two-disc cases at 32^3,
    K = 16, SL nt = 5, sigma2 = 0.05, max_iter 30, grad_tol 1e-3; mean Dice of the
    nearest-warped source labels per variant, from the reference itself."""
    n, h = 32, (1.0, 1.0, 1.0)
    dims = (n, n, n)
    out = {}
    x = np.stack(np.meshgrid(*[np.arange(k) * 1.0 for k in dims], indexing="ij"))
    for seed in (1, 2):
        s, t, sl, tl = (a.astype(np.float32) for a in ref.two_disc_case(dims, h, seed))
        out[f"s{seed}_inputs"] = np.stack([s, t, sl, tl])
        s, t, sl, tl = (a.astype(np.float64) for a in (s, t, sl, tl))
        out[f"s{seed}_initial"] = ref.evaluate(dims, h, warped_labels=sl, target_labels=tl)["dice_mean"]
        for v in ("original", "state_equation", "deformation_state_equation"):
            m = ref.RefModel(s, t, dims, h, (16, 16, 16), v, 5, 0.05)
            r = m.optimize(None, max_iter=30, grad_tol=1e-3)
            fwd, _, _ = m.maps(r["v"])
            wl = ref.warp(sl, x - fwd, dims, h, "nearest")[0]
            out[f"s{seed}_{v}_dice"] = ref.evaluate(dims, h, warped_labels=wl, target_labels=tl)["dice_mean"]
            out[f"s{seed}_{v}_iterations"] = r["iterations"]
            out[f"s{seed}_{v}_stop"] = ref.STOP_REASONS.index(r["stop"])
    np.savez_compressed(os.path.join(HERE, "gate8.npz"), **out)


if __name__ == "__main__":
    if not ref.available():
        sys.exit("build oracle/_ref first: make -C oracle ref")
    spectral()
    interp()
    transport()
    model()
    optimize()
    model_nonstationary()
    synth()
    evaluation()
    cli_register()
    model_rk4()
    gate8()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
