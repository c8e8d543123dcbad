"""Run the REFERENCE (oracle/_ref: the unmodified headers compiled by oracle/Makefile)
offline on the full-size BASELINE configs that tools/ref_config2_golden.py does not
cover, and store golden fixtures under tests/golden/.  Hours of CPU; run here:

    python tools/ref_fullsize_golden.py config3 original [threads]
    python tools/ref_fullsize_golden.py config3 state_equation [threads]
    python tools/ref_fullsize_golden.py config4 [threads]

config3 <variant>: the config-2 pair (180x210x180 brain-like, seed 2006, K = 32,
    nt = 10, sigma2 = 0.01, OptimizeOptions defaults, max_iter 10, pcg cap 5) registered
    with `variant` (BASELINE.json configs[2]; variants.hpp:34, 373-422, 444-527): GN/PCG
    history, final band velocity, compute_maps Jacobian ranges (metrics.hpp:24-65).
config4: the config-2 generator at 256^3, K = 64, nt = 20 (BASELINE.json configs[3]),
    deformation-state.  A full registration is out of reach on the host, so the fixture
    holds one per-op evaluation on a fixed seeded velocity v (the reference's own
    random_band_field generator, synth.hpp): forward with adjoint (energies, cfl),
    gradient, hessvec(dv), and the transported u(1) node (variants.hpp:262-344).
    Gradient / hessvec / u(1) are stored as complex64 (rel. rounding 6e-8, far below the
    1e-4 contract) to keep the fixture small.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2006_06823_b200 import phantoms  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

# config-4 fixed inputs (also read by tests/test_gpu_fullsize.py through the fixture)
C4_V_SEED, C4_V_AMP, C4_V_K0 = 4004, 3.0, 3.0
C4_DV_SEED, C4_DV_AMP, C4_DV_K0 = 4005, 0.5, 4.0


def run_config3(variant, threads):
    ref.set_threads(threads)
    dims, band, nt, sigma2 = (180, 210, 180), (32, 32, 32), 10, 0.01
    I0, I1 = phantoms.brain_pair(dims, seed=2006)
    I0 = I0.astype(np.float32).astype(np.float64)
    I1 = I1.astype(np.float32).astype(np.float64)
    m = ref.RefModel(I0, I1, dims, (1.0, 1.0, 1.0), band, variant, nt, sigma2)
    t0 = time.time()
    r = m.optimize(None, max_iter=10, pcg_max_iter=5)
    wall = time.time() - t0
    hist = np.array([[q.iter, q.energy, q.energy_data, q.energy_reg, q.mse_rel, q.rel_grad, q.pcg_iters,
                      q.pcg_fallback, q.epsilon, q.cfl] for q in r["history"]])
    fwd, inv, jac = m.maps(r["v"])
    np.savez_compressed(os.path.join(GOLD, f"config3_{variant}_ref.npz"), dims=np.array(dims),
                        band=np.array(band), nt=nt, sigma2=sigma2, variant=variant, history=hist,
                        v=r["v"], stop=ref.STOP_REASONS.index(r["stop"]), iterations=r["iterations"],
                        jac=jac, wall_s=wall, threads=threads)
    print("done", variant, r["stop"], r["iterations"], wall, hist[:, [0, 1, 6, 8]], flush=True)


def run_config4(threads):
    ref.set_threads(threads)
    dims, band, nt, sigma2 = (256, 256, 256), (64, 64, 64), 20, 0.01
    sp = (1.0, 1.0, 1.0)
    I0, I1 = phantoms.brain_pair(dims, seed=2006)
    I0 = I0.astype(np.float32).astype(np.float64)
    I1 = I1.astype(np.float32).astype(np.float64)
    v = ref.random_band_field(dims, sp, band, C4_V_SEED, C4_V_AMP, C4_V_K0)[None]
    dv = ref.random_band_field(dims, sp, band, C4_DV_SEED, C4_DV_AMP, C4_DV_K0)[None]
    m = ref.RefModel(I0, I1, dims, sp, band, "deformation_state_equation", nt, sigma2)
    t = {}
    t0 = time.time()
    e = m.forward(v, True)
    t["forward"] = time.time() - t0
    print("forward", e, t, flush=True)
    u = m.series("u")
    t0 = time.time()
    g = m.gradient()
    t["gradient"] = time.time() - t0
    print("gradient", t, flush=True)
    t0 = time.time()
    hv = m.hessvec(dv)
    t["hessvec"] = time.time() - t0
    print("hessvec", t, flush=True)
    m1, res = m.fields()
    np.savez_compressed(os.path.join(GOLD, "config4_ops_ref.npz"), dims=np.array(dims),
                        band=np.array(band), nt=nt, sigma2=sigma2,
                        v_seed=C4_V_SEED, v_amp=C4_V_AMP, v_k0=C4_V_K0,
                        dv_seed=C4_DV_SEED, dv_amp=C4_DV_AMP, dv_k0=C4_DV_K0,
                        v=v.astype(np.complex128), dv=dv.astype(np.complex128),
                        energy=np.array([e["energy"], e["energy_reg"], e["energy_data"], e["cfl"]]),
                        u_final=u[-1].astype(np.complex64), gradient=g.astype(np.complex64),
                        hessvec=hv.astype(np.complex64),
                        m1_sum=float(m1.sum()), m1_sumsq=float((m1 * m1).sum()),
                        res_sumsq=float((res * res).sum()),
                        seconds=np.array([t["forward"], t["gradient"], t["hessvec"]]), threads=threads)
    print("done config4", e, t, flush=True)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "config3":
        run_config3(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 8)
    elif mode == "config4":
        run_config4(int(sys.argv[2]) if len(sys.argv) > 2 else 8)
    else:
        raise SystemExit(__doc__)
