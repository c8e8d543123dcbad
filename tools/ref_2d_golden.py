"""The reference's own 2-D acceptance-gate workloads (proj/tests/acceptance.cpp), run by
the unmodified reference (oracle/_ref) and stored as tests/golden/accept2d_ref.npz for
the device replay (tests/test_gpu_2d.py, tools/acceptance_gpu.py --2d):

  gates 4-6 (run_blob, acceptance.cpp:173-195): blob pairs seeds 1..10 on 64^2, band 16,
    deformation-state, sigma2 0.01, max_iter 15; SL nt = 5 and RK4 nt = 25: final mse_rel,
    converged, GN iterations, min inverse-map Jacobian determinant; full GN history and
    velocity for seeds 1, 2 (SL)
  gate 8 (check_label_overlap, acceptance.cpp:308-345): two-disc cases seeds 1..10, the
    three variants, SL nt = 5, sigma2 0.05, max_iter 30, grad_tol 1e-3: mean Dice of the
    nearest-neighbour-warped source labels

    python tools/ref_2d_golden.py [threads]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

VARIANTS = ["original", "state_equation", "deformation_state_equation"]


def main(threads=2):
    ref.set_threads(threads)
    dims, sp, band = (64, 64), (1.0, 1.0), (16, 16)
    x = np.stack(np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij"))
    out = {}
    t0 = time.time()
    blob = []  # seed, integrator, mse, converged, iters, min_det, stop
    for seed in range(1, 11):
        s, t = ref.blob_pair(dims, sp, seed)
        for integ, nt in (("sl", 5), ("rk4", 25)):
            m = ref.RefModel(s, t, dims, sp, band, "deformation_state_equation", nt, 0.01, integrator=integ)
            r = m.optimize(None, max_iter=15, pcg_max_iter=5)
            fwd, inv, jac = m.maps(r["v"])
            blob.append([seed, 0 if integ == "sl" else 1, r["history"][-1].mse_rel, int(r["converged"]),
                         r["iterations"], jac[2], ref.STOP_REASONS.index(r["stop"])])
            if integ == "sl" and seed <= 2:
                out[f"blob{seed}_history"] = np.array(
                    [[q.iter, q.energy, q.energy_data, q.energy_reg, q.mse_rel, q.rel_grad, q.pcg_iters,
                      q.pcg_fallback, q.epsilon, q.cfl] for q in r["history"]])
                out[f"blob{seed}_v"] = r["v"]
                out[f"blob{seed}_jac"] = jac
            print("blob", seed, integ, blob[-1], flush=True)
    out["blob"] = np.array(blob)
    gate8 = []  # seed, variant, dice, initial dice, mse, iterations, stop
    for seed in range(1, 11):
        src, tgt, sl, tl = ref.two_disc_case(dims, sp, seed)
        init = ref.evaluate(dims, sp, warped_labels=sl, target_labels=tl)["dice_mean"]
        for vi, variant in enumerate(VARIANTS):
            m = ref.RefModel(src, tgt, dims, sp, band, variant, 5, 0.05)
            r = m.optimize(None, max_iter=30, pcg_max_iter=5, grad_tol=1e-3)
            fwd, inv, jac = m.maps(r["v"])
            warped = ref.warp(sl, np.ascontiguousarray(x - fwd), dims, sp, kind="nearest")
            dice = ref.evaluate(dims, sp, warped_labels=warped, target_labels=tl)["dice_mean"]
            gate8.append([seed, vi, dice, init, r["history"][-1].mse_rel, r["iterations"],
                          ref.STOP_REASONS.index(r["stop"])])
            print("gate8", seed, variant, gate8[-1], flush=True)
    out["gate8"] = np.array(gate8)
    out["wall_s"] = time.time() - t0
    out["threads"] = threads
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "accept2d_ref.npz"), **out)
    print("done", out["wall_s"], flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
