"""3-D, band-representation analogs of the reference's acceptance gates
(tests/acceptance.cpp) run on the B200 engine.  One PASS/FAIL line per gate, with
the measured quantity and the gate it is held to, like the reference.

  4. SL nt=5 and RK4 nt=25 agree in final relative MSE over 10 blob cases
     (acceptance.cpp:197-228): mean |gap| <= 0.05
  5. SL per-iteration cost at most half of RK4 (acceptance.cpp:230-247)
  6. inverse-map Jacobian determinant positive on converged runs (acceptance.cpp:249-263)
  8. two-disc label overlap: Dice gain >= 0.15 and deformation-state ordering
     (acceptance.cpp:307-343; the evaluation path: warp_nearest + mean_dice on the device)

The reference runs them in 2-D at 64^2, K = 16; the engine is 3-D, so the cases are
the same generators (blob_pair / two_disc_case, via `lddmm synth`) at 32^3, K = 16.
In 3-D the reference itself ranks deformation-state below the other variants on the
two-disc cases (tests/golden/gate8.npz, checked case by case in
tests/test_gpu_eval.py::test_two_disc_dice_matches_reference), so gate 8's ordering
clause is a 2-D property; its Dice-gain clause holds.
Gates 1-3, 7 and 9 exercise the spatial representation or 2-D operator oracles and
are covered by the parity tests instead (tests/test_gpu_kat.py, tests/test_oracle.py).

    python tools/acceptance_gpu.py [n]      # n = grid points per axis (default 32)
"""
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_06823_b200 import lddmm as L  # noqa: E402

CLI = os.path.join(ROOT, "paper_2006_06823_b200", "lddmm")


def read(base):
    with open(base + ".json") as f:
        side = json.load(f)
    return np.fromfile(base + ".raw", dtype="<f4").astype(np.float64).reshape(side["dims"])


def synth(kind, n, seed, tmp):
    out = os.path.join(tmp, f"{kind}{seed}")
    subprocess.run([CLI, "synth", "--kind", kind, "--d", "3", "--n", str(n), "--seed", str(seed), "--out", out],
                   check=True, capture_output=True)
    names = ["source", "target"] + (["source_labels", "target_labels"] if kind == "discs" else [])
    return [read(os.path.join(out, x)) for x in names]


def report(num, ok, name, detail):
    print(f"[{'PASS' if ok else 'FAIL'}] {num}. {name}: {detail}", flush=True)
    return ok


def run_blob(band, s, t, integ, nt):
    m = L.Model(band, s, t, "deformation_state_equation", nt, 0.01, integrator=integ)
    res = L.optimize(m, None, L.OptimizeOptions(max_iter=15))
    iter_ms = [h.wall_ms for h in res.history if h.iter > 0]
    _, _, jac = L.compute_maps(m, res.v)
    return dict(converged=res.converged, mse=res.history[-1].mse_rel, iter_ms=iter_ms, min_det=jac[2])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    band = L.BandSpec(L.GridSpec((n, n, n)), (16, 16, 16))
    passed = 0
    with tempfile.TemporaryDirectory() as tmp:
        t0 = time.time()
        sl, rk = [], []
        for seed in range(1, 11):
            s, t = synth("blobs", n, seed, tmp)
            sl.append(run_blob(band, s, t, "sl", 5))
            rk.append(run_blob(band, s, t, "rk4", 25))
        secs = time.time() - t0
        gap = float(np.mean([abs(a["mse"] - b["mse"]) for a, b in zip(sl, rk)]))
        passed += report(4, gap <= 0.05 and secs <= 300.0, "sl nt=5 and rk4 nt=25 agree in final relative MSE",
                         f"mean |mse_rel gap| {gap:.4f} over 10 cases (sl {np.mean([a['mse'] for a in sl]):.4f}, "
                         f"rk4 {np.mean([b['mse'] for b in rk]):.4f}), tol 0.05; {secs:.1f} s of 300 s")
        sl_per = float(np.sum([sum(a["iter_ms"]) for a in sl]) / max(1, sum(len(a["iter_ms"]) for a in sl)))
        rk_per = float(np.sum([sum(b["iter_ms"]) for b in rk]) / max(1, sum(len(b["iter_ms"]) for b in rk)))
        passed += report(5, sl_per <= 0.5 * rk_per, "semi-Lagrangian per-iteration cost at most half of RK4",
                         f"per-iteration wall: sl nt=5 {sl_per:.2f} ms, rk4 nt=25 {rk_per:.2f} ms, ratio "
                         f"{sl_per / rk_per:.3f} (gate <= 0.5)")
        conv = [r for r in sl + rk if r["converged"]]
        worst = min((r["min_det"] for r in conv), default=float("inf"))
        passed += report(6, len(conv) >= 1 and worst > 0.0, "inverse-map Jacobian determinant positive on "
                         "converged runs", f"{len(conv)} of {len(sl) + len(rk)} runs converged, min inverse-map "
                         f"det {worst:.3f} (gate > 0)")
        variants = ["original", "state_equation", "deformation_state_equation"]
        dice = {v: 0.0 for v in variants}
        initial = 0.0
        ctx = L.Context(band)
        for seed in range(1, 11):
            s, t, sl_lab, tl_lab = synth("discs", n, seed, tmp)
            initial += L.mean_dice(ctx, sl_lab, tl_lab) / 10.0
            for v in variants:
                m = L.Model(band, s, t, v, 5, 0.05)
                res = L.optimize(m, None, L.OptimizeOptions(max_iter=30, grad_tol=1e-3))
                fwd, _, _ = L.compute_maps(m, res.v)
                warped = L.warp(ctx, sl_lab, fwd, kind="nearest")
                dice[v] += L.mean_dice(ctx, warped, tl_lab) / 10.0
        gain = dice["deformation_state_equation"] - initial
        ordered = all(dice["deformation_state_equation"] >= dice[v] for v in variants[:2])
        passed += report(8, gain >= 0.15 and ordered, "two-disc label overlap: Dice gain and variant ordering",
                         f"mean Dice: initial {initial:.4f}, original {dice['original']:.4f}, state "
                         f"{dice['state_equation']:.4f}, deformation {dice['deformation_state_equation']:.4f}; "
                         f"gain {gain:.4f} (gate >= 0.15), ordering {'holds' if ordered else 'violated'}")
    print(f"{passed} of 4 checks passed")


if __name__ == "__main__":
    main()
