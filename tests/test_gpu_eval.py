"""GPU parity of the evaluation path and the `lddmm` CLI.

- warp_nearest (interp.hpp:213-225): bit-exact labels vs the reference's output;
- map_jacobian_determinant + value_range (metrics.hpp:40-79) of a grid displacement:
  full-grid spectral derivatives in fp64 on the device, |det - ref| <= 1e-5;
- mean_dice (metrics.hpp:92-131): exact integer counts, equal to the reference's value;
- `lddmm register` / `lddmm evaluate` end to end (lddmm_cli.cpp:101-262, cli_smoke.sh):
  every artifact written, GN/PCG history identical to the reference's run on the same
  float32 inputs (tests/golden/cli_register.npz), energies within 1e-5 relative,
  Jacobian ranges and Dice within the tolerances of DESIGN.md.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import lddmm_np as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
CLI = os.path.join(ROOT, "paper_2006_06823_b200", "lddmm")


def ctx_for(dims, h=(1.0, 1.0, 1.0)):
    from paper_2006_06823_b200 import lddmm as L
    return L.Context(L.BandSpec(L.GridSpec(dims, h), (4, 4, 4)))


def test_evaluation_primitives(cuda):
    from paper_2006_06823_b200 import lddmm as L
    z = np.load(os.path.join(GOLD, "evaluation.npz"))
    dims = tuple(int(x) for x in z["dims"])
    ctx = ctx_for(dims)
    disp = z["disp"].astype(np.float32).astype(np.float64)
    wl = L.warp(ctx, z["source_labels"], disp, kind="nearest")
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    assert np.array_equal(wl, O.warp_nearest(z["source_labels"], O.identity_map(g) - disp, g))
    assert np.array_equal(wl, z["warped_labels"])
    assert L.mean_dice(ctx, wl, z["target_labels"]) == float(z["dice_mean"])
    lo, hi, det = L.jacobian(ctx, z["disp"], want_field=True)
    assert np.max(np.abs(det - z["det"])) < 1e-5
    assert abs(lo - z["jac"][0]) < 1e-5 and abs(hi - z["jac"][1]) < 1e-5
    ws = L.warp(ctx, z["source"], z["disp"], kind="cubic")
    assert np.max(np.abs(ws - z["warped_source"])) < 1e-5
    assert abs(L.mse_rel(ws, z["target"], z["source"]) - float(z["mse_rel"])) < 1e-5


def test_dice_edge_cases(cuda):
    """empty inventory -> dice of label 1 (1.0 when both empty); disjoint labels -> 0;
    many labels (> one 64-label pass)."""
    from paper_2006_06823_b200 import lddmm as L
    dims = (8, 8, 8)
    ctx = ctx_for(dims)
    zero = np.zeros(dims)
    assert L.mean_dice(ctx, zero, zero) == 1.0
    a = zero.copy()
    a[0, 0, 0] = 1.0
    assert L.mean_dice(ctx, a, zero) == O.mean_dice(a, zero) == 0.0
    rng = np.random.default_rng(0)
    t = rng.integers(0, 90, size=dims).astype(np.float64)
    w = np.where(rng.random(dims) < 0.7, t, rng.integers(0, 90, size=dims)).astype(np.float64)
    assert L.mean_dice(ctx, w, t) == O.mean_dice(w, t)
    neg = -t - 0.5  # non-integer, negative labels
    assert L.mean_dice(ctx, -w - 0.5, neg) == O.mean_dice(-w - 0.5, neg)


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=900)


def read_field(base):
    with open(base + ".json") as f:
        side = json.load(f)
    data = np.fromfile(base + ".raw", dtype="<f4")
    shape = tuple(side["dims"])
    if side["kind"] == "vector":
        shape = (side["components"],) + shape
    return side, data.reshape(shape)


def test_cli_register_matches_reference(cuda, tmp_path):
    z = np.load(os.path.join(GOLD, "cli_register.npz"))
    r = run("synth", "--kind", "discs", "--d", "3", "--n", "32", "--seed", "5", "--out", str(tmp_path / "d"))
    assert r.returncode == 0, r.stderr
    d = tmp_path / "d"
    out = tmp_path / "reg"
    r = run("register", "--source", str(d / "source.raw"), "--target", str(d / "target.raw"),
            "--source-labels", str(d / "source_labels.raw"), "--target-labels", str(d / "target_labels.raw"),
            "--out", str(out), "--variant", "deformation_state_equation", "--integrator", "sl", "--repr", "band",
            "--band", "16", "--sigma2", "0.01", "--max-iter", "4")
    assert r.returncode == 0, r.stderr
    assert "registration summary" in r.stdout
    for f in ("report.json", "convergence.csv", "summary.txt", "displacement_forward.raw",
              "displacement_forward.json", "displacement_inverse.raw", "warped_source.raw", "velocity.raw",
              "warped_labels.raw"):
        assert (out / f).exists(), f
    with open(out / "report.json") as f:
        rep = json.load(f)
    hist = z["history"]
    from paper_2006_06823_b200.lddmm import STOP_REASONS
    assert rep["stop_reason"] == STOP_REASONS[int(z["stop"])]
    assert rep["iterations"] == int(z["iterations"])
    assert rep["variant"] == "deformation_state_equation" and rep["band"] == [16, 16, 16] and rep["nt"] == 5
    assert abs(rep["final_energy"] - hist[-1, 1]) <= 1e-5 * abs(hist[-1, 1])
    assert abs(rep["mse_rel_final"] - hist[-1, 4]) <= 1e-5
    assert np.allclose([rep["jacobian_forward"]["min"], rep["jacobian_forward"]["max"],
                        rep["jacobian_inverse"]["min"], rep["jacobian_inverse"]["max"]], z["jac"],
                       rtol=1e-3, atol=1e-3)
    assert abs(rep["dice_mean"] - float(z["dice_mean"])) < 2e-3
    rows = np.loadtxt(out / "convergence.csv", delimiter=",", skiprows=1, ndmin=2)
    assert rows.shape[0] == hist.shape[0]
    assert np.array_equal(rows[:, 4], hist[:, 6]) and np.array_equal(rows[:, 5], hist[:, 8])
    assert np.allclose(rows[:, 1], hist[:, 1], rtol=1e-5, atol=0)
    side, fwd = read_field(str(out / "displacement_forward"))
    assert side["kind"] == "vector" and side["components"] == 3 and fwd.shape == (3, 32, 32, 32)
    side, wl = read_field(str(out / "warped_labels"))
    assert side["kind"] == "labels" and set(np.unique(wl)) <= {0.0, 1.0, 2.0}
    # evaluate on the written outputs (lddmm_cli.cpp:236-262)
    r = run("evaluate", "--source", str(d / "source.raw"), "--target", str(d / "target.raw"),
            "--warped", str(out / "warped_source.raw"), "--warped-labels", str(out / "warped_labels.raw"),
            "--target-labels", str(d / "target_labels.raw"), "--displacement",
            str(out / "displacement_inverse.raw"), "--out", str(tmp_path / "eval.json"))
    assert r.returncode == 0, r.stderr
    ev = json.loads(r.stdout)
    assert abs(ev["mse_rel"] - rep["mse_rel_final"]) < 1e-3
    assert ev["dice_mean"] == rep["dice_mean"]
    assert abs(ev["jacobian"]["min"] - rep["jacobian_inverse"]["min"]) < 1e-3
    assert abs(ev["jacobian"]["max"] - rep["jacobian_inverse"]["max"]) < 1e-3
    # warm start from the written velocity (--v0): one more run starts at the optimum
    r = run("register", "--source", str(d / "source.raw"), "--target", str(d / "target.raw"), "--out",
            str(tmp_path / "reg2"), "--variant", "deformation_state_equation", "--band", "16", "--sigma2", "0.01",
            "--max-iter", "1", "--v0", str(out / "velocity.raw"))
    assert r.returncode == 0, r.stderr
    with open(tmp_path / "reg2" / "report.json") as f:
        rep2 = json.load(f)
    assert rep2["mse_rel_initial"] < 0.5 * rep["mse_rel_initial"]


def test_cli_nonstationary_outputs(cuda, tmp_path):
    """--param nonstationary writes velocity_00 .. velocity_nt (lddmm_cli.cpp:136-143)."""
    assert run("synth", "--kind", "blobs", "--d", "3", "--n", "16", "--seed", "3", "--out",
               str(tmp_path / "b")).returncode == 0
    r = run("register", "--source", str(tmp_path / "b" / "source.raw"), "--target",
            str(tmp_path / "b" / "target.raw"), "--out", str(tmp_path / "r"), "--param", "nonstationary",
            "--band", "8", "--nt", "3", "--max-iter", "2", "--variant", "state_equation")
    assert r.returncode == 0, r.stderr
    for i in range(4):
        assert (tmp_path / "r" / f"velocity_{i:02d}.raw").exists()
    with open(tmp_path / "r" / "report.json") as f:
        assert json.load(f)["parameterization"] == "nonstationary"


def test_cli_rk4(cuda, tmp_path):
    """--integrator rk4 on the band representation (lddmm_cli.cpp:216-218: nt defaults to 25)."""
    assert run("synth", "--kind", "blobs", "--d", "3", "--n", "16", "--seed", "3", "--out",
               str(tmp_path / "b")).returncode == 0
    r = run("register", "--source", str(tmp_path / "b" / "source.raw"), "--target",
            str(tmp_path / "b" / "target.raw"), "--out", str(tmp_path / "r"), "--integrator", "rk4",
            "--band", "8", "--max-iter", "2", "--variant", "deformation_state_equation", "--sigma2", "0.01")
    assert r.returncode == 0, r.stderr
    with open(tmp_path / "r" / "report.json") as f:
        rep = json.load(f)
    assert rep["integrator"] == "rk4" and rep["nt"] == 25
    assert rep["mse_rel_final"] < rep["mse_rel_initial"]


@pytest.mark.parametrize("seed", [1, 2])
def test_two_disc_dice_matches_reference(cuda, seed):
    """Acceptance gate 8 analog (acceptance.cpp:307-343) in 3-D: per variant, the
    registration path (GN iterations, stop reason) and the mean Dice of the
    nearest-warped labels equal the reference's on the same float32 inputs
    (tests/golden/gate8.npz).  In 3-D the reference itself ranks deformation-state
    below the other two variants on these cases, so the 2-D ordering gate is not a
    property to require here."""
    from paper_2006_06823_b200 import lddmm as L
    z = np.load(os.path.join(GOLD, "gate8.npz"))
    s, t, sl, tl = (x.astype(np.float64) for x in z[f"s{seed}_inputs"])
    band = L.BandSpec(L.GridSpec(s.shape), (16, 16, 16))
    ctx = L.Context(band)
    assert L.mean_dice(ctx, sl, tl) == float(z[f"s{seed}_initial"])
    for v in ("original", "state_equation", "deformation_state_equation"):
        m = L.Model(band, s, t, v, 5, 0.05)
        res = L.optimize(m, None, L.OptimizeOptions(max_iter=30, grad_tol=1e-3))
        assert res.iterations == int(z[f"s{seed}_{v}_iterations"])
        assert L.STOP_REASONS.index(res.stop) == int(z[f"s{seed}_{v}_stop"])
        fwd, _, _ = L.compute_maps(m, res.v)
        d = L.mean_dice(ctx, L.warp(ctx, sl, fwd, kind="nearest"), tl)
        assert abs(d - float(z[f"s{seed}_{v}_dice"])) < 5e-3


def test_cli_register_2d_matches_reference(cuda, tmp_path):
    """`lddmm register` on a 2-D two-disc fixture (the reference CLI's default use) against
    the reference library run on the same rescaled images: GN path, final energy, mse_rel,
    Jacobian ranges, and the 2-D output layouts."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    r = run("synth", "--kind", "discs", "--d", "2", "--n", "64", "--seed", "5", "--out", str(tmp_path / "d"))
    assert r.returncode == 0, r.stderr
    d, out = tmp_path / "d", tmp_path / "reg"
    r = run("register", "--source", str(d / "source.raw"), "--target", str(d / "target.raw"),
            "--source-labels", str(d / "source_labels.raw"), "--target-labels", str(d / "target_labels.raw"),
            "--out", str(out), "--variant", "deformation_state_equation", "--band", "16", "--sigma2", "0.01",
            "--max-iter", "6")
    assert r.returncode == 0, r.stderr
    with open(out / "report.json") as f:
        rep = json.load(f)
    _, src = read_field(str(d / "source"))
    _, tgt = read_field(str(d / "target"))
    dims = src.shape
    s = ref.rescale_unit(src.astype(np.float64), dims, (1.0, 1.0))
    t = ref.rescale_unit(tgt.astype(np.float64), dims, (1.0, 1.0))
    m = ref.RefModel(s, t, dims, (1.0, 1.0), (16, 16), "deformation_state_equation", 5, 0.01)
    want = m.optimize(None, max_iter=6, pcg_max_iter=5)
    _, _, jac = m.maps(want["v"])
    assert rep["stop_reason"] == want["stop"] and rep["iterations"] == want["iterations"]
    assert abs(rep["final_energy"] - want["history"][-1].energy) <= 1e-5 * abs(want["history"][-1].energy)
    assert abs(rep["mse_rel_final"] - want["history"][-1].mse_rel) <= 1e-5
    assert np.allclose([rep["jacobian_forward"]["min"], rep["jacobian_forward"]["max"],
                        rep["jacobian_inverse"]["min"], rep["jacobian_inverse"]["max"]], jac, atol=1e-4)
    side, fwd = read_field(str(out / "displacement_forward"))
    assert side["components"] == 2 and fwd.shape == (2,) + dims
