"""The drop-in proof: the REFERENCE's own
optimize<Alg> / pcg_solve<Alg> templates (optimizer.hpp:86-262, unmodified header),
instantiated over Model<CudaBandAlgebra> (integration/cuda_band_algebra.hpp: every
Model operator and the TV algebra through the C ABI), register BASELINE config 1
(64^3 sphere -> ellipsoid, K = 16, nt = 10, sigma2 = 0.01) on the B200 and take exactly
the path of the engine's own C++ driver (lddmm_optimize) on the same context: same
stop reason, GN iterations, PCG counts, fallbacks, step lengths, bitwise-equal
energies and final velocity (both drive the same device operators in the same order;
mse_rel is formed on the host by the reference from the fp64 images and the fetched
residual, and on the device by the driver, so it agrees to ~1e-8)."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_optimize")


def test_reference_optimize_over_cuda_band_algebra(cuda):
    if not os.path.exists(EXE):
        pytest.skip("integration/Makefile output missing (built by __graft_entry__.build() with /root/reference)")
    from paper_2006_06823_b200 import phantoms
    I0, I1 = phantoms.sphere_ellipsoid_pair(64)
    with tempfile.TemporaryDirectory() as d:
        p0, p1, vr, vd = (os.path.join(d, x) for x in ("i0.f64", "i1.f64", "v_ref.f64", "v_drv.f64"))
        I0.astype(np.float64).tofile(p0)
        I1.astype(np.float64).tofile(p1)
        out = subprocess.run([EXE, "64", "64", "64", "16", "16", "16", "10", "0.01", "10", p0, p1, vr, vd],
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr
        r = json.loads(out.stdout)
        v_ref, v_drv = np.fromfile(vr), np.fromfile(vd)
    a, b = r["reference_optimize"], r["engine_driver"]
    print(json.dumps({"stop": a["stop"], "iterations": a["iterations"],
                      "pcg": [h["pcg_iters"] for h in a["history"]],
                      "energy": [h["energy"] for h in a["history"]]}))
    assert a["stop"] == b["stop"] and a["iterations"] == b["iterations"]
    assert len(a["history"]) == len(b["history"]) >= 2
    for x, y in zip(a["history"], b["history"]):
        for k in ("iter", "pcg_iters", "pcg_fallback", "epsilon", "energy", "energy_data", "energy_reg", "cfl",
                  "rel_grad"):
            assert x[k] == y[k], (k, x, y)
        # the reference's denominator |I1 - I0|^2 uses the fp64 host images, the engine's
        # the fp32 device copies: ~1e-8 apart (SURVEY.md §8c allows 1e-5)
        assert abs(x["mse_rel"] - y["mse_rel"]) <= 1e-6
    assert np.array_equal(v_ref, v_drv)
