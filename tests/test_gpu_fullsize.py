"""Full-size parity against the REFERENCE itself: the GN-Krylov history and final
velocity of BASELINE.json's configs, produced once by the unmodified reference
(oracle/_ref, tools/ref_config2_golden.py — hours of CPU) and committed as
tests/golden/config{1,2}_ref.npz.  The engine reruns the same registration on the
GPU (fp32 grids, fp64 band algebra) and must take the same path: identical GN
iteration count, PCG iteration counts, step lengths and stop reason; per-iteration
energies within 1e-4 relative; final velocity within 1e-3 relative L2; the
deformation Jacobian range within 1e-3 (optimizer.hpp:143-262, metrics.hpp:24-79).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def pair(tag, dims):
    from paper_2006_06823_b200 import phantoms
    if tag == "config1":
        return phantoms.sphere_ellipsoid_pair(dims[0])
    return phantoms.brain_pair(dims, seed=2006)


@pytest.mark.parametrize("tag", ["config1", "config2"])
def test_registration_matches_reference(cuda, tag):
    path = os.path.join(GOLD, f"{tag}_ref.npz")
    if not os.path.exists(path):
        pytest.skip(f"{tag}_ref.npz not generated (tools/ref_config2_golden.py)")
    from paper_2006_06823_b200 import lddmm as L
    z = np.load(path)
    dims, band = tuple(int(x) for x in z["dims"]), tuple(int(x) for x in z["band"])
    I0, I1 = pair(tag, dims)
    m = L.Model(L.BandSpec(L.GridSpec(dims), band), I0, I1, "deformation_state_equation", int(z["nt"]),
                float(z["sigma2"]))
    res = L.optimize(m, None, L.OptimizeOptions(max_iter=10, pcg_max_iter=5))
    hist = z["history"]
    assert L.STOP_REASONS.index(res.stop) == int(z["stop"])
    assert res.iterations == int(z["iterations"])
    assert len(res.history) == hist.shape[0]
    for r, row in zip(res.history, hist):
        assert r.pcg_iters == int(row[6]) and r.pcg_fallback == bool(row[7]) and r.epsilon == row[8]
        assert abs(r.energy - row[1]) <= 1e-4 * abs(row[1])
        assert abs(r.energy_data - row[2]) <= 1e-4 * abs(row[2])
        assert abs(r.mse_rel - row[4]) <= 1e-4
    assert rel(res.v.numpy(), z["v"]) < 1e-3
    _, _, jac = L.compute_maps(m, res.v)
    assert np.allclose(jac, z["jac"], rtol=1e-3, atol=1e-3)
