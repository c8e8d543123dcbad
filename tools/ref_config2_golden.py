"""Run the REFERENCE (oracle/_ref, unmodified headers) on the bench workload once,
offline, and store its GN-Krylov history and final velocity as a golden fixture
(tests/golden/config2_ref.npz).  Takes O(hours) of CPU; run in this container:

    python tools/ref_config2_golden.py [threads] [config2|config1]

Workload = bench.py's config 2 (180x210x180 brain-like pair, seed 2006, K=32,
nt=10, deformation-state, sigma2=0.01, OptimizeOptions defaults, max_iter=10).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2006_06823_b200 import phantoms  # noqa: E402

threads = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dims, band, nt, sigma2 = (180, 210, 180), (32, 32, 32), 10, 0.01
mode = sys.argv[2] if len(sys.argv) > 2 else "config2"
ref.set_threads(threads)
if mode == "config1":  # BASELINE.json configs[0]: 64^3 sphere -> ellipsoid, K = 16
    dims, band = (64, 64, 64), (16, 16, 16)
    I0, I1 = phantoms.sphere_ellipsoid_pair(64)
else:
    I0, I1 = phantoms.brain_pair(dims, seed=2006)
# the engine consumes fp32 images; feed the reference the identical values
I0 = I0.astype(np.float32).astype(np.float64)
I1 = I1.astype(np.float32).astype(np.float64)
m = ref.RefModel(I0, I1, dims, (1.0, 1.0, 1.0), band, "deformation_state_equation", nt, sigma2)
t0 = time.time()
r = m.optimize(None, max_iter=10, pcg_max_iter=5)
wall = time.time() - t0
hist = np.array([[q.iter, q.energy, q.energy_data, q.energy_reg, q.mse_rel, q.rel_grad, q.pcg_iters,
                  q.pcg_fallback, q.epsilon, q.cfl] for q in r["history"]])
fwd, inv, jac = m.maps(r["v"])
tag = mode
np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"{tag}_ref.npz"), dims=np.array(dims),
                    band=np.array(band), nt=nt, sigma2=sigma2, history=hist, v=r["v"],
                    stop=ref.STOP_REASONS.index(r["stop"]), iterations=r["iterations"], jac=jac,
                    wall_s=wall, threads=threads)
print("done", r["stop"], r["iterations"], wall, hist[:, [0, 1, 6, 8]])
