"""Config 3: the config-2 pair registered with each of the three BL variants
(SPEC.md / variants.hpp:34) on one B200; prints one JSON line per variant with
s/registration, GN/PCG counts, final mse_rel and Jacobian extrema."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_06823_b200 import lddmm as L  # noqa: E402
from paper_2006_06823_b200 import phantoms  # noqa: E402

dims = tuple(int(x) for x in os.environ.get("DIMS", "180,210,180").split(","))
K = int(os.environ.get("BAND", "32"))
nt = int(os.environ.get("NT", "10"))
reps = int(os.environ.get("REPS", "2"))
integ = os.environ.get("INTEGRATOR", "sl")
I0, I1 = phantoms.brain_pair(dims)
d0 = torch.from_numpy(I0).cuda().float()
d1 = torch.from_numpy(I1).cuda().float()
for variant in ("deformation_state_equation", "original", "state_equation"):
    m = L.Model(L.BandSpec(L.GridSpec(dims), (K, K, K)), d0, d1, variant, nt, 0.01, integrator=integ)
    opt = L.OptimizeOptions(max_iter=10, pcg_max_iter=5)
    times = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m.set_images(d0, d1)
        res = L.optimize(m, None, opt)
        m.ctx.sync()
        times.append(time.perf_counter() - t0)
    f, i, jac = L.compute_maps(m, res.v)
    print(json.dumps({"variant": variant, "s_per_registration": min(times[1:]), "stop": res.stop,
                      "iterations": res.iterations, "hessvecs": res.hessvecs, "trials": res.trials,
                      "pcg": [h.pcg_iters for h in res.history[1:]],
                      "mse_rel_final": res.history[-1].mse_rel, "jacobian": list(jac),
                      "dims": dims, "band": K, "nt": nt, "integrator": integ}))
    del m
