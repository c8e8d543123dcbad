"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) runs: one config-2
forward + gradient + Hessian-vector product (tcgen05 z-stage embed / project, the
pipelined TMA gather, the last-block non-finite flag reduction) and a small 20^3
model with all three variants (the small-grid product kernels, the mma.sync small
z stages, the global-memory gather fallback via a large displacement).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [small]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_06823_b200 import lddmm as L  # noqa: E402
from paper_2006_06823_b200 import phantoms  # noqa: E402


def run(dims, band, nt, variants):
    I0, I1 = phantoms.brain_pair(dims, seed=2006)
    rng = np.random.default_rng(0)
    for variant in variants:
        m = L.Model(L.BandSpec(L.GridSpec(dims), band), I0, I1, variant, nt, 0.01)
        v = m.zero_velocity()
        e0 = m.forward(v, True)
        g = m.gradient()
        v = m.velocity(-0.5 * g.numpy() / max(np.abs(g.numpy()).max(), 1e-30))
        e1 = m.forward(v, True)
        g = m.gradient()
        dv = m.velocity(rng.standard_normal(m.ctx.vel_shape) * 0.1)
        hv = m.hessvec(dv)
        print(dims, variant, e0["energy"], e1["energy"], float(np.abs(hv.numpy()).max()), flush=True)
        del m


if __name__ == "__main__":
    run((20, 18, 16), (8, 8, 8), 4, ["deformation_state_equation", "original", "state_equation"])
    if len(sys.argv) < 2 or sys.argv[1] != "small":
        run((180, 210, 180), (32, 32, 32), 10, ["deformation_state_equation"])
    # the gather alone at config 2, including multi-voxel departures (global-memory path)
    ctx = L.Context(L.BandSpec(L.GridSpec((180, 210, 180)), (8, 8, 8)), nt=2)
    ops = L.Ops(ctx)
    import torch
    dep = torch.zeros((3, 180, 210, 180), device="cuda")
    dep[:, :, :, :] = 0.2
    dep[:, 5:9, 10:20, 30:60] = 2.5
    out = ops.gather(torch.randn((3, 180, 210, 180), device="cuda"), dep, 0)
    print("gather ok", float(out.abs().max()))
