"""One GN-iteration's worth of engine work at config 2 for ncu capture.

Runs forward(with adjoint) + gradient + one hessvec + one energy trial once to warm
up, then the same sequence inside cudaProfilerStart/Stop (use ncu
--profile-from-start off).  Prints the engine's launch count for the profiled region.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2006_06823_b200 import lddmm as L
from paper_2006_06823_b200 import phantoms

dims = tuple(int(x) for x in os.environ.get("DIMS", "180,210,180").split(","))
K = int(os.environ.get("BAND", "32"))
nt = int(os.environ.get("NT", "10"))
I0, I1 = phantoms.brain_pair(dims)
d0 = torch.from_numpy(I0).cuda().float()
d1 = torch.from_numpy(I1).cuda().float()
m = L.Model(L.BandSpec(L.GridSpec(dims), (K, K, K)), d0, d1, "deformation_state_equation", nt, 0.01)
rng = np.random.default_rng(0)
v = m.zero_velocity()
res = L.optimize(m, v, L.OptimizeOptions(max_iter=1))
v = res.v


def seq():
    m.forward(v, True)
    g = m.gradient()
    m.hessvec(g)
    m.energy(v)


seq()
torch.cuda.synchronize()
n0 = L.launch_count()
torch.cuda.profiler.start()
seq()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches in profiled region:", L.launch_count() - n0)
