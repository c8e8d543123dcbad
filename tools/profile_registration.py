"""One full config-2 registration (bench.py's workload) inside cudaProfilerStart/Stop,
after one untimed warm-up registration, for an ncu launch list
(ncu --profile-from-start off).  Prints the device time of the profiled registration
measured with CUDA events (run without ncu) and its launch count, so the sum of the
kernel durations can be set against the step time (the difference is inter-kernel
idle time: launch gaps and host round trips of the optimizer's scalar decisions)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2006_06823_b200 import lddmm as L
from paper_2006_06823_b200 import phantoms

dims = (180, 210, 180)
I0, I1 = phantoms.brain_pair(dims, seed=2006)
d0 = torch.from_numpy(I0).cuda().float()
d1 = torch.from_numpy(I1).cuda().float()
m = L.Model(L.BandSpec(L.GridSpec(dims), (32, 32, 32)), d0, d1, "deformation_state_equation", 10, 0.01)
opt = L.OptimizeOptions(max_iter=10, pcg_max_iter=5)
stream = torch.cuda.ExternalStream(m.ctx.stream_ptr(), device="cuda:0")


def reg():
    m.set_images(d0, d1)
    return L.optimize(m, None, opt)


reg()
torch.cuda.synchronize()
n0 = L.launch_count()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record(stream)
r = reg()
e1.record(stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"registration: {e0.elapsed_time(e1):.2f} ms device time, {L.launch_count() - n0} engine launches, "
      f"{r.iterations} GN iterations, {r.hessvecs} hessvecs, {r.trials} trials")
