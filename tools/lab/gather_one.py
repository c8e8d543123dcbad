"""One launch per listed gather impl on the reference's config-2 departure field (for ncu):
    python tools/lab/gather_one.py 4,6 [F]
impl 5 / 6 (planned gather) exist only with tools/lab/gather_class_plan.patch applied; impl 6
reuses the plan of an impl-5 call made first (its own launches come before)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_06823_b200 import lddmm as L  # noqa: E402

impls = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,6").split(",")]
F = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dims = (180, 210, 180)
ctx = L.Context(L.BandSpec(L.GridSpec(dims, (1., 1., 1.)), (32, 32, 32)), nt=10)
ops = L.Ops(ctx)
v = np.load(os.path.join(os.path.dirname(__file__), "..", "..", "tests", "golden", "config2_ref.npz"))["v"][0]
dep, _, _ = ops.departure(v)
coef = torch.randn((F,) + dims, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
for impl in impls:
    if impl == 6:
        ops.gather(coef, dep, 5)
    ops.gather(coef, dep, impl)
torch.cuda.synchronize()
print("done", impls, F)
