"""Gather lab (B200): times the SL gather implementations at a BASELINE shape on a
smooth sub-voxel departure field like the SL steps' (|d| <= CFL ~ 0.27 voxel at config 2)
and checks them bitwise against the global-memory gather (impl 2).

    python tools/lab/gather_lab.py [Nx,Ny,Nz] [cfl]
    LDDMM_GATHER_PIPE=0 python tools/lab/gather_lab.py   # production = previous marching kernel

impl 0 = production dispatch (pipelined kernel when the shape allows), 3 = 8x4-tile window
kernel, 4 = pipelined kernel forced.  Prints one JSON line per (impl, F)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_06823_b200 import lddmm as L  # noqa: E402

dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "180,210,180").split(","))
cfl = float(sys.argv[2]) if len(sys.argv) > 2 else 0.27
real = os.environ.get("GATHER_LAB_REAL", "1") == "1" and dims == (180, 210, 180)
ctx = L.Context(L.BandSpec(L.GridSpec(dims, (1., 1., 1.)), (32, 32, 32) if real else (8, 8, 8)), nt=10 if real else 3)
ops = L.Ops(ctx)
g = torch.Generator(device="cuda").manual_seed(1)
coef = torch.randn((6,) + dims, device="cuda", generator=g)
x = [torch.arange(n, device="cuda", dtype=torch.float32) for n in dims]
X, Y, Z = torch.meshgrid(*x, indexing="ij")
tp = 6.283185307179586
dep = torch.stack([cfl * torch.sin(tp * (2 * X / dims[0] + Y / dims[1]) + a) * torch.cos(tp * Z / dims[2] * (a + 1))
                   for a in range(3)]).contiguous()
if real:
    # the SL departure field of the reference's own final config-2 velocity (config2_ref.npz)
    import numpy as np
    v = np.load(os.path.join(os.path.dirname(__file__), "..", "..", "tests", "golden", "config2_ref.npz"))["v"][0]
    df, db, cfl = ops.departure(v)
    dep = df
    fl = torch.floor(dep)
    G = dims[2] // 4
    grp = torch.roll(fl, 2, dims=3).reshape(3, dims[0], dims[1], G, 4)
    mixed = (grp.amax(-1) != grp.amin(-1))  # (3, Nx, Ny, G)
    mx, my, mz = (mixed[a].float().mean().item() for a in range(3))
    mxy = (mixed[0] | mixed[1])
    w = mxy.reshape(-1)[: (mxy.numel() // 32) * 32].reshape(-1, 32).any(-1).float().mean().item()
    print(json.dumps({"departure": "config2_ref final velocity", "cfl": cfl, "max_abs": dep.abs().max().item(),
                      "groups_mixed_x": mx, "groups_mixed_y": my, "groups_mixed_z": mz,
                      "groups_mixed_xy": mxy.float().mean().item(), "warps32_with_mixed_xy": w}))
ref = {nc: ops.gather(coef[:nc].contiguous(), dep, 2) for nc in (1, 3, 6)}
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream_ptr())  # events on the engine stream the kernels run on
for impl in tuple(int(x) for x in os.environ.get("GATHER_LAB_IMPLS", "0,4,3").split(",")):
    for nc in (3, 6, 1):
        c = coef[:nc].contiguous()
        try:
            out = ops.gather(c, dep, impl)
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"impl": impl, "F": nc, "error": str(exc)}))
            continue
        same = bool(torch.equal(out, ref[nc]))
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record(stream)
            ops.gather(c, dep, impl)
            e.record(stream)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        n = dims[0] * dims[1] * dims[2]
        us = ts[len(ts) // 2]
        print(json.dumps({"impl": impl, "F": nc, "dims": dims, "us_median": round(us, 1), "us_min": round(ts[0], 1),
                          "GBps": round(n * (12 + 8 * nc) / us / 1e3, 1), "bitwise_vs_global": same,
                          "pipe_env": os.environ.get("LDDMM_GATHER_PIPE", "1")}))
