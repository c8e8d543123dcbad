"""The y-stage fusions are exact: band prep fused into the y-stage embed and band
finalize fused into the y-stage project give bitwise the results of the separate
band_prep / band_finalize kernels (the same operations on the same values).  The
switches are read once per process, so each setting runs in its own interpreter."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json
import numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2006_06823_b200 import lddmm as L
from oracle import lddmm_np as O
dims, band = (24, 20, 16), (8, 8, 6)
g = O.Grid(dims, (1.0, 1.0, 1.0)); b = O.Band(g, band)
ctx = L.Context(L.BandSpec(L.GridSpec(dims), band), nt=3, sigma2=1.0)
ops = L.Ops(ctx)
rng = np.random.default_rng(3)
c = O.project(rng.standard_normal((3,) + dims), b)
f = torch.from_numpy(rng.standard_normal((3,) + dims).astype(np.float32)).cuda()
emb = ops.embed(c, 3, prefilter=True).cpu().numpy()
pro = ops.to_complex(ops.project(f))
I0 = O.embed(O.project(rng.standard_normal((1,) + dims), b), b)[0]
I1 = np.roll(I0, 1, axis=0)
m = L.Model(L.BandSpec(L.GridSpec(dims), band), I0, I1, "deformation_state_equation", 4, 0.05)
res = L.optimize(m, None, L.OptimizeOptions(max_iter=3))
np.savez(OUT, emb=emb, pro=pro, energy=np.array([h.energy for h in res.history]))
"""


def run(tmp_path, name, env_extra):
    out = str(tmp_path / f"{name}.npz")
    env = dict(os.environ, **env_extra)
    code = f"ROOT = {ROOT!r}\nOUT = {out!r}\n" + CHILD
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=ROOT, timeout=600)
    return np.load(out)


def test_fused_prep_and_finalize_bitwise(cuda, tmp_path):
    fused = run(tmp_path, "fused", {})
    plain = run(tmp_path, "plain", {"LDDMM_NO_PREP_FUSION": "1", "LDDMM_NO_FIN_FUSION": "1"})
    assert np.array_equal(fused["emb"], plain["emb"])
    assert np.array_equal(fused["pro"], plain["pro"])
    assert np.array_equal(fused["energy"], plain["energy"])
