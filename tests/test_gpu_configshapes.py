"""Primitive parity at the BASELINE grid shapes, where the production kernels that the
small test grids never select actually run: the tcgen05 z-stage embed / project of the
truncated DFT (umma_gemm.cu) and the pipelined TMA SL gather (gather_pipe.cu).

Config 2: 180x210x180, band 32^3.  Config 4: 256^3, band 64^3.  embed / project are
checked against the numpy restatement (oracle/lddmm_np.py, spectral.hpp:242-285) at the
2e-6 relative-L2 tolerance of the small-grid tests (4e-6 at Nz = 256, see below); advect_state (transport.hpp:67-73)
against the reference library itself (oracle/_ref, the unmodified headers) at 5e-6.
"""
import os

import numpy as np
import pytest

from oracle import lddmm_np as O

pytestmark = pytest.mark.gpu

SHAPES = [((180, 210, 180), (32, 32, 32)), ((256, 256, 256), (64, 64, 64))]


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def band_field(g, b, ncomp, seed):
    """Smooth random band coefficients (decaying spectrum, reference DFT order)."""
    rng = np.random.default_rng(seed)
    shape = (ncomp,) + b.bounds
    c = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    k2 = sum(w * w for w in np.meshgrid(*[b.signed_freq(a).astype(float) for a in range(3)], indexing="ij"))
    c = c * np.exp(-0.02 * k2)
    # a real field's spectrum: project the embedded field (Hermitian, band Nyquist zero)
    return O.project(O.embed(c, b), b)


@pytest.mark.parametrize("dims,band", SHAPES)
def test_embed_project_config_shapes(cuda, dims, band):
    from paper_2006_06823_b200 import lddmm as L
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, band)
    ctx = L.Context(L.BandSpec(L.GridSpec(dims), band), nt=2)
    ops = L.Ops(ctx)
    c = band_field(g, b, 3, 1)
    want = O.embed(c, b)
    got = ops.embed(c, 3).cpu().numpy()
    e_embed = rel(got, want)
    rng = np.random.default_rng(2)
    f = rng.standard_normal((3,) + dims).astype(np.float32)
    got_p = ops.to_complex(ops.project(cuda.from_numpy(f).cuda()))
    e_proj = rel(got_p, O.project(f.astype(np.float64), b))
    back = ops.to_complex(ops.project(ops.embed(c, 3)))
    e_rt = rel(back, c)
    print(f"{dims} K={band[0]}: embed {e_embed:.2e}, project {e_proj:.2e}, pi(iota) {e_rt:.2e}")
    # fp32 accumulation over the Nz-long z contraction of the project (256 terms at config
    # 4): the 3xTF32 products are ~fp32-exact, the sums grow like sqrt(Nz) * 2^-24
    tol = 2e-6 if dims[2] <= 192 else 4e-6
    assert e_embed < tol and e_proj < tol and e_rt < tol


@pytest.mark.parametrize("dims,band", SHAPES)
def test_advect_config_shapes_vs_reference(cuda, dims, band):
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2006_06823_b200 import lddmm as L
    ref.set_threads(os.cpu_count() or 1)
    g = O.Grid(dims, (1.0, 1.0, 1.0))
    b = O.Band(g, band)
    ctx = L.Context(L.BandSpec(L.GridSpec(dims), band), nt=2)
    ops = L.Ops(ctx)
    q = band_field(g, b, 3, 3)
    # smooth sub-voxel departure displacement (grid units), SL-step magnitude
    x = O.identity_map(g)
    dep = np.stack([0.3 * np.sin(2 * np.pi * (x[0] / dims[0] + 2 * x[1] / dims[1]) + a) *
                    np.cos(2 * np.pi * (a + 1) * x[2] / dims[2]) for a in range(3)])
    got = ops.to_complex(ops.advect(q, 3, cuda.from_numpy(dep.astype(np.float32)).cuda()))
    pts = np.ascontiguousarray(x + dep.astype(np.float32).astype(np.float64))
    want = ref.advect_band(q, pts, dims, (1.0, 1.0, 1.0), band)
    e = rel(got, want)
    print(f"{dims} K={band[0]}: advect vs reference {e:.2e}")
    assert e < 5e-6


def _embed_project_in_subprocess(env_extra):
    """embed / project of fixed fields at config 2 in a fresh process (the x-stage choice is
    made when the plan is built): returns (embed grid, projected band)."""
    import subprocess
    import sys
    import tempfile
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2006_06823_b200 import lddmm as L
from oracle import lddmm_np as O
dims, band = (180, 210, 180), (32, 32, 32)
ctx = L.Context(L.BandSpec(L.GridSpec(dims), band), nt=2)
ops = L.Ops(ctx)
rng = np.random.default_rng(3)
b = O.Band(O.Grid(dims, (1.0, 1.0, 1.0)), band)
c = O.project(rng.standard_normal((3,) + dims), b)
f = torch.from_numpy(rng.standard_normal((3,) + dims).astype(np.float32)).cuda()
np.savez(sys.argv[1], e=ops.embed(c, 3).cpu().numpy(), p=ops.to_complex(ops.project(f)))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        env = dict(os.environ, **env_extra)
        subprocess.run([sys.executable, "-c", code, out], check=True, env=env, timeout=600)
        z = np.load(out)
        return z["e"], z["p"]


def test_xstage_tensor_cores_match_ffma(cuda):
    """The tcgen05 x stage (umma_xstage.cu, 3xTF32 complex GEMM, production at config 2)
    against the FFMA x stage (LDDMM_UMMA_X=0) on the same inputs: embed and project agree
    to fp32 accuracy (both are ~1e-7 from the fp64 transform), and they are not bitwise
    equal — the tensor-core path really ran."""
    e1, p1 = _embed_project_in_subprocess({})
    e0, p0 = _embed_project_in_subprocess({"LDDMM_UMMA_X": "0"})
    de, dp = rel(e1, e0), rel(p1, p0)
    print(f"x stage tcgen05 vs FFMA at config 2: embed {de:.2e}, project {dp:.2e}")
    assert de < 1e-6 and dp < 1e-6
    assert not (np.array_equal(e1, e0) and np.array_equal(p1, p0))
