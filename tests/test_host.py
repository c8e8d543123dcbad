"""CPU tests of the host side: the C ABI library loads and exports every symbol
include/lddmm_cuda.h declares (no compute calls without a GPU), the synthetic
volumes are deterministic, the reference cost model matches the transform
counts read off the reference code, and the bench JSON contract."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "lddmm_cuda.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lddmm_[a-z0-9_]+)\s*\(", txt)))


def test_capi_exports_every_declared_symbol():
    lib_path = os.path.join(ROOT, "paper_2006_06823_b200", "liblddmm_cuda.so")
    if not os.path.exists(lib_path):
        pytest.fail("liblddmm_cuda.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(lib_path)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_mirror_fails_loudly_without_gpu():
    import torch
    from paper_2006_06823_b200 import lddmm as L
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises((L.CudaError, RuntimeError)):
        L.Model(L.BandSpec(L.GridSpec((8, 8, 8)), (4, 4, 4)), np.zeros((8, 8, 8)), np.zeros((8, 8, 8)))


def test_phantoms_deterministic():
    from paper_2006_06823_b200 import phantoms
    s1, t1 = phantoms.brain_pair((24, 28, 20), seed=7)
    s2, t2 = phantoms.brain_pair((24, 28, 20), seed=7)
    assert np.array_equal(s1, s2) and np.array_equal(t1, t2)
    assert s1.min() == 0.0 and s1.max() == 1.0
    assert not np.array_equal(s1, t1)
    a, b = phantoms.sphere_ellipsoid_pair(32)
    assert a.shape == (32, 32, 32) and 0.0 <= a.min() and a.max() == 1.0


def test_reference_cost_model_counts():
    """Transform counts per GN iteration (4,939 full-grid FFTs and 794 scalar
    gathers at nt = 10 for 5 PCG + 1 trial)."""
    from oracle import ref
    c = ref.defstate_op_counts(10, 1, 5, 1)
    base = ref.defstate_op_counts(10, 0, 5, 1)
    assert c["fft"] - base["fft"] == 4939
    # scalar gathers: warps (prefilter + gather) + the provider's departure gathers
    assert (c["warp"] + c["gath"]) - (base["warp"] + base["gath"]) == 794
    m = ref.defstate_op_counts_measured(10, 1, 5, 1)
    assert m["fft"] == 4939


def test_oracle_reference_build_matches_numpy_fft():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    dims, h, band = (12, 10, 8), (1.0, 1.0, 1.0), (6, 6, 4)
    rng = np.random.default_rng(0)
    f = rng.standard_normal((1,) + dims)
    c = ref.project(f, dims, h, band)
    F = np.fft.fftn(f[0])
    idx = lambda K, N: [k if k < K // 2 else k - K + N for k in range(K)]  # noqa: E731
    want = F[np.ix_(idx(6, 12), idx(6, 10), idx(4, 8))].copy()
    for a, K in enumerate(band):
        sl = [slice(None)] * 3
        sl[a] = K // 2
        want[tuple(sl)] = 0
    assert np.max(np.abs(c[0] - want)) < 1e-12


def test_bench_reference_arm_runs_small(monkeypatch, capsys):
    """bench.py --impl reference prints one JSON line with the contract keys (tiny grid)."""
    import importlib
    import json
    import sys
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    monkeypatch.setattr(bench, "DIMS", (24, 20, 16))
    monkeypatch.setattr(bench, "BAND", (8, 8, 8))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"])
    bench.main()
    line = capsys.readouterr().out.strip().splitlines()[-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "higher_is_better"):
        assert k in d
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is False
