"""The `lddmm` command-line front end (paper_2006_06823_b200/csrc/cli.cpp), the
drop-in for the reference driver tools/lddmm_cli.cpp.  CPU-side checks: the
`synth` generators against the reference's own blob_pair / two_disc_case
(synth.hpp:182-259, golden fixtures from tests/golden/make_golden.py), the
.raw/.json sidecar format (io.hpp:94-164) and the usage exit codes
(lddmm_cli.cpp:333-358).  The GPU end-to-end run is in test_gpu_eval.py."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2006_06823_b200", "lddmm")
GOLD = os.path.join(ROOT, "tests", "golden")


def run(*args):
    if not os.path.exists(CLI):
        pytest.fail(f"{CLI} missing: build with __graft_entry__.build()")
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)


def read_field(base):
    with open(base + ".json") as f:
        side = json.load(f)
    data = np.fromfile(base + ".raw", dtype="<f4")
    shape = tuple(side["dims"])
    if side["kind"] == "vector":
        shape = (side["components"],) + shape
    return side, data.reshape(shape)


@pytest.mark.parametrize("d", [2, 3])
def test_synth_matches_reference(tmp_path, d):
    z = np.load(os.path.join(GOLD, "synth.npz"))
    r = run("synth", "--kind", "blobs", "--d", str(d), "--n", "16", "--seed", "3", "--out", str(tmp_path / "b"))
    assert r.returncode == 0, r.stderr
    for name in ("source", "target"):
        side, f = read_field(str(tmp_path / "b" / name))
        assert side == {"dims": [16] * d, "spacing": [1.0] * d, "kind": "scalar", "components": 1}
        assert np.max(np.abs(f - z[f"blobs{d}_{name}"].astype(np.float32))) <= 2e-7
    r = run("synth", "--kind", "discs", "--d", str(d), "--n", "16", "--seed", "5", "--out", str(tmp_path / "d"))
    assert r.returncode == 0, r.stderr
    for name in ("source", "target", "source_labels", "target_labels"):
        side, f = read_field(str(tmp_path / "d" / name))
        want = z[f"discs{d}_{name}"].astype(np.float32)
        if name.endswith("labels"):
            assert side["kind"] == "labels"
            assert np.array_equal(f, want)
        else:
            assert np.max(np.abs(f - want)) <= 2e-7


def test_usage_and_input_errors(tmp_path):
    assert run("--help").returncode == 0
    assert run("register", "--help").returncode == 0
    assert run().returncode == 1
    assert run("bogus").returncode == 1
    assert run("register", "--source", "a.raw").returncode == 1  # missing required options
    assert run("synth", "--out", str(tmp_path), "--bogus", "1").returncode == 1
    assert run("synth", "--out", str(tmp_path), "--d", "4").returncode == 1
    assert run("synth", "--out", str(tmp_path), "--kind", "rotation").returncode == 1
    r = run("register", "--source", str(tmp_path / "nope.raw"), "--target", str(tmp_path / "nope.raw"),
            "--out", str(tmp_path / "o"))
    assert r.returncode == 1 and "cannot open sidecar" in r.stderr
    # the spatial representation is outside the engine: status 1 with a reason
    assert run("synth", "--kind", "blobs", "--n", "16", "--out", str(tmp_path / "b2")).returncode == 0
    r = run("register", "--source", str(tmp_path / "b2" / "source.raw"), "--target",
            str(tmp_path / "b2" / "target.raw"), "--out", str(tmp_path / "o3"), "--repr", "spatial")
    assert r.returncode == 1 and "spatial" in r.stderr
    # payload / sidecar mismatch (io.hpp:66-80)
    with open(tmp_path / "b2" / "source.raw", "ab") as f:
        f.write(b"\0\0\0\0")
    r = run("evaluate", "--source", str(tmp_path / "b2" / "source.raw"), "--target",
            str(tmp_path / "b2" / "target.raw"))
    assert r.returncode == 1 and "payload size mismatch" in r.stderr


def test_evaluate_mse_only(tmp_path):
    """`evaluate` with only images needs no GPU: mse_rel on the host (metrics.hpp:82-89)."""
    assert run("synth", "--kind", "blobs", "--d", "3", "--n", "16", "--out", str(tmp_path / "b")).returncode == 0
    r = run("evaluate", "--source", str(tmp_path / "b" / "source.raw"), "--target",
            str(tmp_path / "b" / "target.raw"), "--out", str(tmp_path / "e.json"))
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep == {"mse_rel": 1.0}
    with open(tmp_path / "e.json") as f:
        assert json.load(f) == rep
