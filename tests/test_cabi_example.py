"""The standalone C++ program examples/trace_cabi.cpp drives the library
through include/dist.h alone (no Python, no torch on its path): trace ->
depth map -> normal map for one view.  The CPU test checks that it builds and
fails loudly without a device; the GPU test checks its outputs equal the
Python package's bit for bit (same kernels, same inputs)."""
from __future__ import annotations

import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "trace_cabi")


@pytest.fixture(scope="module")
def exe():
    if not os.path.exists(os.path.join(ROOT, "paper_1911_13225_b200", "libdist_b200.so")):
        pytest.skip("libdist_b200.so not built")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    return EXE


def _job(path, net, code, intr, pose, cfg):
    """Write the flat job file examples/trace_cabi.cpp reads."""
    from paper_1911_13225_b200 import _lib
    from paper_1911_13225_b200.camera import camera_struct
    L = len(net.weights)
    dims = [net.weights[0][0].shape[0] if net.skip < 0 else net.latent_dim + 3]
    dims += [W.shape[1] for W, _ in net.weights]
    fin = {"tanh": 0, "linear": 1, "sigmoid": 2}[net.final_activation]
    with open(path, "wb") as f:
        f.write(struct.pack("<5i", L, net.latent_dim, net.skip, fin, _lib.PREC[net.precision]))
        f.write(np.asarray(dims, dtype="<i4").tobytes())
        for W, b in net.weights:
            f.write(np.ascontiguousarray(W, dtype="<f8").tobytes())
            f.write(np.ascontiguousarray(b, dtype="<f8").tobytes())
        f.write(np.asarray(code, dtype="<f8").tobytes())
        f.write(bytes(camera_struct(intr, pose, 0)))
        f.write(bytes(_lib.config_struct(cfg)))


def _read_out(path, n, max_steps):
    raw = open(path, "rb").read()
    o = 0
    stats = np.frombuffer(raw, "<i8", 4, o); o += 32
    live = np.frombuffer(raw, "<i8", max_steps, o); o += 8 * max_steps
    depth = np.frombuffer(raw, "<f8", n, o); o += 8 * n
    status = np.frombuffer(raw, "u1", n, o); o += n
    normals = np.frombuffer(raw, "<f8", 3 * n, o); o += 24 * n
    assert o == len(raw)
    return stats, live, depth, status, normals


def test_example_builds_and_fails_loudly_without_device(exe, tmp_path):
    """Built against include/dist.h; with no GPU it exits non-zero with the
    library's error message instead of computing anything."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_1911_13225_b200 as st
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision="fp64")
    job = tmp_path / "job.bin"
    _job(job, net, rng.normal(0.0, 0.3, 2), st.Intrinsics(width=32, height=32),
         st.look_at((0.0, 0.0, -2.0)), st.TraceConfig())
    p = subprocess.run([exe, str(job), str(tmp_path / "out.bin")], capture_output=True, text=True)
    assert p.returncode != 0
    assert "dist_device_info" in p.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp64", "fp16x3"])
def test_example_matches_python_package(exe, tmp_path, prec):
    import json

    import paper_1911_13225_b200 as st
    if prec == "fp64":
        rng = np.random.default_rng(7)
        net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision=prec)
        code, res = rng.normal(0.0, 0.3, 2), 64
    else:
        net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
        code, res = np.random.default_rng(3).normal(0.0, 0.1, 256), 128
    intr, pose, cfg = st.Intrinsics(width=res, height=res), st.look_at((0.3, 0.2, -2.0)), st.TraceConfig()
    job, out = tmp_path / "job.bin", tmp_path / "out.bin"
    _job(job, net, code, intr, pose, cfg)
    p = subprocess.run([exe, str(job), str(out)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    info = json.loads(p.stdout)
    assert info["sm_count"] >= 1 and info["launches"] > 0
    stats, live, depth, status, normals = _read_out(out, res * res, cfg.max_steps)

    r = st.trace(net, code, intr, pose, cfg)
    assert int(stats[0]) == r.total_queries
    assert list(live[:len(r.live_counts)]) == list(r.live_counts)
    assert np.array_equal(status, r.state.status)
    assert np.array_equal(depth, st.depth_map(r).reshape(-1))
    assert np.array_equal(normals, st.normal_map(r).reshape(-1))
    assert info["converged"] == int(np.sum(r.state.status == 1)) > 0
