"""pose objective and recovery against the reference golden."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_weights, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _setup(st, prec):
    g = load_golden("pose32.npz")
    net = st.NeuralField(golden_weights(g), latent_dim=2, precision=prec)
    obs = [st.Observation("depth", g["obs_depth"]), st.Observation("silhouette", g["obs_sil"])]
    cfg = st.TraceConfig(alpha=1.0, k_samples=1, coarse_start_scale=1)
    return g, net, obs, st.Intrinsics(width=32, height=32), cfg


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 1e-3)])
def test_pose_objective_vs_reference(st, prec, tol):
    g, net, obs, intr, cfg = _setup(st, prec)
    tot, terms, grad, q = st.pose_objective(net, g["code"], obs, intr, g["params"], cfg,
                                            st.LossWeights())
    assert abs(tot - float(g["total"])) < tol * abs(float(g["total"]))
    assert np.linalg.norm(grad - g["grad"]) / np.linalg.norm(g["grad"]) < tol
    if prec == "fp64":
        assert q == int(g["queries"])


def test_recover_pose_history_vs_reference(st):
    g, net, obs, intr, cfg = _setup(st, "fp64")
    best, rep = st.recover_pose(net, g["code"], obs, intr, st.Pose.from_params(g["params"]),
                                iters=5, cfg=cfg, lr_decay_every=2)
    np.testing.assert_allclose(rep.losses, g["rp_losses"], rtol=1e-9, atol=1e-12)
    assert rep.best_iter == int(g["rp_best_iter"])
    np.testing.assert_allclose(best.params(), g["rp_best"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("k", [1, 3])
def test_pose_objective_device_equals_host_path(st, monkeypatch, k):
    """The device objective (dist_pose_samples/seeds/grad) against the
    HeadBundle host path: K samples per pixel sharing one unit of depth weight,
    a depth observation with untrusted and non-finite pixels, unrecorded
    pixels through the silhouette term, a perturbed pose."""
    from paper_1911_13225_b200 import optimize
    g, net, _, intr, _ = _setup(st, "fp64")
    cfg = st.TraceConfig(alpha=1.0, k_samples=k, coarse_start_scale=1)
    dimg = np.array(g["obs_depth"], dtype=np.float64)
    dimg[3, :] = np.inf
    mask = np.ones(dimg.shape, bool)
    mask[:, 5] = False
    obs = [st.Observation("depth", dimg, mask), st.Observation("silhouette", g["obs_sil"])]
    params = np.asarray(g["params"], dtype=np.float64) + np.array([0.01, -0.02, 0.015, 0.02, 0.0, -0.01])
    w = st.LossWeights(depth=3.0, silhouette=0.7)
    a = st.pose_objective(net, g["code"], obs, intr, params, cfg, w)
    monkeypatch.setattr(optimize, "_DEVICE_POSE", False)
    b = st.pose_objective(net, g["code"], obs, intr, params, cfg, w)
    assert abs(a[0] - b[0]) <= 1e-12 * abs(b[0])
    for key in b[1]:
        assert abs(a[1][key] - b[1][key]) <= 1e-12 * abs(b[1][key]) + 1e-15
    np.testing.assert_allclose(a[2], b[2], rtol=1e-10, atol=1e-13)
    assert a[3] == b[3]


def test_pose_objective_device_fp16x3_8x512(st, monkeypatch):
    """The tensor-core decoder through the device pose objective and the host
    path: the same device kernels evaluate the same points."""
    from paper_1911_13225_b200 import optimize
    from paper_1911_13225_b200.workloads import target_code
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    intr = st.Intrinsics(width=64, height=64)
    pose = st.look_at((0.3, 0.4, -2.2))
    cfg = st.TraceConfig(k_samples=3)
    code = target_code(1)
    m = st.render(net, code, intr, pose, cfg, with_normals=False)
    obs = [st.Observation("depth", m.depth), st.Observation("silhouette", m.mask.astype(np.float64))]
    params = pose.params() + np.array([0.02, 0.01, -0.01, 0.0, 0.03, 0.0])
    a = st.pose_objective(net, code, obs, intr, params, cfg, st.LossWeights())
    monkeypatch.setattr(optimize, "_DEVICE_POSE", False)
    b = st.pose_objective(net, code, obs, intr, params, cfg, st.LossWeights())
    assert abs(a[0] - b[0]) <= 1e-9 * abs(b[0])
    np.testing.assert_allclose(a[2], b[2], rtol=1e-6, atol=1e-9)
    assert a[3] == b[3]
    assert np.linalg.norm(a[2]) > 0


def test_recover_pose_device_equals_host_fp32_k3(st, monkeypatch):
    """recover_pose through the device objective and the host path, fp32
    decoder, K = 3, learning-rate decay: the same iterate history."""
    from paper_1911_13225_b200 import optimize
    g, _, obs, intr, _ = _setup(st, "fp64")
    net = st.NeuralField(golden_weights(g), latent_dim=2, precision="fp32")
    cfg = st.TraceConfig(alpha=1.0, k_samples=3, coarse_start_scale=1)
    p0 = st.Pose.from_params(np.asarray(g["params"]) + np.array([0.02, 0.0, -0.01, 0.01, 0.02, 0.0]))
    kw = dict(iters=6, cfg=cfg, lr_decay_every=3)
    best_d, rep_d = st.recover_pose(net, g["code"], obs, intr, p0, **kw)
    monkeypatch.setattr(optimize, "_DEVICE_POSE", False)
    best_h, rep_h = st.recover_pose(net, g["code"], obs, intr, p0, **kw)
    np.testing.assert_allclose(rep_d.losses, rep_h.losses, rtol=1e-9)
    np.testing.assert_allclose(rep_d.grad_norms, rep_h.grad_norms, rtol=1e-6)
    assert rep_d.best_iter == rep_h.best_iter and rep_d.total_queries == rep_h.total_queries
    np.testing.assert_allclose(best_d.params(), best_h.params(), rtol=1e-9, atol=1e-12)
