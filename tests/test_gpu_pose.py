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
