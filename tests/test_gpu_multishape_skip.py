"""Multi-shape batching (C5 pattern: several latents x views in one trace and one
objective) and the DeepSDF skip-layer layout, against the oracle."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import sdf_oracle as orc  # noqa: E402  (checker only)


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("bf16x3", 2e-3), ("fp16x3", 2e-3)])
def test_two_shapes_two_views_each(st, prec, tol):
    res, S, VPS = 32, 2, 2
    rng = np.random.default_rng(5)
    ws = orc.geometric_init(256, (512,) * 8, 0)
    dec = orc.Decoder(ws, 256)
    codes = rng.normal(0, 0.1, (S, 256))
    targets = codes + rng.normal(0, 0.05, (S, 256))
    views, sov, obs = [], [], []
    cfg = orc.Cfg(k_samples=3)
    for s in range(S):
        for k in range(VPS):
            cam = orc.cam_look_at(orc.ring_eye(k + 2 * s, 8), res, res)
            views.append((st.Intrinsics(width=res, height=res), st.Pose(cam.omega, cam.t)))
            sov.append(s)
            obs.append(orc.depth_map(orc.trace(lambda p: dec(p, targets[s]), cam, cfg), cfg))
    net = st.NeuralField(ws, latent_dim=256, precision=prec)
    opt = st.LatentOptimizer(net, views, {"depth": np.stack(obs)}, codes, st.TraceConfig(k_samples=3),
                             shape_of_view=sov)
    opt.objective()
    grad = opt.grad.cpu().numpy()
    terms = opt.shape_terms.cpu().numpy()
    for s in range(S):
        g_ref = np.zeros(256)
        tot_ref = 0.0
        for v in range(len(views)):
            if sov[v] != s:
                continue
            cam = orc.Cam(res, res, views[v][1].omega, views[v][1].t)
            t, _, g, _, _, _ = orc.objective(dec, codes[s], cam, cfg, orc.Weights(latent=0.0),
                                             depth=obs[v])
            tot_ref += t
            g_ref += g
        g_ref += 2.0 * codes[s]
        tot_ref += float(codes[s] @ codes[s])
        assert np.linalg.norm(grad[s] - g_ref) / np.linalg.norm(g_ref) < tol, s
        assert abs(terms[s, 0] - tot_ref) < tol * abs(tot_ref), s


def test_deepsdf_skip_layout_fp64_vs_oracle(st):
    D, res = 16, 32
    ws = orc.geometric_init(D, (128,) * 6, 3, skip=3)
    dec = orc.Decoder(ws, D, skip=3)
    code = np.random.default_rng(2).normal(0, 0.1, D)
    net = st.NeuralField(ws, latent_dim=D, precision="fp64", skip=3)
    pts = np.random.default_rng(3).uniform(-0.8, 0.8, (300, 3))
    np.testing.assert_allclose(net.evaluate(pts, code), dec(pts, code), rtol=0, atol=1e-12)
    import torch
    seed = np.random.default_rng(4).standard_normal(300)
    _, gc, gp = net.vjp_device(torch.from_numpy(pts), code, torch.from_numpy(seed))
    ref = dec.backward(pts, code, seed)
    np.testing.assert_allclose(gc.cpu().numpy()[0], ref["code"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(gp.cpu().numpy(), ref["points"], rtol=1e-9, atol=1e-12)
    cam = orc.cam_look_at(orc.ring_eye(1, 8), res, res)
    T = orc.trace(lambda p: dec(p, code), cam, orc.Cfg(k_samples=3))
    r = st.trace(net, code, st.Intrinsics(width=res, height=res), st.Pose(cam.omega, cam.t),
                 st.TraceConfig(k_samples=3))
    assert r.live_counts == T.live_counts
    assert np.array_equal(r.state.status, T.status)
