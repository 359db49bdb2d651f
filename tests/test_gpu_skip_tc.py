"""The DeepSDF layout on the tensor cores (north_star: "8x512 MLP with the
latent concatenated to xyz and the layer-4 skip"): layer 4 consumes
concat(h, code, xyz) (the oracle's Decoder(skip=4), after
fields.py:239-247).  The tcgen05 kernels fold the skip layer's code rows into a
per-shape bias and its xyz rows into the epilogue, pad the 253-wide layer 3 to
512, and take the skip layer's own column sums in the head kernel's backward.
Checked in fp16x3 against the fp64 oracle: decoder values, trace, normals,
the fused objective's gradient and the taped vjp.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import sdf_oracle as orc  # noqa: E402  (checker only)

pytestmark = pytest.mark.gpu

SKIP, D = 4, 256


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


@pytest.fixture(scope="module")
def nets(st):
    ws = orc.geometric_init(D, (512,) * 8, 0, skip=SKIP)
    dec = orc.Decoder(ws, D, skip=SKIP)
    f16 = st.NeuralField(ws, latent_dim=D, precision="fp16x3", skip=SKIP)
    return ws, dec, f16


def _code(seed=1):
    return np.random.default_rng(seed).normal(0.0, 0.1, D)


def test_skip_decoder_eval_fp16x3(st, nets):
    ws, dec, f16 = nets
    assert [w.shape for w, _ in ws][SKIP - 1:SKIP + 1] == [(512, 253), (512, 512)]
    pts = np.random.default_rng(0).uniform(-0.9, 0.9, (20000, 3))
    ref = dec(pts, _code())
    got = f16.evaluate(pts, _code())
    assert np.max(np.abs(got - ref)) < 2e-6
    assert abs(np.mean(got - ref)) < 2e-7           # the calibrated head gain removes the bias
    g = f16.head_gain()[0]
    assert 1.0 < g < 1.0001


def test_skip_decoder_trace_fp16x3_vs_oracle(st, nets):
    ws, dec, f16 = nets
    res, code = 64, _code()
    cam = orc.cam_look_at(orc.ring_eye(1, 8), res, res)
    T = orc.trace(lambda p: dec(p, code), cam, orc.Cfg(k_samples=3))
    r = st.trace(f16, code, st.Intrinsics(width=res, height=res), st.Pose(cam.omega, cam.t),
                 st.TraceConfig(k_samples=3))
    assert (T.status == 1).sum() > 500
    band = (T.margin_f < 1e-5) | (T.margin_esc < 1e-6)
    assert not np.any(((r.state.status == 1) != (T.status == 1)) & ~band)
    mism = (r.state.status != T.status) | (r.state.steps != T.steps)
    assert (mism & ~band).sum() <= 1
    both = (r.state.status == 1) & (T.status == 1) & ~mism
    assert np.max(np.abs(r.state.d[both] - T.d[both]) / T.d[both]) <= 1e-4
    # normals at the traced points: the (mid, diff) probes through the skip layer
    from paper_1911_13225_b200.shading import device_normals
    n16 = device_normals(r.device).cpu().numpy().reshape(-1, 3)
    r.device.field = f16.with_precision("fp64")
    n64 = device_normals(r.device).cpu().numpy().reshape(-1, 3)
    hit = np.linalg.norm(n64, axis=1) > 0
    assert hit.sum() > 500 and np.max(np.linalg.norm(n16 - n64, axis=1)[hit]) < 1e-4


def test_skip_decoder_objective_fp16x3_vs_oracle(st, nets):
    ws, dec, f16 = nets
    res = 64
    cam = orc.cam_look_at(orc.ring_eye(1, 8), res, res)
    ocfg = orc.Cfg(k_samples=3)
    obs = orc.depth_map(orc.trace(lambda p: dec(p, _code(1)), cam, ocfg), ocfg)
    sil = np.isfinite(obs).astype(np.float64)
    code = _code(2)
    tot_o, _, g_o, _, _, _ = orc.objective(dec, code, cam, ocfg, orc.Weights(), depth=obs, silhouette=sil)
    tot, _, g, _, _ = st.completion_objective(
        f16, code, [st.Observation("depth", obs), st.Observation("silhouette", sil)],
        st.Intrinsics(width=res, height=res), st.Pose(cam.omega, cam.t), st.TraceConfig(k_samples=3),
        st.LossWeights())
    assert abs(tot - tot_o) <= 1e-3 * abs(tot_o)
    assert np.linalg.norm(g - g_o) / np.linalg.norm(g_o) < 1e-3


def test_skip_decoder_vjp_fp16x3_vs_oracle(st, nets):
    """dist_eval_vjp on the tensor cores: the code gradient (layer 0 + the skip
    layer's code rows) and the point gradient (both xyz inputs)."""
    ws, dec, f16 = nets
    pts = np.random.default_rng(3).uniform(-0.7, 0.7, (3000, 3))
    seed = np.abs(np.random.default_rng(4).standard_normal(3000)) * 1e-3   # coherent, loss-like
    code = _code()
    _, gc, gp = f16.vjp_device(torch.from_numpy(pts), code, torch.from_numpy(seed))
    ref = dec.backward(pts, code, seed)
    gc = gc.cpu().numpy()[0]
    assert np.linalg.norm(gc - ref["code"]) / np.linalg.norm(ref["code"]) < 1e-3
    gp = gp.cpu().numpy()
    assert np.linalg.norm(gp - ref["points"]) / np.linalg.norm(ref["points"]) < 2e-3


def test_skip_batched_shapes_and_record(st, nets):
    """Two shapes in one optimiser with the ReLU-mask record (backward-only
    head tiles through the skip layer) equal independent optimisers bit for bit."""
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views
    ws, dec, f16 = nets
    cfg = st.TraceConfig(k_samples=3)
    views = ring_views(2, 64)
    obs = [render_depth_observations(f16, _code(s + 5), views[s:s + 1], cfg).cpu().numpy() for s in range(2)]
    z0 = np.stack([np.full(D, 0.01), np.full(D, -0.01)])
    both = st.LatentOptimizer(f16, views, {"depth": np.concatenate(obs)}, z0, cfg, shape_of_view=[0, 1],
                              max_iters=2, relu_masks=True)
    both.step()
    both.step()
    for s in range(2):
        one = st.LatentOptimizer(f16, views[s:s + 1], {"depth": obs[s]}, z0[s:s + 1], cfg, max_iters=2,
                                 relu_masks=True)
        one.step()
        one.step()
        np.testing.assert_array_equal(both.code.cpu().numpy()[s], one.code.cpu().numpy()[0])
    assert np.all(np.isfinite(both.code.cpu().numpy()))
