"""photometric warp kernels and reconstruct_multiview vs the reference."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_weights, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _views(st, g):
    intr = st.Intrinsics(width=24, height=24)
    return intr, [st.look_at(e) for e in g["eyes"]]


def test_photometric_loss_and_visibility_vs_reference(st):
    g = load_golden("multiview24.npz")
    intr, poses = _views(st, g)
    d, im = g["depths"], g["images"]
    l, dz = st.photometric_loss(d[0], im[0], intr, poses[0], im[1], intr, poses[1], d[1])
    assert abs(l - float(g["ph_loss"])) < 1e-12
    np.testing.assert_allclose(dz, g["ph_dz"], rtol=1e-9, atol=1e-12)
    vis = st.visibility_mask(d[0], intr, poses[0], d[1], intr, poses[1])
    assert np.array_equal(vis, g["ph_vis"])


def test_reconstruct_multiview_history_vs_reference(st):
    g = load_golden("multiview24.npz")
    intr, poses = _views(st, g)
    net = st.NeuralField(golden_weights(g), latent_dim=2, precision="fp64")
    cfg = st.TraceConfig(alpha=1.0, k_samples=1, coarse_start_scale=1)
    best, rep = st.reconstruct_multiview(net, list(g["images"]), [(intr, p) for p in poses],
                                         code0=g["code"] + 0.1, iters=3, views_per_iter=2,
                                         cfg=cfg, seed=1)
    np.testing.assert_allclose(rep.losses, g["mv_losses"], rtol=1e-9, atol=1e-12)
    assert rep.best_iter == int(g["mv_best_iter"])
    np.testing.assert_allclose(best, g["mv_best"], rtol=1e-9, atol=1e-12)


def test_reconstruct_multiview_device_loop_equals_host_loop(st, monkeypatch):
    """The device-resident iterate (dist_photo_heads/depth/seeds, one reverse
    sweep over all views, Adam with the best-iterate record on the device)
    against the per-view host loop (HeadBundle per view) on the reference's
    multiview golden scene: same losses, terms, best iterate and code up to
    summation order, and no host round trip inside the loop."""
    from paper_1911_13225_b200 import _lib, optimize
    g = load_golden("multiview24.npz")
    intr, poses = _views(st, g)
    net = st.NeuralField(golden_weights(g), latent_dim=2, precision="fp64")
    cfg = st.TraceConfig(alpha=1.0, k_samples=1, coarse_start_scale=1)
    kw = dict(code0=g["code"] + 0.1, iters=5, views_per_iter=3, cfg=cfg, seed=4)
    images, views = list(g["images"]), [(intr, p) for p in poses]
    n0 = _lib.lib().dist_launch_count()
    best_d, rep_d = st.reconstruct_multiview(net, images, views, **kw)
    assert _lib.lib().dist_launch_count() > n0
    monkeypatch.setattr(optimize, "_DEVICE_MULTIVIEW", False)
    best_h, rep_h = st.reconstruct_multiview(net, images, views, **kw)
    np.testing.assert_allclose(rep_d.losses, rep_h.losses, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose([t["photometric"] for t in rep_d.terms],
                               [t["photometric"] for t in rep_h.terms], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(rep_d.grad_norms, rep_h.grad_norms, rtol=1e-10, atol=1e-15)
    assert rep_d.best_iter == rep_h.best_iter
    assert rep_d.total_queries == rep_h.total_queries
    np.testing.assert_allclose(best_d, best_h, rtol=1e-12, atol=1e-15)


def test_attribute_field_and_map_vs_reference(st):
    """sigmoid-head colour MLP at hit points."""
    g = load_golden("attr32.npz")
    aw = [(g[f"AW{i}"], g[f"Ab{i}"]) for i in range(int(g["An_layers"]))]
    attr = st.AttributeField(aw, shape_dim=2, attr_dim=1)
    np.testing.assert_allclose(attr.evaluate(g["pts"], g["acode"]), g["vals"], rtol=0, atol=1e-13)
    net = st.NeuralField(golden_weights(g), latent_dim=2)
    maps = st.render(net, g["code"], st.Intrinsics(width=32, height=32), st.look_at((0.0, 0.0, -2.0)),
                     st.TraceConfig(), attr_field=attr, attr_code=g["acode"])
    np.testing.assert_allclose(maps.attribute, g["amap"], rtol=0, atol=1e-12)


def test_reconstruct_multiview_device_loop_tensor_core_decoder(st, monkeypatch):
    """The device iterate on the 8x512 fp16x3 decoder (K = 3 records, the
    default coarse-to-fine start) against the per-view host loop: the same
    kernels evaluate the same sample points, so the histories agree to
    summation order."""
    from paper_1911_13225_b200 import optimize
    from paper_1911_13225_b200.workloads import ring_views, target_code
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    views = ring_views(6, 64)
    yy, xx = np.mgrid[0:64, 0:64] / 64.0
    images = [np.stack([0.5 + 0.5 * np.sin(9 * xx + k), 0.5 + 0.5 * np.cos(7 * yy - k), xx * yy], axis=2)
              for k in range(6)]
    kw = dict(code0=target_code(1) * 0.9, iters=3, views_per_iter=3, cfg=st.TraceConfig(k_samples=3), seed=2)
    best_d, rep_d = st.reconstruct_multiview(net, images, views, **kw)
    monkeypatch.setattr(optimize, "_DEVICE_MULTIVIEW", False)
    best_h, rep_h = st.reconstruct_multiview(net, images, views, **kw)
    np.testing.assert_allclose(rep_d.losses, rep_h.losses, rtol=1e-9)
    np.testing.assert_allclose(best_d, best_h, rtol=1e-7, atol=1e-12)
    assert rep_d.best_iter == rep_h.best_iter and rep_d.total_queries == rep_h.total_queries
    assert min(rep_d.grad_norms) > 0


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_attribute_channels_one_hidden_stack(st, prec):
    """dist_eval_channels (the hidden stack once, then the m heads) equals each
    channel's own single-output decoder bit for bit, with a shape+attribute
    code and a 3-channel head."""
    rng = np.random.default_rng(5)
    attr = st.AttributeField.init(shape_dim=3, attr_dim=2, hidden=(32, 48, 32), out_dim=3, rng=rng,
                                  precision=prec)
    pts = rng.uniform(-1, 1, (1000, 3))
    code = rng.normal(0, 0.3, 5)
    got = attr.evaluate(pts, code)
    ref = np.stack([ch.evaluate(pts, code) for ch in attr._channels], axis=1)
    assert got.shape == (1000, 3)
    np.testing.assert_array_equal(got, ref)


def test_reconstruct_multiview_device_zero_iters_and_all_views(st):
    """Edge cases of the device loop: no iterate returns the start code; every
    view sampled each iterate (views_per_iter >= n_views)."""
    g = load_golden("multiview24.npz")
    intr, poses = _views(st, g)
    net = st.NeuralField(golden_weights(g), latent_dim=2, precision="fp64")
    cfg = st.TraceConfig(alpha=1.0, k_samples=1, coarse_start_scale=1)
    views = [(intr, p) for p in poses]
    best, rep = st.reconstruct_multiview(net, list(g["images"]), views, code0=g["code"] + 0.1, iters=0,
                                         cfg=cfg)
    np.testing.assert_array_equal(best, g["code"] + 0.1)
    assert rep.losses == [] and rep.best_iter == -1
    best, rep = st.reconstruct_multiview(net, list(g["images"]), views, code0=g["code"] + 0.1, iters=2,
                                         views_per_iter=len(views) + 3, cfg=cfg)
    assert len(rep.losses) == 2 and np.all(np.isfinite(rep.losses)) and rep.total_queries > 0
