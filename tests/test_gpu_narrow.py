"""The narrow-decoder march (csrc/mlp_small.cuh; trace.cu k_march_resident /
k_march_small): decoders whose hidden layers are all <= 64 wide -- the
reference's tiny_net (C1, conftest.py:33-39) -- march one ray per thread with
the decoder staged in shared memory, all slots of a level in one cooperative
launch (and, when the level fits the grid, the ray state resident in shared
memory with activations in registers for widths <= 32).  Parity is
the reference's: per-step query counts and ray status exactly, depth to
1e-9 in fp64 (tracer.py:221-252 restated by the oracle)."""
from __future__ import annotations

import numpy as np
import pytest

import sdf_oracle as orc  # noqa: E402  (checker only)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _check(st, net, dec, code, res, eye_k, cfg_kw, prec, exact=True):
    cam = orc.cam_look_at(orc.ring_eye(eye_k, 8), res, res)
    T = orc.trace(lambda p: dec(p, code), cam, orc.Cfg(**cfg_kw))
    r = st.trace(net, code, st.Intrinsics(width=res, height=res), st.Pose(cam.omega, cam.t),
                 st.TraceConfig(**cfg_kw))
    if prec == "fp64" and exact:
        assert r.live_counts == T.live_counts
        assert np.array_equal(r.state.status, T.status)
        hit = T.status == 1
        assert np.max(np.abs(r.state.d[hit] - T.d[hit])) < 1e-9
    else:   # the trajectory band of SURVEY 8c
        band = (T.margin_f < 1e-5) | (T.margin_esc < 1e-6)
        assert not np.any(((r.state.status == 1) != (T.status == 1)) & ~band)
        mism = (r.state.status != T.status) | (r.state.steps != T.steps)
        assert (mism & ~band).sum() <= (2 if prec == "fp64" else 8)
    return T


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("dynamic", [True, False])
def test_tiny_net_trace(st, prec, dynamic):
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision=prec)
    code = rng.normal(0.0, 0.3, 2)
    dec = orc.Decoder(net.weights, 2)
    T = _check(st, net, dec, code, 64, 0, dict(k_samples=3, use_dynamic_mask=dynamic), prec)
    assert (T.status == 1).sum() > 100


@pytest.mark.parametrize("width", [32, 48])
def test_narrow_skip_net_trace(st, width):
    """A 4 x width decoder with a layer-2 skip (the pre-skip layer width-11
    wide): the skip layer's folded code rows + xyz term in the one-ray-per-
    thread path (32: register activations; 48: shared-memory activations)."""
    D = 8
    ws = orc.geometric_init(D, (width,) * 4, 5, skip=2)
    dec = orc.Decoder(ws, D, skip=2)
    net = st.NeuralField(ws, latent_dim=D, precision="fp64", skip=2)
    code = np.random.default_rng(2).normal(0, 0.1, D)
    # fp64 against numpy's BLAS summation order: one ray at its escape test
    # differs by a step, so the band contract rather than exact counts
    T = _check(st, net, dec, code, 64, 1, dict(k_samples=2), "fp64", exact=False)
    assert (T.status == 1).sum() > 100


def test_narrow_widest_and_odd_widths(st):
    """64-wide (the path's limit) and odd widths (the 4-column blocks' tail)."""
    D = 3
    for hidden in ((64, 64, 64), (13, 7, 21)):
        ws = orc.geometric_init(D, hidden, 11)
        dec = orc.Decoder(ws, D)
        net = st.NeuralField(ws, latent_dim=D, precision="fp64")
        code = np.random.default_rng(4).normal(0, 0.1, D)
        _check(st, net, dec, code, 32, 2, dict(k_samples=1), "fp64")


def test_narrow_batched_views_and_shapes(st):
    """Two shapes x two views in one batched trace equal four single traces bit for bit."""
    from paper_1911_13225_b200.tracer import host_result, trace_views
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision="fp64")
    codes = np.stack([rng.normal(0.0, 0.3, 2), rng.normal(0.0, 0.3, 2)])
    views = []
    for k in range(2):
        cam = orc.cam_look_at(orc.ring_eye(k, 8), 64, 64)
        views.append((st.Intrinsics(width=64, height=64), st.Pose(cam.omega, cam.t)))
    cfg = st.TraceConfig(k_samples=3)
    sov = [0, 0, 1, 1]
    dt = trace_views(net, codes, views + views, cfg, shape_of_view=sov)
    for v in range(4):
        one = host_result(trace_views(net, codes[sov[v]], [views[v % 2]], cfg), 0)
        got = host_result(dt, v)
        assert got.live_counts == one.live_counts
        np.testing.assert_array_equal(got.state.d, one.state.d)
        np.testing.assert_array_equal(got.state.status, one.state.status)


def test_tiny_iterate_under_1ms(st):
    """C1 (one 64^2 completion iterate of the tiny net) in <= 1 ms of device
    time, eager and CUDA-graph replayed."""
    import torch
    from paper_1911_13225_b200.shading import device_maps
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision="fp64")
    code = rng.normal(0.0, 0.3, 2)
    intr, pose = st.Intrinsics(width=64, height=64), st.look_at((0.0, 0.0, -2.0))
    cfg = st.TraceConfig(k_samples=3)
    obs = {"depth": device_maps(st.trace_views(net, code + 0.05, [(intr, pose)], cfg))[0]}
    opt = st.LatentOptimizer(net, [(intr, pose)], obs, code[None], cfg, max_iters=64)
    for fn in (opt.step, opt.step_graph):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"C1 iterate {fn.__name__}: {ms:.3f} ms")
        assert ms <= 1.0
