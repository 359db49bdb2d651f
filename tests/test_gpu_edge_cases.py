"""Edge cases the reference tests for this path (test_tracer.py, test_optimize.py,
test_fields.py): all-background views, a camera inside the unit sphere, empty
point sets, the configuration boundaries, and the validation errors -- the GPU
path against the CPU oracle or the reference's documented behaviour."""
from __future__ import annotations

import warnings

import numpy as np
import pytest

import sdf_oracle as orc  # noqa: E402  (checker only)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _tiny(st, prec="fp64"):
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision=prec)
    return net, rng.normal(0.0, 0.3, 2)


def _oracle_trace(net, code, res, pose, **cfg):
    dec = orc.Decoder(net.weights, 2)
    return orc.trace(lambda p: dec(p, code), orc.Cam(res, res, pose.omega, pose.t), orc.Cfg(**cfg))


def test_all_background_view(st):
    """Looking away from the shape: every ray escapes, the depth map is +inf,
    and complete_shape without a silhouette refuses to start
    (optimize.py:160-165, test_optimize.py:163)."""
    net, code = _tiny(st)
    intr, pose = st.Intrinsics(width=32, height=32), st.look_at((0.0, 0.0, -2.0), (0.0, 0.0, -4.0))
    r = st.trace(net, code, intr, pose, st.TraceConfig())
    T = _oracle_trace(net, code, 32, pose)
    assert np.array_equal(r.state.status, T.status)
    assert not np.any(r.state.status == 1)
    assert np.all(np.isinf(st.depth_map(r)))
    obs = [st.Observation("depth", np.full((32, 32), 1.5))]
    with pytest.raises(st.OptimizationError):
        st.complete_shape(net, obs, intr, pose, iters=2)


def test_camera_inside_unit_sphere(st):
    """Camera centre inside the unit sphere: a RuntimeWarning and every ray
    starts at d = 0 (tracer.py:100-102, test_tracer.py:91-98); the march then
    matches the oracle bit for bit."""
    net, code = _tiny(st)
    pose = st.look_at((0.0, 0.0, -0.5))
    with pytest.warns(RuntimeWarning):
        r = st.trace(net, code, st.Intrinsics(width=32, height=32), pose, st.TraceConfig())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        T = _oracle_trace(net, code, 32, pose)
    assert r.live_counts == T.live_counts
    assert np.array_equal(r.state.status, T.status)
    assert np.array_equal(r.state.steps, T.steps)


@pytest.mark.parametrize("prec", ["fp64", "bf16x3"])
def test_empty_point_set(st, prec):
    """Zero points evaluate to an empty array and a zero code gradient."""
    import torch
    if prec == "fp64":
        net, code = _tiny(st)
    else:
        net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
        code = np.zeros(256)
    assert net.evaluate(np.zeros((0, 3)), code).shape == (0,)
    f, gc, gp = net.vjp_device(torch.zeros((0, 3), dtype=torch.float64), code,
                               torch.zeros(0, dtype=torch.float64))
    assert f.numel() == 0 and float(gc.abs().sum()) == 0.0 and gp.numel() == 0


@pytest.mark.parametrize("max_steps,k", [(1, 1), (2, 16), (100, 16), (7, 1)])
def test_config_boundaries_bitexact_fp64(st, max_steps, k):
    """max_steps down to 1 and k_samples at both ends (1, 16): the fp64 GPU
    march equals the oracle -- counts, status and steps exactly, distances to
    the last ulp (FMA contraction differs from numpy)."""
    net, code = _tiny(st)
    pose = st.look_at((0.0, 0.0, -2.0))
    cfg = st.TraceConfig(max_steps=max_steps, k_samples=k)
    r = st.trace(net, code, st.Intrinsics(width=64, height=64), pose, cfg)
    T = _oracle_trace(net, code, 64, pose, max_steps=max_steps, k_samples=k)
    assert r.live_counts == T.live_counts and r.total_queries == T.total_queries
    assert np.array_equal(r.state.status, T.status) and np.array_equal(r.state.steps, T.steps)
    np.testing.assert_allclose(r.state.d, T.d, rtol=1e-14, atol=0)
    fin = np.isfinite(T.tk_a)
    assert np.array_equal(np.isfinite(r.state.topk_absf), fin)
    np.testing.assert_allclose(r.state.topk_absf[fin], T.tk_a[fin], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("w,h,cs", [(48, 20, 4), (37, 23, 1), (64, 8, 2), (12, 100, 4)])
def test_nonsquare_ragged_views_bitexact_fp64(st, w, h, cs):
    """Non-square views whose ray counts are not a multiple of the 128-row
    tile, with and without coarse-to-fine (camera.py:25-61 takes fx from the
    width only; tracer.py:225-250 splits a w/cs x h/cs grid): the fp64 GPU march
    equals the oracle exactly, and the depth map is laid out height x width."""
    net, code = _tiny(st)
    pose = st.look_at((0.3, 0.2, -2.0))
    cfg = st.TraceConfig(coarse_start_scale=cs, k_samples=3)
    r = st.trace(net, code, st.Intrinsics(width=w, height=h), pose, cfg)
    dec = orc.Decoder(net.weights, 2)
    T = orc.trace(lambda p: dec(p, code), orc.Cam(w, h, pose.omega, pose.t),
                  orc.Cfg(coarse_start_scale=cs, k_samples=3))
    assert r.live_counts == T.live_counts and r.total_queries == T.total_queries
    assert np.array_equal(r.state.status, T.status) and np.array_equal(r.state.steps, T.steps)
    np.testing.assert_allclose(r.state.d, T.d, rtol=1e-14, atol=0)
    assert st.depth_map(r).shape == (h, w)
    assert np.any(r.state.status == 1) and np.any(r.state.status != 1)


def test_validation_errors(st):
    """Configuration and shape errors raise ValueError before any launch."""
    net, code = _tiny(st)
    pose = st.look_at((0.0, 0.0, -2.0))
    with pytest.raises(ValueError):
        st.TraceConfig(k_samples=0)
    with pytest.raises(ValueError):
        st.TraceConfig(alpha=2.0)
    with pytest.raises(ValueError):   # 30 is not divisible by the coarse scale 4
        st.trace(net, code, st.Intrinsics(width=30, height=32), pose, st.TraceConfig())
    with pytest.raises(ValueError):   # one trace call, one resolution
        st.trace_views(net, code, [(st.Intrinsics(width=32, height=32), pose),
                                   (st.Intrinsics(width=64, height=64), pose)])
    with pytest.raises(ValueError):   # the field expects a latent code
        net.evaluate(np.zeros((4, 3)), None)
    with pytest.raises(ValueError):
        net.evaluate(np.zeros((4, 3)), np.zeros(3))


def test_concurrent_traces_on_two_streams_match_sequential(st):
    """One immutable decoder handle, two traces (different codes and views)
    enqueued on two CUDA streams at once: per-call workspaces keep them apart,
    and each result equals the same trace run alone (include/dist.h: handles are
    safe across streams; consecutive march steps use programmatic dependent
    launch within a stream)."""
    import torch
    from paper_1911_13225_b200.workloads import ring_views
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    cfg = st.TraceConfig(k_samples=3)
    rng = np.random.default_rng(11)
    jobs = [(rng.normal(0, 0.1, 256), ring_views(4, 128, first=0, total=8, stride=2)),
            (rng.normal(0, 0.1, 256), ring_views(4, 128, first=1, total=8, stride=2))]

    def grab(dt):
        return (dt.status.cpu().numpy(), dt.steps.cpu().numpy(), dt.d.cpu().numpy(),
                dt.topk_f.cpu().numpy())

    alone = []
    for z, views in jobs:
        alone.append(grab(st.trace_views(net, z, views, cfg)))
        torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [None, None]
    for rep in range(2):
        for k, (z, views) in enumerate(jobs):
            with torch.cuda.stream(streams[k]):
                out[k] = st.trace_views(net, z, views, cfg)
        torch.cuda.synchronize()
        for k in range(2):
            got = grab(out[k])
            for a, b in zip(got, alone[k]):
                np.testing.assert_array_equal(a, b)


# --- non-finite fields on the decoder paths (tracer.py:170-176) -------------------

@pytest.mark.parametrize("prec", ["fp64", "fp16x3"])
def test_nan_code_exhausts_its_views_only(st, prec):
    """Two shapes in one batched trace, one code NaN: every ray of the NaN
    shape's view exhausts at its first query (NaN propagates through the ReLU
    layers as np.maximum does, fields.py:239-247) with its nan_count, while the
    other view equals its trace alone -- on the SIMT and the tcgen05 march."""
    from paper_1911_13225_b200.tracer import host_result
    from paper_1911_13225_b200.workloads import ring_views
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    z = np.random.default_rng(1).normal(0.0, 0.1, (2, 256))
    z[1, 3] = np.nan
    views = ring_views(2, 32)
    cfg = st.TraceConfig(k_samples=3)
    dt = st.trace_views(net, z, views, cfg, shape_of_view=[0, 1])
    bad = host_result(dt, 1)
    hit0 = bad.state.steps > 0
    assert hit0.any()
    assert np.all(bad.state.status[hit0] == st.EXHAUSTED) and np.all(np.isnan(bad.state.b[hit0]))
    assert np.all(bad.state.steps[hit0] == 1) and bad.live_counts == [int(dt.stats()["nan_count"])]
    good = host_result(dt, 0)
    alone = host_result(st.trace_views(net, z[0], views[:1], cfg), 0)
    for k in ("status", "steps", "d"):
        np.testing.assert_array_equal(getattr(good.state, k), getattr(alone.state, k), err_msg=k)
    assert good.live_counts == alone.live_counts


@pytest.mark.parametrize("prec", ["fp16x3", "bf16x3"])
def test_dynamic_mask_off_on_tensor_cores(st, prec):
    """tracer.py:158-168 on the tcgen05 march: without the live mask the whole
    grid is queried and dead rays' values discarded -- the marched values are
    bit-identical, only the query count grows (test_tracer.py:260-270)."""
    g = __import__("conftest").load_golden("geo64.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, int(g["seed"]), precision=prec)
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"])
    on = st.trace(net, g["code"], intr, pose, st.TraceConfig(k_samples=3))
    off = st.trace(net, g["code"], intr, pose, st.TraceConfig(k_samples=3, use_dynamic_mask=False))
    for k in ("status", "steps", "d", "b", "topk_d", "topk_f"):
        np.testing.assert_array_equal(getattr(on.state, k), getattr(off.state, k), err_msg=k)
    assert off.total_queries > on.total_queries
    # the reference's count without the mask: every ray of the level, each step
    assert all(c in (16 * 16, 32 * 32, 64 * 64) for c in off.live_counts)


def test_tensor_core_precision_refuses_unsupported_shapes(st):
    """A tensor-core precision on a decoder the tcgen05 kernels cannot tile
    (a skip at the top hidden layer, a first hidden layer narrower than 512)
    raises instead of silently running SIMT."""
    with pytest.raises(ValueError):   # skip at the top hidden layer
        st.NeuralField.geometric(256, (512,) * 8, 0, skip=7, precision="fp16x3").handle()
    with pytest.raises(ValueError):   # a 256-wide first hidden layer
        st.NeuralField.geometric(64, (256,) * 4, 0, precision="bf16x3").handle()
    st.NeuralField.geometric(256, (512,) * 8, 0, skip=7, precision="fp32").handle()
    st.NeuralField.geometric(256, (512,) * 8, 0, skip=4, precision="fp16x3").handle()   # DeepSDF: tiled


@pytest.mark.parametrize("prec", ["fp64", "fp16x3"])
def test_graph_replayed_iterates_equal_eager(st, prec):
    """LatentOptimizer.step_graph (one CUDA graph per iterate, the Adam
    iteration index on the device) gives the eager iterates bit for bit: codes,
    loss history and best iterate."""
    import time
    import torch
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    if prec == "fp64":
        net, code = _tiny(st)
        views = [(st.Intrinsics(width=64, height=64), st.look_at((0.0, 0.0, -2.0)))]
        obs = render_depth_observations(net, code + 0.05, views, st.TraceConfig(k_samples=3))
        z0 = np.zeros((1, 2))
    else:
        net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
        views = ring_views(2, 64)
        obs = render_depth_observations(net, target_code(1), views, st.TraceConfig(k_samples=3))
        z0 = np.zeros((1, 256))
    cfg = st.TraceConfig(k_samples=3)
    runs = {}
    for mode in ("eager", "graph"):
        opt = st.LatentOptimizer(net, views, {"depth": obs}, z0, cfg, max_iters=12)
        codes = []
        for _ in range(6):
            (opt.step if mode == "eager" else opt.step_graph)()
            codes.append(opt.code.cpu().numpy().copy())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(6):
            (opt.step if mode == "eager" else opt.step_graph)()
        torch.cuda.synchronize()
        runs[mode] = (np.stack(codes), opt.losses(), int(opt.best_iter[0].item()),
                      (time.perf_counter() - t0) / 6 * 1e3)
    assert np.array_equal(runs["eager"][0], runs["graph"][0])
    assert np.array_equal(runs["eager"][1], runs["graph"][1])
    assert runs["eager"][2] == runs["graph"][2]
    print(f"{prec}: ms per iterate eager {runs['eager'][3]:.3f} graph {runs['graph'][3]:.3f}")
