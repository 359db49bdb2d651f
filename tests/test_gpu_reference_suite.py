"""The reference's own hot-path tests, restated against the drop-in.

Each test follows one test of /root/reference/pkg/tests (cited by file:line)
with the same fixtures (`small_camera` 32^2 from (0,0,-2), `tiny_net`,
conftest.py:15-39), assertions and tolerances, run through this package's
public API: analytic and fake fields go through the plugin seam (trace of a
duck-typed field: the march on the device, the field's own evaluate per
step), the tiny latent net through the device decoder (fp64).
"""
from __future__ import annotations

import numpy as np
import pytest

from analytic_fields import NanField, Plane, Sphere, sphere_depth_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


@pytest.fixture(scope="module")
def small_camera(st):
    return st.Intrinsics(width=32, height=32), st.look_at((0.0, 0.0, -2.0))


@pytest.fixture(scope="module")
def tiny_net(st):
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision="fp64")
    return net, rng.normal(0.0, 0.3, 2)


def _plain(st, **kw):
    return st.TraceConfig(**{"alpha": 1.0, "coarse_start_scale": 1, **kw})


def _one_ray_cam(st):
    """test_tracer.py:21-24: one +z ray from (0,0,-2), the pixel on-axis."""
    return (st.Intrinsics(focal_mm=1.0, sensor_mm=1.0, width=1, height=1),
            st.Pose(np.zeros(3), np.array([0.0, 0.0, 2.0])))


FRONT = dict(normal=(0.0, 0.0, -1.0), offset=-0.3)   # test_tracer.py:36


# --- tracer (pkg/tests/test_tracer.py) --------------------------------------

def test_march_step_update_rule_exact(st):
    """test_tracer.py:103-113 (one step: max_steps=1)."""
    intr, pose = _one_ray_cam(st)
    r = st.trace(Plane(**FRONT), None, intr, pose, st.TraceConfig(alpha=1.5, coarse_start_scale=1,
                                                                     max_steps=1))
    assert r.live_counts == [1] and r.nan_count == 0
    assert r.state.b[0] == 1.3
    assert r.state.d[0] == 1.0 + 1.5 * 1.3
    assert r.state.steps[0] == 1


def test_unit_alpha_head_on_plane_converges_in_two_queries(st):
    """test_tracer.py:116-127."""
    intr, pose = _one_ray_cam(st)
    r = st.trace(Plane(**FRONT), None, intr, pose, _plain(st))
    assert r.state.status[0] == st.CONVERGED and r.state.steps[0] == 2
    assert r.state.b[0] == pytest.approx(0.0, abs=1e-15)
    assert r.state.d[0] == pytest.approx(2.3, abs=1e-15)
    assert r.total_queries == 2


def test_convergence_check_runs_after_the_advance(st):
    """test_tracer.py:130-142: the converging query still moves the ray by
    alpha * b (the record keeps that query's d and f)."""
    intr, pose = _one_ray_cam(st)
    r = st.trace(Plane(**FRONT), None, intr, pose,
                 st.TraceConfig(alpha=1.5, epsilon=1e-2, coarse_start_scale=1))
    s = r.state
    assert s.status[0] == st.CONVERGED and s.b[0] != 0.0
    assert s.topk_f[0, 0] == s.b[0]
    assert s.d[0] == s.topk_d[0, 0] + 1.5 * s.b[0]


def test_dead_rays_stay_frozen(st, small_camera):
    """test_tracer.py:151-169: a ray's (d, steps) never change after it stops."""
    intr, pose = small_camera
    short = st.trace(Sphere(0.5), None, intr, pose, _plain(st, max_steps=8)).state
    full = st.trace(Sphere(0.5), None, intr, pose, _plain(st)).state
    stopped = (short.status == st.CONVERGED) | (short.status == st.ESCAPED)
    assert stopped.sum() > 100
    assert np.array_equal(full.d[stopped], short.d[stopped])
    assert np.array_equal(full.steps[stopped], short.steps[stopped])
    assert np.array_equal(full.status[stopped], short.status[stopped])


def test_nan_field_exhausts_rays(st):
    """test_tracer.py:172-184."""
    intr, pose = _one_ray_cam(st)
    r = st.trace(NanField(), None, intr, pose, st.TraceConfig(coarse_start_scale=1))
    assert r.nan_count > 0
    assert r.state.status[0] == st.EXHAUSTED
    assert np.isnan(r.state.b[0])


def test_partial_nan_field_matches_oracle(st, small_camera):
    """NaN on half the scene: exactly those rays exhaust, with the oracle's
    nan_count, live counts and states (tracer.py:170-176)."""
    import sdf_oracle as orc
    intr, pose = small_camera
    field = NanField(x_nan=0.1, base=Sphere(0.5))
    cfg = st.TraceConfig(k_samples=3)
    r = st.trace(field, None, intr, pose, cfg)
    T = orc.trace(lambda p: field.evaluate(p), orc.Cam(32, 32, pose.omega, pose.t), orc.Cfg(k_samples=3))
    assert r.nan_count == T.nan_count > 0
    assert r.live_counts == T.live_counts
    assert np.array_equal(r.state.status, T.status) and np.array_equal(r.state.steps, T.steps)
    assert np.array_equal(np.isnan(r.state.b), np.isnan(T.b))
    ok = ~np.isnan(T.b)
    np.testing.assert_allclose(r.state.d[ok], T.d[ok], rtol=1e-12, atol=0)


def test_sphere_depth_matches_quadratic_oracle(st, small_camera):
    """test_tracer.py:190-208."""
    intr, pose = small_camera
    plain = _plain(st)
    result = st.trace(Sphere(0.5), None, intr, pose, plain)
    depth = st.depth_map(result)
    ref = sphere_depth_image(intr, pose, 0.5)
    both = np.isfinite(depth) & np.isfinite(ref)
    assert both.sum() > 100
    err = np.abs(depth[both] - ref[both])
    assert np.median(err) < plain.epsilon
    pts, rows = st.surface_points(result)
    vn = np.abs(np.einsum("ij,ij->i", pts / np.linalg.norm(pts, axis=1, keepdims=True),
                          result.state.bundle.dirs[rows]))
    flat = np.zeros(intr.height * intr.width)
    flat[result.state.bundle.pixels[rows, 1] * intr.width + result.state.bundle.pixels[rows, 0]] = vn
    assert np.all(err * flat.reshape(depth.shape)[both] < 3 * plain.epsilon)
    # test_tracer.py:211-217: the mask agrees with the quadratic away from the limb
    assert (np.isfinite(depth) != np.isfinite(ref)).mean() < 0.02


def test_recorded_samples_replay_bitwise(st, small_camera):
    """test_tracer.py:220-236."""
    intr, pose = small_camera
    field = Sphere(0.5)
    cfg = st.TraceConfig(alpha=1.5, coarse_start_scale=1, k_samples=3)
    s = st.trace(field, None, intr, pose, cfg).state
    rows = np.nonzero(s.status == st.CONVERGED)[0][:50]
    assert rows.size == 50
    for i in rows:
        for k in range(3):
            if not np.isfinite(s.topk_absf[i, k]):
                continue
            p = s.bundle.origin + s.topk_d[i, k] * s.bundle.dirs[i]
            assert field.evaluate(p[None, :])[0] == s.topk_f[i, k]
    assert np.all(np.diff(s.topk_absf[rows], axis=1) >= 0.0)
    assert np.all(s.topk_absf[rows, 0] < cfg.epsilon)


def test_query_audit_and_max_steps(st, small_camera):
    """test_tracer.py:239-257."""
    intr, pose = small_camera
    r = st.trace(Sphere(0.5), None, intr, pose, st.TraceConfig(alpha=1.0))
    assert sum(r.live_counts) == r.total_queries > 0
    r1 = st.trace(Sphere(0.5), None, intr, pose, _plain(st, max_steps=1))
    s = r1.state.status
    assert not (s == st.CONVERGED).any() and (s == st.EXHAUSTED).any()
    assert np.all(r1.state.steps[s == st.EXHAUSTED] == 1)


def test_dynamic_mask_changes_cost_not_values(st, small_camera):
    """test_tracer.py:260-270, through the plugin seam and the device decoder."""
    intr, pose = small_camera
    on = st.trace(Sphere(0.5), None, intr, pose, _plain(st))
    off = st.trace(Sphere(0.5), None, intr, pose, _plain(st, use_dynamic_mask=False))
    assert np.array_equal(on.state.d, off.state.d)
    assert np.array_equal(on.state.status, off.state.status)
    assert off.total_queries > on.total_queries


def test_coarse_to_fine_saves_queries(st, small_camera):
    """test_tracer.py:273-287."""
    from scipy import ndimage
    intr, pose = small_camera
    plain = st.trace(Sphere(0.5), None, intr, pose, _plain(st))
    coarse = st.trace(Sphere(0.5), None, intr, pose, st.TraceConfig(alpha=1.0, coarse_start_scale=4))
    assert coarse.total_queries < plain.total_queries
    dp, dc = st.depth_map(plain), st.depth_map(coarse)
    both = np.isfinite(dp) & np.isfinite(dc)
    interior = ndimage.binary_erosion(both)
    assert interior.sum() > 50
    assert np.max(np.abs(dp[interior] - dc[interior])) < 5 * 5e-5
    assert (np.isfinite(dp) != np.isfinite(dc)).mean() < 0.02


def test_overshoot_records_negative_samples(st, small_camera):
    """test_tracer.py:290-302."""
    intr, pose = small_camera

    def neg_frac(alpha):
        r = st.trace(Sphere(0.5), None, intr, pose, st.TraceConfig(alpha=alpha, coarse_start_scale=1))
        conv = r.state.status == st.CONVERGED
        return float((r.state.topk_f[conv, 0] < 0.0).mean())

    f15, f10 = neg_frac(1.5), neg_frac(1.0)
    assert f15 >= 0.10 and f15 > f10


def test_trace_rejects_indivisible_resolution(st):
    """test_tracer.py:305-309."""
    with pytest.raises(ValueError):
        st.trace(Sphere(), None, st.Intrinsics(width=30, height=30), st.look_at((0.0, 0.0, -2.0)),
                 st.TraceConfig(coarse_start_scale=4))


# --- shading heads (pkg/tests/test_shading.py) --------------------------------

def test_surrogate_depth_reproduces_trace_bitwise(st, small_camera):
    """test_shading.py:232-244."""
    intr, pose = small_camera
    field = Sphere(0.5)
    result = st.trace(field, None, intr, pose, _plain(st))
    heads = st.diff_heads(result, field)
    rows = np.nonzero(heads.converged)[0]
    assert rows.size > 100
    for r in rows[:40]:
        i = heads.ray_index[r]
        assert heads.depth_value[heads.best_sample[r]] == st.ray_distance(result.state, i, 1.0)
    assert np.array_equal(heads.depth_image(intr.height, intr.width), st.depth_map(result))


def test_sample_point_grads_are_field_gradients(st, small_camera):
    """test_shading.py:261-270."""
    intr, pose = small_camera
    field = Sphere(0.5)
    result = st.trace(field, None, intr, pose, _plain(st))
    heads = st.diff_heads(result, field)
    grads = heads.backward(depth_seed=np.ones(heads.sample_d.shape[0]))
    pts = result.state.bundle.origin + heads.sample_d[:, None] * \
        result.state.bundle.dirs[heads.ray_index][heads.sample_pixel]
    assert np.max(np.abs(grads["sample_point_grads"] - field.spatial_gradient(pts))) < 1e-12


def test_head_weights_sum_to_one_per_pixel(st, small_camera):
    """test_shading.py:273-284."""
    intr, pose = small_camera
    result = st.trace(Sphere(0.5), None, intr, pose,
                      st.TraceConfig(alpha=1.5, coarse_start_scale=1, k_samples=3))
    heads = st.diff_heads(result, Sphere(0.5))
    acc = np.zeros(heads.pixels.shape[0])
    np.add.at(acc, heads.sample_pixel, heads.sample_weight)
    assert np.allclose(acc, 1.0, atol=1e-12)
    counts = np.bincount(heads.sample_pixel)
    assert counts.max() == 3 and counts.min() >= 1


def test_code_gradient_matches_fd(st, tiny_net, small_camera):
    """test_shading.py:287-309 (tiny_net, device decoder fp64)."""
    net, code = tiny_net
    intr, pose = small_camera
    result = st.trace(net, code, intr, pose, st.TraceConfig(coarse_start_scale=1))
    heads = st.diff_heads(result, net, code)
    m, p = heads.sample_d.shape[0], heads.pixels.shape[0]
    assert heads.converged.sum() > 50
    rng = np.random.default_rng(0)
    wd, ws = rng.standard_normal(m), rng.standard_normal(p)
    g = heads.backward(depth_seed=wd)["code"]
    gs = heads.backward(sil_seed=ws)["code"]
    h = 1e-6
    for k in range(2):
        e = np.zeros(2)
        e[k] = h
        dp, sp, _ = heads.evaluate_at(code + e)
        dm, sm, _ = heads.evaluate_at(code - e)
        fd_d = (np.sum(wd * dp) - np.sum(wd * dm)) / (2 * h)
        fd_s = (np.sum(ws * sp) - np.sum(ws * sm)) / (2 * h)
        assert abs(g[k] - fd_d) / max(abs(fd_d), 1e-9) < 1e-4
        assert abs(gs[k] - fd_s) / max(abs(fd_s), 1e-9) < 1e-4


def test_normal_head_gradient_matches_fd(st, tiny_net, small_camera):
    """test_shading.py:312-330."""
    net, code = tiny_net
    intr, pose = small_camera
    result = st.trace(net, code, intr, pose, st.TraceConfig(coarse_start_scale=1))
    heads = st.diff_heads(result, net, code, want_normals=True)
    W = np.random.default_rng(1).standard_normal((heads.pixels.shape[0], 3))
    g = heads.backward(normal_seed=W)["code"]
    h = 1e-6
    for k in range(2):
        e = np.zeros(2)
        e[k] = h
        _, _, np_ = heads.evaluate_at(code + e)
        _, _, nm_ = heads.evaluate_at(code - e)
        fd = (np.sum(W * np_) - np.sum(W * nm_)) / (2 * h)
        assert abs(g[k] - fd) / max(abs(fd), 1e-9) < 1e-3
    assert heads.backward(normal_seed=W)["surface_point_grads"].shape == (int(heads.converged.sum()), 3)


def test_evaluate_at_is_pure(st, tiny_net, small_camera):
    """test_shading.py:333-345."""
    net, code = tiny_net
    intr, pose = small_camera
    result = st.trace(net, code, intr, pose, st.TraceConfig(coarse_start_scale=1))
    heads = st.diff_heads(result, net, code)
    before = heads.depth_value.copy()
    d_same, _, _ = heads.evaluate_at(code)
    assert np.array_equal(d_same, before)
    heads.evaluate_at(code + 0.1)
    assert np.array_equal(heads.depth_value, before)
    d_state = result.state.d.copy()
    heads.backward(depth_seed=np.ones_like(heads.sample_d))
    assert np.array_equal(result.state.d, d_state)


def test_eval_field_taped_backward(st, tiny_net):
    """fields.py:355-373 / autodiff.py:220-255: the taped evaluation's
    gradients equal the vjp of the decoder; leaves points and code."""
    net, code = tiny_net
    pts = np.random.default_rng(3).uniform(-0.6, 0.6, (200, 3))
    te = st.eval_field_taped(net, pts, code)
    np.testing.assert_array_equal(te.values, net.evaluate(pts, code))
    seed = np.random.default_rng(4).standard_normal(200)
    g = st.backward(te.tape, te.output, seed)
    assert set(g) == {"points", "code"} and g["points"].shape == (200, 3)
    h = 1e-6
    for k in range(2):
        e = np.zeros(2)
        e[k] = h
        fd = (seed @ net.evaluate(pts, code + e) - seed @ net.evaluate(pts, code - e)) / (2 * h)
        assert abs(g["code"][k] - fd) < 1e-6 * max(1.0, abs(fd))
    ta = st.eval_field_taped(Sphere(0.5), pts)
    ga = st.backward(ta.tape, ta.output, seed)
    np.testing.assert_allclose(ga["points"], seed[:, None] * Sphere(0.5).spatial_gradient(pts))
    with pytest.raises(ValueError):
        st.backward(te.tape, te.output, seed[:10])
    with pytest.raises(ValueError):
        st.eval_field_taped(net, pts, code, want_weights=True)


# --- drivers (pkg/tests/test_optimize.py) -----------------------------------------

MATCHED = dict(alpha=1.0, k_samples=1, coarse_start_scale=1)   # test_optimize.py:18-22


def test_complete_shape_true_code_is_a_fixed_point(st, tiny_net, small_camera):
    """test_optimize.py:108-120 (tiny_net instead of the fitted sphere family)."""
    net, z_true = tiny_net
    intr, pose = small_camera
    cfg = st.TraceConfig(**MATCHED)
    obs = st.Observation("depth", st.depth_map(st.trace(net, z_true, intr, pose, cfg)))
    code, report = st.complete_shape(net, [obs], intr, pose, code0=z_true, iters=5, cfg=cfg,
                                     weights=st.LossWeights(latent=0.0))
    assert np.array_equal(code, z_true)
    assert report.losses == [0.0] * 5


def test_complete_shape_report_replays_exactly(st, tiny_net, small_camera):
    """test_optimize.py:123-134."""
    net, z_true = tiny_net
    intr, pose = small_camera
    cfg = st.TraceConfig(**MATCHED)
    obs = st.Observation("depth", st.depth_map(st.trace(net, z_true, intr, pose, cfg)))
    code, report = st.complete_shape(net, [obs], intr, pose, iters=8, cfg=cfg, weights=st.LossWeights())
    total, _, _, _, _ = st.completion_objective(net, code, [obs], intr, pose, cfg, st.LossWeights())
    assert total == report.best_loss
    assert report.losses[report.best_iter] == report.best_loss


# --- batched views keep the reference's per-view level loop (tracer.py:236-252) ---

class _HalfConst:
    """f = 1e-5 (< eps: converged at once) where x < 0, a radius-0.5 sphere elsewhere."""
    latent_dim = 0

    def evaluate(self, points, code=None):
        p = np.atleast_2d(points)
        f = np.linalg.norm(p, axis=1) - 0.5
        return np.where(p[:, 0] < 0.0, 1e-5, f)


def _views(st, eyes, res=32):
    return [(st.Intrinsics(width=res, height=res), st.look_at(e)) for e in eyes]


def test_batched_views_keep_their_own_step_budget(st):
    """View A's coarse levels empty after one step each while view B marches
    every slot: with max_steps = 6 the reference gives A three steps and its
    rays converge, however many slots B uses.  A batched trace must equal each
    view traced alone (per-ray state and the views' own live_counts)."""
    from paper_1911_13225_b200.tracer import host_result, trace_external
    views = _views(st, [(-3.0, 0.0, 0.0), (3.0, 0.2, 0.1)])
    cfg = st.TraceConfig(max_steps=6)
    f = _HalfConst()
    both = trace_external(f, None, views, cfg)
    for v in range(2):
        alone = host_result(trace_external(f, None, [views[v]], cfg), 0)
        mine = host_result(both, v)
        assert mine.live_counts == alone.live_counts, v
        assert mine.total_queries == alone.total_queries
        for k in ("status", "steps", "d", "topk_d", "topk_absf"):
            np.testing.assert_array_equal(getattr(mine.state, k), getattr(alone.state, k), err_msg=k)
    a = host_result(both, 0)
    assert (a.state.status == st.CONVERGED).sum() > 50 and len(a.live_counts) == 3


def test_batched_decoder_views_equal_single_view_traces(st, tiny_net):
    """The same property through the device decoder (fp64 SIMT march): three
    views of the tiny net, one far away, a tight step budget."""
    from paper_1911_13225_b200.tracer import host_result
    net, code = tiny_net
    views = _views(st, [(0.0, 0.0, -2.0), (0.0, 0.3, -9.0), (1.5, 0.0, -1.2)])
    cfg = st.TraceConfig(max_steps=7, k_samples=3)
    both = st.trace_views(net, code, views, cfg)
    for v in range(3):
        alone = host_result(st.trace_views(net, code, [views[v]], cfg), 0)
        mine = host_result(both, v)
        assert mine.live_counts == alone.live_counts, v
        for k in ("status", "steps", "d", "topk_d"):
            np.testing.assert_array_equal(getattr(mine.state, k), getattr(alone.state, k), err_msg=k)
