"""GPU parity of heads, losses, the fused objective and Adam vs the reference goldens."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import cfg_from, golden_weights, load_golden

pytestmark = pytest.mark.gpu

import sdf_oracle as orc  # noqa: E402  (checker only)


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _setup_tiny(st):
    g = load_golden("tiny64.npz")
    net = st.NeuralField(golden_weights(g), latent_dim=2, precision="fp64")
    res = int(g["res"])
    intr, pose = st.Intrinsics(width=res, height=res), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    return g, net, intr, pose, cfg


def test_tiny_heads_values_and_backward(st):
    g, net, intr, pose, cfg = _setup_tiny(st)
    r = st.trace(net, g["code"], intr, pose, cfg)
    h = st.diff_heads(r, net, g["code"], want_normals=True)
    assert np.array_equal(h.ray_index, g["h_ray_index"])
    assert np.array_equal(h.best_sample, g["h_best"])
    np.testing.assert_allclose(h.sample_d, g["h_sample_d"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(h.sample_f, g["h_sample_f"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(h.normal_value, g["h_normal"], rtol=0, atol=1e-8)
    out = h.backward(depth_seed=g["bw_depth_seed"], sil_seed=g["bw_sil_seed"],
                     normal_seed=g["bw_normal_seed"])
    np.testing.assert_allclose(out["code"], g["bw_code"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(out["sample_point_grads"], g["bw_points"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(out["surface_point_grads"], g["bw_surface"], rtol=1e-6, atol=1e-8)


def test_tiny_completion_objective_all_terms(st):
    g, net, intr, pose, cfg = _setup_tiny(st)
    obs = [st.Observation("depth", g["obs_depth"]), st.Observation("silhouette", g["obs_sil"]),
           st.Observation("normal", g["obs_normal"])]
    tot, terms, grad, n_conv, q = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                          st.LossWeights())
    assert n_conv == int(g["obj_nconv"]) and q == int(g["obj_queries"])
    assert abs(tot - float(g["obj_total"])) < 1e-9
    np.testing.assert_allclose(grad, g["obj_grad"], rtol=1e-7, atol=1e-9)


def test_tiny_fused_objective_depth_only(st):
    g, net, intr, pose, cfg = _setup_tiny(st)
    obs = [st.Observation("depth", g["obs_depth"])]
    tot, terms, grad, n_conv, q = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                          st.LossWeights())
    assert abs(tot - float(g["objd_total"])) < 1e-10
    np.testing.assert_allclose(grad, g["objd_grad"], rtol=1e-9, atol=1e-12)


def test_tiny_fused_objective_depth_and_silhouette(st):
    g, net, intr, pose, cfg = _setup_tiny(st)
    dec = orc.Decoder(golden_weights(g), 2)
    cam = orc.Cam(64, 64, g["omega"], g["t"])
    ocfg = orc.Cfg(k_samples=3)
    tot_o, terms_o, g_o, n_o, q_o, _ = orc.objective(dec, g["code"], cam, ocfg, orc.Weights(),
                                                     depth=g["obs_depth"], silhouette=g["obs_sil"])
    obs = [st.Observation("depth", g["obs_depth"]), st.Observation("silhouette", g["obs_sil"])]
    tot, terms, grad, n_conv, q = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                          st.LossWeights())
    assert n_conv == n_o and q == q_o
    assert abs(terms["silhouette"] - terms_o["silhouette"]) < 1e-12
    assert abs(tot - tot_o) < 1e-10
    np.testing.assert_allclose(grad, g_o, rtol=1e-9, atol=1e-12)


def test_tiny_complete_shape_matches_reference(st):
    g, net, intr, pose, cfg = _setup_tiny(st)
    obs = [st.Observation("depth", g["obs_depth"])]
    best, rep = st.complete_shape(net, obs, intr, pose, code0=np.zeros(2), iters=4, cfg=cfg)
    np.testing.assert_allclose(rep.losses, g["cs_losses"], rtol=1e-9, atol=1e-12)
    assert rep.best_iter == int(g["cs_best_iter"])
    np.testing.assert_allclose(best, g["cs_best"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 1e-3), ("bf16x3", 1e-3), ("fp16x3", 1e-3)])
def test_geo64_objective(st, prec, tol):
    g = load_golden("geo64.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, int(g["seed"]), precision=prec)
    res = int(g["res"])
    intr, pose = st.Intrinsics(width=res, height=res), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    obs = [st.Observation("depth", g["obs_depth"])]
    tot, terms, grad, n_conv, q = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                          st.LossWeights())
    ref = g["obj_grad"]
    assert abs(tot - float(g["obj_total"])) <= tol * abs(float(g["obj_total"]))
    assert np.linalg.norm(grad - ref) / np.linalg.norm(ref) < tol


# Grazing pixels (grad f . v >= -0.1, factor > 10) are excluded by one rule in
# the kernel and the oracle (heads.cuh kImplicitGrazing), so no single pixel's
# surface-point error is amplified past 10x.
@pytest.mark.parametrize("prec,tol", [("fp64", 1e-8), ("bf16x3", 1e-3), ("fp16x3", 1e-3)])
def test_implicit_gradient_mode_vs_oracle(st, prec, tol):
    g = load_golden("geo64.npz")
    seed = int(g["seed"])
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision=prec)
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    obs = [st.Observation("depth", g["obs_depth"])]
    tot, _, grad, _, _ = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                 st.LossWeights(), grad_mode="implicit")
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, seed), 256)
    cam = orc.Cam(64, 64, g["omega"], g["t"])
    tot_o, _, g_o, _, _, _ = orc.objective(dec, g["code"], cam, orc.Cfg(k_samples=3), orc.Weights(),
                                           depth=g["obs_depth"], implicit=True)
    assert abs(tot - tot_o) < 1e-9 + tol * abs(tot_o)
    assert np.linalg.norm(grad - g_o) / np.linalg.norm(g_o) < tol
    # the implicit and surrogate gradients differ (SURVEY 0 finding 4)
    assert np.linalg.norm(g_o - g["obj_grad"]) / np.linalg.norm(g["obj_grad"]) > 1e-2


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-8), ("fp16x3", 1e-3)])
def test_implicit_unit_normal_mode_vs_oracle(st, prec, tol):
    """grad_mode="implicit_unit": the north_star's literal dd/dz = -(1/(n.v)) df/dz
    with n the unit Eq. 3 normal, against the oracle's restatement."""
    g = load_golden("geo64.npz")
    seed = int(g["seed"])
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision=prec)
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    obs = [st.Observation("depth", g["obs_depth"])]
    tot, _, grad, _, _ = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                 st.LossWeights(), grad_mode="implicit_unit")
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, seed), 256)
    cam = orc.Cam(64, 64, g["omega"], g["t"])
    tot_o, _, g_o, _, _, _ = orc.objective(dec, g["code"], cam, orc.Cfg(k_samples=3), orc.Weights(),
                                           depth=g["obs_depth"], implicit="unit")
    _, _, g_raw, _, _, _ = orc.objective(dec, g["code"], cam, orc.Cfg(k_samples=3), orc.Weights(),
                                         depth=g["obs_depth"], implicit=True)
    assert abs(tot - tot_o) < 1e-9 + tol * abs(tot_o)
    assert np.linalg.norm(grad - g_o) / np.linalg.norm(g_o) < tol
    # |grad f| != 1 for the random-init decoder, so the two implicit variants differ
    assert np.linalg.norm(g_o - g_raw) / np.linalg.norm(g_raw) > 1e-3


def test_tiny_complete_shape_all_terms_matches_reference(st):
    """complete_shape with depth + silhouette + normal observations runs the
    normal term on the device (losses.py:94-111, shading.py:259-269): the
    reference's 4-iterate history, per-iterate normal term and best code."""
    g, net, intr, pose, cfg = _setup_tiny(st)
    n = load_golden("normals64.npz")
    obs = [st.Observation("depth", g["obs_depth"]), st.Observation("silhouette", g["obs_sil"]),
           st.Observation("normal", g["obs_normal"])]
    best, rep = st.complete_shape(net, obs, intr, pose, code0=np.zeros(2), iters=4, cfg=cfg)
    np.testing.assert_allclose(rep.losses, n["cs_losses"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose([t["normal"] for t in rep.terms], n["cs_normal_terms"], rtol=1e-9,
                               atol=1e-12)
    assert rep.best_iter == int(n["cs_best_iter"]) and rep.total_queries == int(n["cs_queries"])
    np.testing.assert_allclose(best, n["cs_best"], rtol=1e-9, atol=1e-12)


def test_tiny_normal_only_masked_objective(st):
    """A normal observation with a mask (Observation.valid, losses.py:36-40) alone."""
    g, net, intr, pose, cfg = _setup_tiny(st)
    n = load_golden("normals64.npz")
    obs = [st.Observation("normal", g["obs_normal"], n["nmask"])]
    tot, terms, grad, _, _ = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                     st.LossWeights())
    assert abs(terms["normal"] - float(n["nobj_normal"])) < 1e-10
    assert abs(tot - float(n["nobj_total"])) < 1e-10
    np.testing.assert_allclose(grad, n["nobj_grad"], rtol=1e-8, atol=1e-11)


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 1e-3), ("bf16x3", 1e-3), ("fp16x3", 1e-3)])
def test_geo64_objective_all_terms(st, prec, tol):
    """Depth + silhouette + normal objective of the standard 8x512 decoder
    against the reference (tests/golden/normals64.npz), every precision."""
    n = load_golden("normals64.npz")
    g = load_golden("geo64.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(n["geo_omega"], n["geo_t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    obs = [st.Observation("depth", n["geo_obs_depth"]), st.Observation("silhouette", n["geo_obs_sil"]),
           st.Observation("normal", n["geo_obs_normal"])]
    tot, terms, grad, n_conv, q = st.completion_objective(net, g["code"], obs, intr, pose, cfg,
                                                          st.LossWeights())
    ref = n["geo_grad"]
    assert abs(tot - float(n["geo_total"])) <= tol * abs(float(n["geo_total"]))
    assert abs(terms["normal"] - float(n["geo_normal"])) <= tol * abs(float(n["geo_normal"]))
    assert np.linalg.norm(grad - ref) / np.linalg.norm(ref) < tol


@pytest.mark.gpu
def test_complete_shape_report_matches_reference_file(st, tmp_path):
    """The reference CLI's report of a 3-iteration complete_shape (tiny net, 32^2,
    tests/golden/ref_report.json) is reproduced in fp64: losses, best iterate and
    query count; the written report carries the same fields."""
    import json
    from conftest import GOLDEN
    from paper_1911_13225_b200 import formats as fm
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision="fp64")
    code = rng.normal(0.0, 0.3, 2)
    intr, pose = st.Intrinsics(width=32, height=32), st.look_at((0.0, 0.0, -2.0))
    res = st.trace(net, code + 0.05, intr, pose, st.TraceConfig())
    obs = [st.Observation("depth", st.depth_map(res))]
    _, rep = st.complete_shape(net, obs, intr, pose, iters=3)
    ref = json.load(open(os.path.join(GOLDEN, "ref_report.json")))
    np.testing.assert_allclose(rep.losses, ref["losses"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(rep.grad_norms, ref["grad_norms"], rtol=1e-8)
    assert rep.best_iter == ref["best_iter"] and rep.total_queries == ref["total_queries"]
    fm.save_report(rep, tmp_path / "r.json", "complete-depth")
    mine = json.load(open(tmp_path / "r.json"))
    assert set(mine) == set(ref) and mine["format"] == "sdftrace-report/1"
    # per-iterate loss terms as the reference records them
    assert set(rep.terms[0]) == {"depth", "latent"}
    assert abs(rep.terms[0]["depth"] * 10.0 + rep.terms[0]["latent"] - rep.losses[0]) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("k", [-24, -12, 12, 24])
def test_backward_exactly_linear_in_power_of_two_weight(st, k):
    """Size-independent property of the fused fp16x2 backward: the power-of-two
    row scales absorb a 2^k loss weight exactly, so the latent gradient scales
    bit-exactly (no fp16 overflow or underflow; the exact
    fixed-point column sums, common.cuh fx_t, resolve 2^-95 and hold per-sample
    contributions below 2^31, and convert to fp64 with one rounding)."""
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="bf16x3")
    views = ring_views(2, 128)
    cfg = st.TraceConfig(k_samples=3)
    obs = render_depth_observations(field, target_code(1), views, cfg)
    grads = []
    for w in (10.0, 10.0 * 2.0 ** k):
        opt = st.LatentOptimizer(field, views, {"depth": obs}, np.full((1, 256), 0.01), cfg,
                                 st.LossWeights(depth=w, latent=0.0), max_iters=1)
        opt.objective()
        grads.append(opt.grad.cpu().numpy()[0])
    assert np.all(np.isfinite(grads[1])) and np.linalg.norm(grads[0]) > 0
    assert np.array_equal(grads[1], grads[0] * 2.0 ** k)
