"""Parity of the tcgen05 split-precision (bf16x3) decoder path against the
reference fp64 goldens and the oracle.

Contract of the tensor-core modes (the same as the full-size
tests/test_gpu_fullsize.py): decoder values within 2e-5 of fp64; outside
SURVEY 8(c)'s trajectory band (oracle margin_f / margin_esc below 1e-5 /
1e-6) hit masks exact and step counts exact for all but 0.1% of rays (rays
whose grazing trajectory drifts by the TMEM truncation bias); total queries
within 0.2%; depth of matched rays within 1e-4 relative; latent gradient
within 1e-3 relative.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cfg_from, load_golden

pytestmark = pytest.mark.gpu

import sdf_oracle as orc  # noqa: E402  (checker only)


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def test_tc_eval_matches_fp64(st):
    rng = np.random.default_rng(0)
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp64")
    code = rng.normal(0, 0.1, 256)
    for n in [1, 77, 128, 129, 5000]:
        pts = rng.uniform(-0.9, 0.9, (n, 3))
        ref = net.evaluate(pts, code)
        tc = net.with_precision("bf16x3").evaluate(pts, code)
        assert np.max(np.abs(tc - ref)) < 2e-5, n
        assert abs(np.mean(tc - ref)) < 5e-6, n


@pytest.mark.parametrize("prec", ["bf16x3", "fp16x3"])
@pytest.mark.parametrize("name", ["geo64.npz", "geo32s1.npz"])
def test_tc_trace_parity_contract(st, name, prec):
    g = load_golden(name)
    res, seed = int(g["res"]), int(g["seed"])
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision=prec)
    intr, pose = st.Intrinsics(width=res, height=res), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    r = st.trace(net, g["code"], intr, pose, cfg)
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, seed), 256)
    T = orc.trace(lambda p: dec(p, g["code"]), orc.Cam(res, res, g["omega"], g["t"]),
                  orc.Cfg(k_samples=3))
    assert np.array_equal(T.status, g["status"])
    mism = (r.state.status != g["status"]) | (r.state.steps != g["steps"])
    band = (T.margin_f < 1e-5) | (T.margin_esc < 1e-6)
    assert not np.any(((r.state.status == 1) != (g["status"] == 1)) & ~band)
    assert (mism & ~band).sum() <= max(1, 1e-3 * mism.size), np.nonzero(mism & ~band)
    assert abs(r.total_queries - int(g["total_queries"])) <= 2e-3 * int(g["total_queries"])
    dm = st.depth_map(r).reshape(-1)
    both = (r.state.status == 1) & (g["status"] == 1) & ~mism & ~band
    ref = g["depth"].reshape(-1)
    assert np.max(np.abs(dm[both] - ref[both]) / ref[both]) <= 1e-4


@pytest.mark.parametrize("w,h,cs", [(72, 40, 4), (45, 31, 1)])
def test_tc_trace_nonsquare_ragged_vs_oracle(st, w, h, cs):
    """The fp16x3 tcgen05 march on non-square views whose live sets never fill
    the last 128-row tile (2,880 and 1,395 rays): the module docstring's
    contract against the fp64 oracle on the same decoder, code and camera."""
    g = load_golden("geo64.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, int(g["seed"]), precision="fp16x3")
    cfg = st.TraceConfig(**{**cfg_from(g["cfg"]), "coarse_start_scale": cs})
    r = st.trace(net, g["code"], st.Intrinsics(width=w, height=h), st.Pose(g["omega"], g["t"]), cfg)
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, int(g["seed"])), 256)
    T = orc.trace(lambda p: dec(p, g["code"]), orc.Cam(w, h, g["omega"], g["t"]),
                  orc.Cfg(k_samples=3, coarse_start_scale=cs))
    assert np.any(T.status == 1) and np.any(T.status != 1)
    mism = (r.state.status != T.status) | (r.state.steps != T.steps)
    band = (T.margin_f < 1e-5) | (T.margin_esc < 1e-6)
    assert not np.any(((r.state.status == 1) != (T.status == 1)) & ~band)
    assert (mism & ~band).sum() <= max(1, 1e-3 * mism.size), np.nonzero(mism & ~band)
    tq = sum(T.live_counts)
    assert abs(r.total_queries - tq) <= 2e-3 * tq
    both = (r.state.status == 1) & (T.status == 1) & ~mism & ~band
    assert both.sum() > 0
    assert np.max(np.abs(r.state.d[both] - T.d[both]) / T.d[both]) <= 1e-4


def test_tc_objective_gradient_nonsquare(st):
    """Depth + silhouette completion objective (optimize.py:102-138) on a
    72x40 view in fp16x3: loss and latent gradient within 1e-3 relative of
    the fp64 oracle on the same observations."""
    g = load_golden("geo64.npz")
    w, h = 72, 40
    seed = int(g["seed"])
    intr, pose = st.Intrinsics(width=w, height=h), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    obs_run = st.trace(st.NeuralField.geometric(256, (512,) * 8, seed, precision="fp64"),
                       g["z_true"], intr, pose, cfg)
    depth, sil = st.depth_map(obs_run), st.hard_mask(obs_run).astype(np.float64)
    assert depth.shape == (h, w)
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision="fp16x3")
    tot, terms, grad, n_conv, q = st.completion_objective(
        net, g["code"], [st.Observation("depth", depth), st.Observation("silhouette", sil)],
        intr, pose, cfg, st.LossWeights())
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, seed), 256)
    rt, rterms, rg, rconv, rq, _ = orc.objective(
        dec, g["code"], orc.Cam(w, h, g["omega"], g["t"]), orc.Cfg(k_samples=3), orc.Weights(),
        depth=depth, silhouette=sil)
    assert np.linalg.norm(grad - rg) / np.linalg.norm(rg) < 1e-3
    assert abs(tot - rt) < 1e-3 * abs(rt)
    assert abs(q - rq) <= 2e-3 * rq


def test_tc_objective_gradient(st):
    g = load_golden("geo64.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, int(g["seed"]), precision="bf16x3")
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    tot, terms, grad, n_conv, q = st.completion_objective(
        net, g["code"], [st.Observation("depth", g["obs_depth"])], intr, pose, cfg, st.LossWeights())
    ref = g["obj_grad"]
    assert np.linalg.norm(grad - ref) / np.linalg.norm(ref) < 1e-3
    assert abs(tot - float(g["obj_total"])) < 1e-3 * abs(float(g["obj_total"]))


# C2 (256^2 depth + normal render) against the reference itself, every
# precision: tests/test_gpu_fullsize.py::test_c2_render_vs_reference


@pytest.mark.parametrize("prec", ["bf16x3", "fp16x3"])
def test_tc_pair_normals_same_points(st, prec):
    """Tensor-core (mid, diff) probe pairs (always fp16x3) vs the fp64 probes at
    the SAME traced surface points (north_star: normals within 1e-4)."""
    from paper_1911_13225_b200.shading import device_normals
    code = np.random.default_rng(1).normal(0.0, 0.1, 256)
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    view = [(st.Intrinsics(width=128, height=128), st.look_at((0.0, 0.0, -2.0)))]
    dt = st.trace_views(net, code, view, st.TraceConfig())
    n_tc = device_normals(dt).cpu().numpy().reshape(-1, 3)
    dt.field = net.with_precision("fp64")
    n_64 = device_normals(dt).cpu().numpy().reshape(-1, 3)
    hit = np.linalg.norm(n_64, axis=1) > 0
    assert hit.sum() > 1000
    nd = np.linalg.norm(n_tc - n_64, axis=1)[hit]
    assert np.percentile(nd, 99) < 2e-5 and nd.max() < 1e-4


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("bf16x3", 5e-3)])
def test_depth_and_silhouette_objective_vs_oracle(st, prec, tol):
    """The C4 loss (depth + silhouette hinge, losses.py:54-91) on the 8x512 decoder."""
    g = load_golden("geo64.npz")
    seed = int(g["seed"])
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, seed), 256)
    cam = orc.Cam(64, 64, g["omega"], g["t"])
    ocfg = orc.Cfg(k_samples=3)
    T = orc.trace(lambda p: dec(p, g["z_true"]), cam, ocfg)
    sil = orc.hard_mask(T).astype(np.float64)
    tot_o, terms_o, g_o, n_o, q_o, _ = orc.objective(dec, g["code"], cam, ocfg, orc.Weights(),
                                                     depth=g["obs_depth"], silhouette=sil)
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision=prec)
    obs = [st.Observation("depth", g["obs_depth"]), st.Observation("silhouette", sil)]
    tot, terms, grad, n_conv, q = st.completion_objective(
        net, g["code"], obs, st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"]),
        st.TraceConfig(**cfg_from(g["cfg"])), st.LossWeights())
    assert abs(terms["silhouette"] - terms_o["silhouette"]) < tol * max(abs(terms_o["silhouette"]), 1e-3)
    assert abs(tot - tot_o) < tol * abs(tot_o)
    assert np.linalg.norm(grad - g_o) / np.linalg.norm(g_o) < tol


@pytest.mark.parametrize("S,kind", [(1, "coherent"), (3, "coherent"), (1, "random")])
def test_tc_vjp_matches_fp64(st, S, kind):
    """dist_eval_vjp on a bf16x3 decoder runs the fused tensor-core head kernel
    (given seeds, fp16x2 dgrad, per-point xyz gradient); f, the code gradient
    and d(seed.f)/dp agree with the fp64 SIMT path.  Coherent seeds (the sign
    of f, as a depth loss gives) are the real use; random-sign seeds cancel in
    the code gradient and amplify relative error for every reduced-precision
    mode (fp32 SIMT: 1.3e-3), so they get a looser bar."""
    import torch
    rng = np.random.default_rng(5)
    n = 5000
    p = rng.normal(size=(n, 3))
    p *= rng.uniform(0.3, 0.9, (n, 1)) / np.linalg.norm(p, axis=1, keepdims=True)
    codes = rng.normal(0.0, 0.1, (S, 256))
    sid = torch.from_numpy(rng.integers(0, S, n).astype(np.int32))
    P = torch.from_numpy(p)
    nets = {prec: st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec) for prec in ("fp64", "bf16x3")}
    f_ref = nets["fp64"].evaluate_device(P, torch.from_numpy(codes), sid).cpu().numpy() \
        if S > 1 else nets["fp64"].evaluate(p, codes[0])
    sign = rng.choice([-1.0, 1.0], n) if kind == "random" else np.sign(f_ref)
    sd = torch.from_numpy(sign * rng.uniform(0.5, 1.0, n) / n)
    out = {}
    for prec, net in nets.items():
        f, gc, gp = net.vjp_device(P, torch.from_numpy(codes), sd, shape_ids=sid)
        out[prec] = (f.cpu().numpy(), gc.cpu().numpy(), gp.cpu().numpy())
    (f64, g64, p64), (f16, g16, p16) = out["fp64"], out["bf16x3"]
    assert np.max(np.abs(f16 - f64)) < 2e-5
    tol_g, tol_p = (1e-3, 2e-3) if kind == "coherent" else (1e-2, 5e-3)
    assert np.linalg.norm(g16 - g64) < tol_g * np.linalg.norm(g64)
    assert np.linalg.norm(p16 - p64) < tol_p * np.linalg.norm(p64)


@pytest.mark.parametrize("prec", ["bf16x3", "fp16x3"])
def test_c3_full_size_vs_fp32(st, prec):
    """BASELINE config 3 at full size (8 ring views x 512^2, the bench workload):
    one latent-optimisation iterate on the tensor cores (bf16x3) against the
    fp32 SIMT path on the same inputs -- queries, loss and latent gradient."""
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    views = ring_views(8, 512)
    cfg = st.TraceConfig(k_samples=3)
    ref_field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp32")
    obs = render_depth_observations(ref_field, target_code(1), views, cfg)
    out = {}
    for p in ("fp32", prec):
        field = ref_field if p == "fp32" else ref_field.with_precision(p)
        opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=1)
        dt = opt.objective()
        out[p] = (dt.stats()["total_queries"], float(opt.shape_terms[0, 0].item()),
                  opt.grad.cpu().numpy()[0])
    (q32, l32, g32), (q16, l16, g16) = out["fp32"], out[prec]
    assert abs(q16 - q32) <= 1e-3 * q32
    assert abs(l16 - l32) <= 3e-4 * abs(l32)   # measured 8.4e-5
    assert np.linalg.norm(g16 - g32) <= 1e-3 * np.linalg.norm(g32)


def test_optimisation_loss_curves_track_fp32(st):
    """The latent-optimisation loop (trace + fused heads + backward + Adam) over
    8 ring views at 128^2 for 10 iterates: the split-precision loss curves track
    the fp32 SIMT run (at full size and 200 iterates: 5e-5)."""
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    views = ring_views(8, 128)
    cfg = st.TraceConfig(k_samples=3)
    ref = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp32")
    obs = render_depth_observations(ref, target_code(1), views, cfg)
    curves = {}
    for prec in ("fp32", "fp16x3", "bf16x3"):
        field = ref if prec == "fp32" else ref.with_precision(prec)
        opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=10)
        for _ in range(10):
            opt.step()
        curves[prec] = opt.losses()[:, 0]
    assert curves["fp32"][-1] < 0.7 * curves["fp32"][0]   # the loop makes progress
    for prec in ("fp16x3", "bf16x3"):
        rel = np.abs(curves[prec] - curves["fp32"]) / np.abs(curves["fp32"])
        assert rel.max() < 1e-3, (prec, rel.max())


@pytest.mark.parametrize("depth", [4, 12])
@pytest.mark.parametrize("prec", ["fp16x3", "bf16x3"])
def test_other_depths_on_tensor_cores(st, depth, prec):
    """The tensor-core kernels take the number of hidden GEMMs at run time:
    4x512 and 12x512 geometric decoders, evaluation and the fused objective
    gradient against fp64 SIMT on the same 64^2 view."""
    rng = np.random.default_rng(3)
    code = rng.normal(0.0, 0.1, 256)
    pts = rng.uniform(-0.8, 0.8, (4096, 3))
    f64 = st.NeuralField.geometric(256, (512,) * depth, 0, precision="fp64")
    tcf = f64.with_precision(prec)
    assert np.max(np.abs(tcf.evaluate(pts, code) - f64.evaluate(pts, code))) < 5e-5
    intr, pose = st.Intrinsics(width=64, height=64), st.look_at((0.0, 0.3, -2.0))
    cfg = st.TraceConfig(k_samples=3)
    obs = [st.Observation("depth", st.depth_map(st.trace(f64, code + 0.05, intr, pose, cfg)))]
    t64, _, g64, _, _ = st.completion_objective(f64, code, obs, intr, pose, cfg, st.LossWeights())
    ttc, _, gtc, _, _ = st.completion_objective(tcf, code, obs, intr, pose, cfg, st.LossWeights())
    assert abs(ttc - t64) <= 1e-3 * abs(t64)
    assert np.linalg.norm(gtc - g64) <= 1e-3 * np.linalg.norm(g64)


@pytest.mark.parametrize("latent", [0, 64])
def test_other_latent_sizes_on_tensor_cores(st, latent):
    """Latent size only enters the folded layer-0 bias c0: an unconditioned
    8x512 decoder (latent 0) and latent 64, fp16x3 against fp64."""
    rng = np.random.default_rng(4)
    code = rng.normal(0.0, 0.1, latent) if latent else None
    pts = rng.uniform(-0.8, 0.8, (4096, 3))
    f64 = st.NeuralField.geometric(latent, (512,) * 8, 0, precision="fp64")
    tcf = f64.with_precision("fp16x3")
    assert np.max(np.abs(tcf.evaluate(pts, code) - f64.evaluate(pts, code))) < 5e-5
    intr, pose = st.Intrinsics(width=64, height=64), st.look_at((0.0, 0.3, -2.0))
    r64 = st.trace(f64, code, intr, pose, st.TraceConfig())
    rtc = st.trace(tcf, code, intr, pose, st.TraceConfig())
    assert np.array_equal(r64.state.status, rtc.state.status)
    both = np.isfinite(st.depth_map(r64)) & np.isfinite(st.depth_map(rtc))
    assert np.max(np.abs(st.depth_map(rtc)[both] - st.depth_map(r64)[both]) /
                  st.depth_map(r64)[both]) < 2e-4


@pytest.mark.parametrize("prec", ["fp16x3", "bf16x3"])
def test_ring_trace_parity_vs_fp64_north_star_band(st, prec):
    """8 ring views x 128^2 of the standard decoder traced in fp64 SIMT and on
    the tensor cores: outside the north_star band (final |SDF| within 1e-5 of
    eps in either trace) hit masks and step counts agree up to the trajectory
    floor, and depth of rays converged in both agrees to 1e-4 relative (full
    size: scripts/c3_trace_parity_fp64.py)."""
    from paper_1911_13225_b200.shading import device_maps
    from paper_1911_13225_b200.workloads import ring_views, target_code
    cfg = st.TraceConfig(k_samples=3)
    views = ring_views(8, 128)
    f64 = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp64")
    out = {}
    for p, field in (("fp64", f64), (prec, f64.with_precision(prec))):
        dt = st.trace_views(field, target_code(1), views, cfg)
        depth, _, _ = device_maps(dt, True, False, False)
        out[p] = (dt.status.cpu().numpy(), dt.steps.cpu().numpy(), dt.b.cpu().numpy(),
                  depth.cpu().numpy().reshape(-1), dt.stats()["total_queries"])
    (s0, n0, b0, d0, q0), (s1, n1, b1, d1, q1) = out["fp64"], out[prec]
    eps = cfg.epsilon
    band = (np.abs(np.abs(b0) - eps) < 1e-5) | (np.abs(np.abs(b1) - eps) < 1e-5)
    n = s0.size
    assert ((s0 != s1) & ~band).sum() <= 1e-4 * n          # full size: 8 / 2.1M (fp16x3)
    assert ((n0 != n1) & ~band).sum() <= 2e-3 * n          # full size: 0.05% (fp16x3)
    assert abs(q1 - q0) <= 5e-4 * q0                      # 128^2 bf16x3: 1.1e-4
    conv = (s0 == 1) & (s1 == 1) & ~band
    assert conv.sum() > 0.2 * n
    rel = np.abs(d1[conv] - d0[conv]) / np.abs(d0[conv])
    assert rel.max() <= 1e-4


@pytest.mark.parametrize("kw", [
    dict(alpha=1.0, k_samples=1, epsilon=1e-3, coarse_start_scale=1),
    dict(alpha=1.9, k_samples=5, coarse_start_scale=2, split_interval=2),
    dict(alpha=1.5, k_samples=3, max_steps=20),
    dict(alpha=1.5, k_samples=2, use_dynamic_mask=False),
])
def test_tc_trace_config_variants_vs_oracle(st, kw):
    """TraceConfig corners on the fp16x3 march (plain and strongly over-relaxed steps,
    K = 1 and 5, coarse starts 1 / 2 / 4, split every 2 steps, a tight step
    budget, the dynamic mask off) against the fp64 oracle under the module's
    band contract, with per-pixel step counts and the query total."""
    res, seed = 32, 3
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision="fp16x3")
    code = np.random.default_rng(11).normal(0, 0.1, 256) * 0.3
    cam = orc.cam_look_at(orc.ring_eye(2, 8), res, res)
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, seed), 256)
    T = orc.trace(lambda p: dec(p, code), cam, orc.Cfg(**kw))
    r = st.trace(net, code, st.Intrinsics(width=res, height=res), st.Pose(cam.omega, cam.t),
                 st.TraceConfig(**kw))
    band = (T.margin_f < 1e-5) | (T.margin_esc < 1e-6)
    mism = (r.state.status != T.status) | (r.state.steps != T.steps)
    assert not np.any(((r.state.status == 1) != (T.status == 1)) & ~band)
    assert (mism & ~band).sum() <= max(1, 1e-3 * mism.size), np.nonzero(mism & ~band)
    tq = sum(T.live_counts)
    assert abs(r.total_queries - tq) <= max(2, 2e-3 * tq)
    if kw.get("max_steps", 100) == 20:
        assert (T.status == 3).sum() > 0   # the budget exhausts rays
    assert (T.status == 1).sum() > 50
