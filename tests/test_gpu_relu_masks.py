"""The ReLU-mask record (include/dist.h dist_ray_state.relu_masks): the march
stores the ReLU masks of every sample its own queries put in the top-K record,
and the objective then runs only the backward sweep for those samples instead
of re-evaluating the taped forward (shading.py:185-206 recomputes exactly the
values the march computed, tracer.py:141 records f).

Checked here: the recorded bits against an fp64 forward of the same points
(flips only at the ReLU kink), the slot bookkeeping (own/inherited flags and a
permutation of K+1 slots per ray), and the objective with and without the
record against each other and against the fp64 oracle."""
from __future__ import annotations

import numpy as np
import pytest

import sdf_oracle as orc  # noqa: E402  (checker only)
from conftest import cfg_from, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _preacts(weights, code, pts):
    """fp64 pre-activations of every ReLU layer (the reference's forward,
    fields.py:239-247: x = [code, p], relu(x W + b), tanh head)."""
    x = np.concatenate([np.broadcast_to(code, (len(pts), len(code))), pts], axis=1)
    out = []
    for W, b in weights[:-1]:
        y = x @ W + b
        out.append(y)
        x = np.maximum(y, 0.0)
    return out, np.tanh(x @ weights[-1][0] + weights[-1][1])[:, 0]


@pytest.mark.parametrize("prec", ["fp16x3", "bf16x3"])
def test_recorded_masks_match_fp64_forward(st, prec):
    from paper_1911_13225_b200.camera import generate_rays
    g = load_golden("geo64.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, int(g["seed"]), precision=prec)
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    opt = st.LatentOptimizer(net, [(intr, pose)], {"depth": g["obs_depth"]},
                             np.asarray(g["code"]).reshape(1, -1), cfg, relu_masks=True)
    opt.objective()
    dt = opt.last_trace
    K, nm = cfg.k_samples, len(net.weights) - 1
    n = 64 * 64
    slots = dt.topk_slot.cpu().numpy().astype(np.int64)            # [n, K+1]
    rec = dt.relu_masks.cpu().numpy().view(np.uint32).reshape(n, K + 1, nm, 16)
    tk_d, tk_f = dt.topk_d.cpu().numpy(), dt.topk_f.cpu().numpy()
    tk_a = dt.topk_absf.cpu().numpy()
    # every ray's physical slots are a permutation of 0..K; the own flag is
    # set only on filled records
    assert np.all(np.sort(slots & 0x7F, axis=1) == np.arange(K + 1))
    own = (slots[:, :K] & 0x80) != 0
    assert not np.any(own & ~np.isfinite(tk_a))
    assert own.sum() > 0.5 * np.isfinite(tk_a).sum()   # most records are this ray's own queries
    rays = generate_rays(intr, pose, 1)
    r_idx, k_idx = np.nonzero(own)
    pts = rays.origin + tk_d[r_idx, k_idx][:, None] * rays.dirs[r_idx]
    pre, f64 = _preacts(net.weights, np.asarray(g["code"]), pts)
    # the march's f of the record against fp64 at the same point
    np.testing.assert_allclose(tk_f[r_idx, k_idx], f64, atol=2e-5, rtol=0)
    words = rec[r_idx, slots[r_idx, k_idx] & 0x7F]                # [m, nm, 16]
    # record word 4 q4 + 2 nh + c holds columns nh 256 + 64 q4 + 32 c + bit (tc_mlp.cu put_mask)
    perm = np.empty(16, dtype=np.int64)
    for q4 in range(4):
        for nh in range(2):
            for c in range(2):
                perm[nh * 8 + 2 * q4 + c] = 4 * q4 + 2 * nh + c
    words = np.ascontiguousarray(words[..., perm])
    bits = np.unpackbits(words.view(np.uint8), axis=-1, bitorder="little").reshape(len(r_idx), nm, 512)
    flips = 0
    for layer in range(nm):
        want = pre[layer] > 0
        bad = bits[:, layer].astype(bool) != want
        flips += int(bad.sum())
        if bad.any():   # only at the kink: |pre-activation| tiny against the layer's scale
            scale = np.abs(pre[layer]).max(axis=1, keepdims=True)
            assert np.all(np.abs(pre[layer])[bad] < 1e-4 * np.broadcast_to(scale, bad.shape)[bad])
    assert flips <= 1e-5 * bits.size, flips


@pytest.mark.parametrize("prec", ["fp16x3", "bf16x3"])
def test_objective_with_mask_record_vs_without_and_oracle(st, prec):
    g = load_golden("geo64.npz")
    seed = int(g["seed"])
    net = st.NeuralField.geometric(256, (512,) * 8, seed, precision=prec)
    intr, pose = st.Intrinsics(width=64, height=64), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    code = np.asarray(g["code"]).reshape(1, -1)
    out = {}
    for rm in (False, True):
        opt = st.LatentOptimizer(net, [(intr, pose)], {"depth": g["obs_depth"]}, code, cfg,
                                 relu_masks=rm)
        opt.objective()
        out[rm] = (opt.shape_terms[0, 0].item(), opt.grad[0].cpu().numpy(),
                   opt.head_counts.cpu().numpy().tolist())
    assert out[True][2] == out[False][2]
    assert abs(out[True][0] - out[False][0]) < 1e-4 * abs(out[False][0])
    gr = out[False][1]
    assert np.linalg.norm(out[True][1] - gr) / np.linalg.norm(gr) < 5e-4
    # both against the fp64 oracle objective (the golden of test_gpu_heads)
    ref = g["obj_grad"]
    assert abs(out[True][0] - float(g["obj_total"])) <= 1e-3 * abs(float(g["obj_total"]))
    assert np.linalg.norm(out[True][1] - ref) / np.linalg.norm(ref) < 1e-3


def test_mask_record_c3_scale_gradient(st):
    """Two C3 views at 512^2 (every sample path of the bench): the objective
    with the record equals the re-evaluated one within the split arithmetic's
    noise, and the sample split covers every seeded sample."""
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    views = ring_views(8, 512)[:2]
    cfg = st.TraceConfig(k_samples=3)
    obs = render_depth_observations(net, target_code(1), views, cfg)
    z0 = np.random.default_rng(5).normal(0, 0.05, (1, 256))
    out = {}
    for rm in (False, True):
        opt = st.LatentOptimizer(net, views, {"depth": obs}, z0, cfg, relu_masks=rm)
        opt.objective()
        out[rm] = (opt.shape_terms[0, 0].item(), opt.grad[0].cpu().numpy(),
                   opt.head_counts.cpu().numpy().tolist())
    assert out[True][2] == out[False][2]
    assert abs(out[True][0] - out[False][0]) < 1e-4 * abs(out[False][0])
    gr = out[False][1]
    assert np.linalg.norm(out[True][1] - gr) / np.linalg.norm(gr) < 5e-4


@pytest.mark.parametrize("prec", ["fp16x3", "bf16x3"])
def test_mask_record_silhouette_and_shapes(st, prec):
    """Silhouette seeds (slot 0 of every recorded ray, escaped rays included)
    and two shapes in one optimiser: the record changes nothing beyond the
    split arithmetic's noise, per shape."""
    from paper_1911_13225_b200.shading import device_maps
    from paper_1911_13225_b200.workloads import ring_views
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    views = ring_views(4, 128)
    cfg = st.TraceConfig(k_samples=3)
    rng = np.random.default_rng(11)
    z_true = rng.normal(0, 0.1, (2, 256))
    sov = [0, 1, 0, 1]
    dt = st.trace_views(net, z_true, views, cfg, shape_of_view=sov)
    status = dt.status.cpu().numpy().reshape(4, 128, 128)
    depth, _, _ = device_maps(dt, True, False, False)
    obs = {"silhouette": (status == 1).astype(np.float64), "depth": depth}
    z0 = rng.normal(0, 0.05, (2, 256))
    out = {}
    for rm in (False, True):
        opt = st.LatentOptimizer(net, views, obs, z0, cfg, shape_of_view=sov, relu_masks=rm)
        opt.objective()
        out[rm] = (opt.shape_terms[:, 0].cpu().numpy(), opt.grad.cpu().numpy(),
                   opt.head_counts.cpu().numpy().tolist())
    assert out[True][2] == out[False][2]
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=1e-4)
    for s in range(2):
        gr = out[False][1][s]
        assert np.linalg.norm(out[True][1][s] - gr) / np.linalg.norm(gr) < 1e-3


@pytest.mark.parametrize("cfg_kw", [
    {"k_samples": 3, "use_dynamic_mask": False},   # every ray queried every step
    {"k_samples": 1, "coarse_start_scale": 1},     # one level: the record starts at init
    {"k_samples": 2, "max_steps": 4},              # the budget ends inside the coarse levels
])
def test_mask_record_trace_variants(st, cfg_kw):
    """Configurations that change which queries reach the record: the
    objective with the record equals the re-evaluated one."""
    from paper_1911_13225_b200.workloads import ring_views
    from paper_1911_13225_b200.shading import device_maps
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    views = ring_views(2, 128)
    cfg = st.TraceConfig(**cfg_kw)
    z_true = np.random.default_rng(3).normal(0, 0.1, 256)
    depth, _, _ = device_maps(st.trace_views(net, z_true, views, cfg), True, False, False)
    z0 = np.random.default_rng(4).normal(0, 0.05, (1, 256))
    out = {}
    for rm in (False, True):
        opt = st.LatentOptimizer(net, views, {"depth": depth}, z0, cfg, relu_masks=rm)
        opt.objective()
        out[rm] = (opt.shape_terms[0, 0].item(), opt.grad[0].cpu().numpy(),
                   opt.head_counts.cpu().numpy().tolist())
    assert out[True][2] == out[False][2]
    assert abs(out[True][0] - out[False][0]) <= 1e-4 * abs(out[False][0]) + 1e-12
    gr = out[False][1]
    if np.linalg.norm(gr) > 0:
        assert np.linalg.norm(out[True][1] - gr) / np.linalg.norm(gr) < 1e-3


def test_mask_record_deep_decoder_many_tiles(st):
    """A 12 x 512 decoder (12 mask layers) with enough samples for several
    backward-only tiles per CTA pair, so the next tile's masks and first
    operand are staged while the current tile's last GEMM runs."""
    from paper_1911_13225_b200.shading import device_maps
    from paper_1911_13225_b200.workloads import ring_views
    net = st.NeuralField.geometric(256, (512,) * 12, 0, precision="fp16x3")
    views = ring_views(4, 128)
    cfg = st.TraceConfig(k_samples=3)
    z_true = np.random.default_rng(3).normal(0, 0.1, 256)
    depth, _, _ = device_maps(st.trace_views(net, z_true, views, cfg), True, False, False)
    z0 = np.random.default_rng(4).normal(0, 0.05, (1, 256))
    out = {}
    for rm in (False, True):
        opt = st.LatentOptimizer(net, views, {"depth": depth}, z0, cfg, relu_masks=rm)
        opt.objective()
        out[rm] = (opt.shape_terms[0, 0].item(), opt.grad[0].cpu().numpy(),
                   opt.head_counts.cpu().numpy().tolist())
    assert out[True][2][1] > 4 * 148 * 64    # > 4 tiles per CTA pair on a B200
    assert abs(out[True][0] - out[False][0]) <= 1e-4 * abs(out[False][0])
    gr = out[False][1]
    assert np.linalg.norm(out[True][1] - gr) / np.linalg.norm(gr) < 1e-3
