"""BASELINE configs C4 and C5 on the product path.

* C4 (1024^2 coarse-to-fine, 32 ring views): the full 32-view fp16x3 trace,
  view 0 against the unmodified reference (tests/golden/c4_1024_v0.npz,
  oracle/make_fullsize.py c4) under the tests/test_gpu_fullsize.py contract,
  then one silhouette-supervised iterate of all 32 views.
* C5 (many latents): a batched multi-shape optimiser is the same computation
  as one optimiser per shape -- each view's march keeps its own budget, and
  the exact fixed-point column sums make every shape's gradient independent
  of what else is in the batch -- so the iterates are bit-identical.  Checked
  at a reduced size (4 shapes x 2 views x 128^2, the C5 structure).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import parity_full as pf

pytestmark = pytest.mark.gpu

C4_FIX = os.path.join(pf.GOLDEN, "c4_1024_v0.npz")


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


@pytest.mark.skipif(not os.path.exists(C4_FIX), reason="C4 fixture not generated")
def test_c4_32_views_1024_vs_reference(st):
    from paper_1911_13225_b200.shading import device_maps
    from paper_1911_13225_b200.workloads import ring_eye
    g = pf.load("c4_1024_v0.npz")
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    z = np.random.default_rng(1).normal(0.0, 0.1, 256)
    views = [(st.Intrinsics(width=1024, height=1024), st.look_at(ring_eye(k, 32))) for k in range(32)]
    np.testing.assert_allclose(views[0][1].t, g["t"], rtol=0, atol=0)
    cfg = st.TraceConfig()
    dt = st.trace_views(net, z, views, cfg)
    n = 1024 * 1024
    depth, mask, sil = device_maps(dt, True, True, True)
    s = pf.compare_trace(g, dt.status[:n].cpu().numpy(), dt.steps[:n].cpu().numpy(),
                         depth[0].cpu().numpy(), dt.stats()["live_counts_per_view"][0])
    assert s["hitmask_diff_out_of_band"] == 0
    assert s["mismatch_out_of_band"] <= 1e-4 * n, s["out_of_band_rays"][:10]
    assert s["depth_rel_max"] <= 1e-4 and s["live_over_bound"] == 0
    # one silhouette-supervised iterate over all 32 views (C4's loss)
    import torch
    target = mask.to(dtype=torch.float64)
    opt = st.LatentOptimizer(net, views, {"silhouette": target}, np.zeros((1, 256)), cfg,
                             st.LossWeights(), max_iters=1)
    opt.step()
    g0 = opt.grad.cpu().numpy()[0]
    vt = opt.view_terms.cpu().numpy()
    assert np.all(np.isfinite(g0)) and np.linalg.norm(g0) > 0
    assert np.all(vt[:, 1] >= 0.0) and vt[:, 1].sum() > 0.0


@pytest.mark.parametrize("prec", ["fp16x3", "fp64"])
def test_c5_batched_shapes_equal_independent_optimisers(st, prec):
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    cfg = st.TraceConfig(k_samples=3)
    S, VP, res = 4, 2, 128 if prec == "fp16x3" else 64
    views, sov, obs = [], [], []
    for s in range(S):
        vs = ring_views(VP, res, first=s, total=VP * S, stride=S)
        views += vs
        sov += [s] * VP
        obs.append(render_depth_observations(net, target_code(s), vs, cfg).cpu().numpy())
    z0 = np.stack([np.full(256, 0.01 * (s + 1)) for s in range(S)])
    batched = st.LatentOptimizer(net, views, {"depth": np.concatenate(obs)}, z0, cfg,
                                 shape_of_view=sov, max_iters=2)
    batched.step()
    batched.step()
    for s in range(S):
        one = st.LatentOptimizer(net, views[s * VP:(s + 1) * VP], {"depth": obs[s]}, z0[s:s + 1], cfg,
                                 max_iters=2)
        one.step()
        one.step()
        np.testing.assert_array_equal(batched.code.cpu().numpy()[s], one.code.cpu().numpy()[0])
        np.testing.assert_array_equal(batched.losses()[:, s], one.losses()[:, 0])
