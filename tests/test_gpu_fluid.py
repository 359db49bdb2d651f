"""The fluid tensor-core march (csrc/tc_mlp.cu MarchFluid): consecutive slots
of a level overlap (slot s + 1 claims slot s's survivors as they appear)
instead of each slot waiting for the previous one's last partial wave.  The
per-ray arithmetic is unchanged, so a fluid trace must equal the stepped one
(DIST_TC_STEPPED=1) bit for bit: ray states, top-K records, the ReLU-mask
records they point at, per-view live counts and the audit counters."""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_1911_13225_b200 as st
    return st


def _trace(field, codes, views, cfg, relu, stepped, shape_of_view=None):
    import torch
    from paper_1911_13225_b200.tracer import trace_views
    if stepped:
        os.environ["DIST_TC_STEPPED"] = "1"
    try:
        dt = trace_views(field, codes, views, cfg, shape_of_view, relu_masks=relu)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("DIST_TC_STEPPED", None)
    out = {k: getattr(dt, k).cpu().numpy() for k in
           ("d", "b", "status", "steps", "topk_d", "topk_f", "topk_absf", "live_counts_dev", "stats_dev")}
    if relu:
        K = cfg.k_samples
        slots = dt.topk_slot.cpu().numpy()
        masks = dt.relu_masks.cpu().numpy().reshape(slots.shape[0], K + 1, -1)
        filled = np.isfinite(out["topk_absf"])
        # the records the objective reads: logical k -> physical slot tk_p & 0x7f
        phys = (slots[:, :K] & 0x7F).astype(np.int64)
        rec = np.take_along_axis(masks, phys[:, :, None], axis=1)
        rec[~filled] = 0
        out["records"] = rec
        out["slots"] = np.where(filled, slots[:, :K], 0)
    return out


@pytest.mark.parametrize("relu", [False, True])
def test_fluid_equals_stepped(st, relu):
    from paper_1911_13225_b200.workloads import ring_views, target_code
    field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    views = ring_views(3, 256)   # fine level 197K rays: 1,536 tiles, fluid on every level but the first
    cfg = st.TraceConfig(k_samples=3)
    a = _trace(field, target_code(1), views, cfg, relu, stepped=False)
    b = _trace(field, target_code(1), views, cfg, relu, stepped=True)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["stats_dev"][0] > 100000


def test_fluid_two_shapes_and_skip_layout(st):
    """Batched shapes (per-shape code rows in the tiles) and the DeepSDF skip
    layout through the fluid march."""
    from paper_1911_13225_b200.workloads import ring_views
    field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3", skip=4)
    views = ring_views(2, 256)
    codes = np.stack([np.random.default_rng(s).normal(0, 0.1, 256) for s in (3, 4)])
    cfg = st.TraceConfig(k_samples=2)
    a = _trace(field, codes, views, cfg, False, stepped=False, shape_of_view=[0, 1])
    b = _trace(field, codes, views, cfg, False, stepped=True, shape_of_view=[0, 1])
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_fluid_budget_and_nan_rays(st):
    """A tight step budget (max_steps 12: rays still marching at the end are
    EXHAUSTED) and a shape whose code is NaN (every ray of its views stops at
    its first query, counted as NaN) through the fluid march."""
    from paper_1911_13225_b200.workloads import ring_views, target_code
    field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
    views = ring_views(2, 256)
    codes = np.stack([target_code(1), np.full(256, np.nan)])
    cfg = st.TraceConfig(k_samples=3, max_steps=12)
    a = _trace(field, codes, views, cfg, False, stepped=False, shape_of_view=[0, 1])
    b = _trace(field, codes, views, cfg, False, stepped=True, shape_of_view=[0, 1])
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["stats_dev"][1] > 0              # NaN queries counted
    assert (a["status"] == 3).sum() > 1000    # budget-exhausted rays (EXHAUSTED)
