"""Per-phase timeline of one tile of the tensor-core kernels on a B200.

With DIST_TC_TIMELINE=1 the first epilogue thread of CTA 0 appends
(mark id << 56 | %globaltimer) pairs to a device buffer per kernel
(csrc/tc_core.cuh DIST_TL_MARK); this script runs
  * k_tc_mlp on a 1M-point evaluation (same tile loop as a march step) and
  * k_tc_heads in one C3 latent-optimisation iterate (8 views x 512^2),
and prints the phase durations of two tiles of each (the head kernel with
and without the ReLU-mask record: DIST_TC_TIMELINE=1 / 2 select which).

  python scripts/tile_timeline.py
"""
from __future__ import annotations

import ctypes
import os
import sys

os.environ["DIST_TC_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200 import _lib  # noqa: E402
from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code  # noqa: E402

MLP = {1: "tile start", 2: "layer0 A ready", 10: "prev tile rows done", 3: "D (nh=0 half) ready", 4: "A ready",
       9: "head done", 11: "nh=1 MMAs past K 3 (afree)", 12: "parked copied", 13: "K 0..3 announced",
       14: "nh=1 half done"}
HEADS = {1: "tile start", 2: "layer0 A ready", 3: "fwd D ready", 4: "fwd A ready", 5: "seed done",
         6: "bwd A0 ready", 7: "bwd D ready", 8: "bwd A ready", 9: "colsum done", 10: "colsum chunks done"}


def show(fn, names, label):
    buf = (ctypes.c_ulonglong * 4096)()
    fn(buf, 4096)
    a = np.array(buf[:], dtype=np.uint64)
    ids = (a >> np.uint64(56)).astype(int)
    t = (a & np.uint64((1 << 56) - 1)).astype(np.int64)
    n = int(np.argmax(ids == 0)) if (ids == 0).any() else len(ids)
    ids, t = ids[:n], t[:n]
    starts = np.nonzero(ids == 1)[0]
    for k in range(1, min(3, len(starts) - 1)):
        s, e = starts[k], starts[k + 1]
        print(f"--- {label} tile {k}: {(t[e] - t[s]) / 1e3:.1f} us")
        for i in range(s, e):
            dt = (t[i] - t[i - 1]) / 1e3 if i > s else 0.0
            print(f"  {names[ids[i]]:20s} +{(t[i] - t[s]) / 1e3:7.2f} us  (dt {dt:6.2f})")


MMA = {20: "MMA: K 0..3 of A seen", 21: "MMA: K 0..3 issued", 22: "MMA: K 4..7 of A seen"}


def merged(fn, label, ntiles=1):
    """The epilogue thread's marks and the MMA thread's (buffer upper half) on one clock."""
    buf = (ctypes.c_ulonglong * 4096)()
    fn(buf, 4096)
    a = np.array(buf[:], dtype=np.uint64)
    ids = (a >> np.uint64(56)).astype(int)
    t = (a & np.uint64((1 << 56) - 1)).astype(np.int64)
    ev = [(t[i], ids[i]) for i in range(4096) if ids[i] != 0]
    ev.sort()
    starts = [k for k, (_, i) in enumerate(ev) if i == 1]
    names = {**MLP, **MMA}
    for k in range(1, min(1 + ntiles, len(starts) - 1)):
        s, e = starts[k], starts[k + 1]
        print(f"--- {label} tile {k} (epilogue + MMA thread marks)")
        for j in range(s, e):
            print(f"  {names.get(ev[j][1], ev[j][1]):28s} +{(ev[j][0] - ev[s][0]) / 1e3:7.2f} us")


def main():
    lib = _lib.lib()
    field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="bf16x3")
    code = np.random.default_rng(2).normal(0, 0.1, 256)
    pts = torch.from_numpy(np.random.default_rng(0).uniform(-0.8, 0.8, (1 << 20, 3))).cuda()
    field.evaluate_device(pts, code)
    torch.cuda.synchronize()
    show(lib.dist_debug_mlp_timeline, MLP, "k_tc_mlp")
    merged(lib.dist_debug_mlp_timeline, "k_tc_mlp")
    if os.environ.get("TL_MLP_ONLY"):
        return
    if os.environ.get("TL_MARCH"):
        # a bulk march step: the last slot of a trace cut at max_steps = 8 is
        # the second full-resolution slot (2 x 1e6 rays of 8 ring views)
        f16 = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
        from paper_1911_13225_b200.tracer import trace_views
        trace_views(f16, target_code(1), ring_views(8, 512), st.TraceConfig(k_samples=3, max_steps=8),
                    relu_masks=True)
        torch.cuda.synchronize()
        merged(lib.dist_debug_mlp_timeline, "k_tc_mlp march (fluid, mask record)")
        return
    views = ring_views(8, 512)
    cfg = st.TraceConfig(k_samples=3)
    obs = render_depth_observations(field, target_code(1), views, cfg)
    for env, label, rm in (("1", "k_tc_heads (full: taped forward + backward)", False),
                           ("2", "k_tc_heads<BWD> (ReLU-mask record: backward only)", True)):
        os.environ["DIST_TC_TIMELINE"] = env
        opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=4,
                                 relu_masks=rm)
        opt.step()
        opt.step()
        torch.cuda.synchronize()
        show(lib.dist_debug_heads_timeline, HEADS, label)


if __name__ == "__main__":
    main()
