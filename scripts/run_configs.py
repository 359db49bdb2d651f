"""Run every BASELINE.json config once at full size on one B200 and print one
JSON line per config (time per iterate / render, rays/s, queries).  C3 is the
bench.py workload; the others are parity-tested at small sizes in tests/ and
run here for scale.

  python scripts/run_configs.py [--only C4] [--precision fp16x3|bf16x3|fp32]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200.shading import device_maps, device_normals  # noqa: E402
from paper_1911_13225_b200.workloads import ring_views, target_code  # noqa: E402


def timed(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = None
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def c1(prec):
    """64^2 depth render + one latent-gradient step, tiny random-init MLP (conftest tiny_net)."""
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision="fp32")
    code = rng.normal(0.0, 0.3, 2)
    intr, pose = st.Intrinsics(width=64, height=64), st.look_at((0.0, 0.0, -2.0))
    cfg = st.TraceConfig(k_samples=3)
    obs = {"depth": device_maps(st.trace_views(net, code + 0.05, [(intr, pose)], cfg))[0]}
    opt = st.LatentOptimizer(net, [(intr, pose)], obs, code[None], cfg, max_iters=64)
    opt.step()
    ms, _ = timed(opt.step, 20)
    return {"config": "C1 64^2 tiny MLP, one completion iterate (trace+heads+backward+Adam)",
            "precision": "fp32 (SIMT: widths < 512)", "ms_per_iter": ms, "rays_per_s": 64 * 64 / ms * 1e3}


def c2(prec):
    """256^2 depth + normal render of the 8x512 decoder."""
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    code = np.random.default_rng(1).normal(0.0, 0.1, 256)
    view = [(st.Intrinsics(width=256, height=256), st.look_at((0.0, 0.0, -2.0)))]
    cfg = st.TraceConfig()

    def run():
        dt = st.trace_views(net, code, view, cfg)
        device_maps(dt)
        device_normals(dt)
        return dt
    run()
    ms, dt = timed(run, 3)
    return {"config": "C2 256^2 depth+normal render, 8x512 decoder", "precision": prec,
            "ms_per_render": ms, "rays_per_s": 256 * 256 / ms * 1e3,
            "trace_queries": dt.stats()["total_queries"]}


def _latent_opt(name, prec, views, codes0, targets, shape_of_view, cfg, sil=False):
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    dt = st.trace_views(net, targets, views, cfg, shape_of_view)
    d, m, _ = device_maps(dt, True, sil, False)
    obs = {"silhouette": m.to(torch.float64)} if sil else {"depth": d}
    del dt
    opt = st.LatentOptimizer(net, views, obs, codes0, cfg, shape_of_view=shape_of_view, max_iters=8)
    opt.step()
    ms, _ = timed(opt.step, 2)
    rays = len(views) * views[0][0].width * views[0][0].height
    q = int(opt.last_trace.stats_dev[0].item())
    return {"config": name, "precision": prec, "relu_mask_record": opt.relu_masks,
            "ms_per_iter": ms, "rays_per_s": rays / ms * 1e3,
            "rays_per_iter": rays, "trace_queries": q,
            "peak_mem_gb": torch.cuda.max_memory_allocated() / 2**30}


def c3(prec):
    views = ring_views(8, 512)
    return _latent_opt("C3 8 views x 512^2 depth-supervised latent optimisation (bench.py)", prec,
                       views, np.zeros((1, 256)), target_code(1)[None], None,
                       st.TraceConfig(k_samples=3))


def c4(prec):
    views = ring_views(32, 1024)
    return _latent_opt("C4 32 views x 1024^2 coarse-to-fine, aggressive, silhouette loss", prec,
                       views, np.zeros((1, 256)), target_code(1)[None], None,
                       st.TraceConfig(alpha=1.5, coarse_start_scale=4, k_samples=1), sil=True)


def c5(prec, group=None):
    """64 independent latents x 16 views.  group=None: one optimiser over all
    1024 views (the ReLU-mask record would need 550 GB: off).  group=G: the
    latents in groups of G shapes, one optimiser each, stepped in turn within
    an iterate (independent problems, identical arithmetic per shape), so each
    group's record fits and the objective skips the re-evaluated forward."""
    S, VPS = 64, 16
    targets = np.stack([np.random.default_rng(s).normal(0.0, 0.1, 256) for s in range(S)])
    cfg = st.TraceConfig(k_samples=3)
    name = "C5 64 latents x 16 views x 512^2 batched inverse optimisation (one GPU)"
    if not group:
        views, sov = [], []
        for s in range(S):
            for v in ring_views(VPS, 512):
                views.append(v)
                sov.append(s)
        return _latent_opt(name, prec, views, np.zeros((S, 256)), targets, sov, cfg)
    net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=prec)
    opts = []
    for g0 in range(0, S, group):
        views, sov = [], []
        for s in range(group):
            for v in ring_views(VPS, 512):
                views.append(v)
                sov.append(s)
        dt = st.trace_views(net, targets[g0:g0 + group], views, cfg, sov)
        d, _, _ = device_maps(dt, True, False, False)
        del dt
        opts.append(st.LatentOptimizer(net, views, {"depth": d}, np.zeros((group, 256)), cfg,
                                       shape_of_view=sov, max_iters=8))

    def step():
        for o in opts:
            o.step()
            o.last_trace = None   # the next group reuses the cached ray-state/record blocks
    step()
    ms, _ = timed(step, 2)
    rays = S * VPS * 512 * 512
    return {"config": name + f", latents in groups of {group}", "precision": prec,
            "relu_mask_record": opts[0].relu_masks, "ms_per_iter": ms, "rays_per_s": rays / ms * 1e3,
            "rays_per_iter": rays, "peak_mem_gb": torch.cuda.max_memory_allocated() / 2**30}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--precision", default="fp16x3")
    ap.add_argument("--c5-group", type=int, default=4,
                    help="C5 latents per optimiser (0: all 64 in one)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for name, fn in [("C1", c1), ("C2", c2), ("C3", c3), ("C4", c4), ("C5", c5)]:
        if args.only and name not in args.only.split(","):
            continue
        torch.cuda.reset_peak_memory_stats()
        t0 = time.perf_counter()
        out = fn(args.precision, args.c5_group) if name == "C5" else fn(args.precision)
        out["wall_s"] = time.perf_counter() - t0
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
