"""BASELINE config 3 end to end: 200 latent-optimisation iterates over 8 ring
views of 512^2 (depth-supervised, z0 = 0, target z* = N(0, 0.1^2)), in the
tensor-core modes.  Prints one JSON line per mode with the loss curve
(every 10th iterate), time per iterate, the best iterate and the relative
distance of the final code to z*; the curves of the two split modes should
agree to the parity bars of DESIGN.md section 5.

  python scripts/c3_full_run.py [--iters 200] [--modes fp16x3,bf16x3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code  # noqa: E402


def run(mode: str, iters: int, relu_masks="auto"):
    field = st.NeuralField.geometric(256, (512,) * 8, 0, precision=mode)
    views = ring_views(8, 512)
    cfg = st.TraceConfig(k_samples=3)
    z_true = target_code(1)
    obs = render_depth_observations(field, z_true, views, cfg)
    opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=iters,
                             relu_masks=relu_masks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        opt.step()
    e1.record()
    torch.cuda.synchronize()
    losses = opt.losses()[:, 0]
    z = opt.code.cpu().numpy()[0]
    zb = opt.best_code.cpu().numpy()[0]
    return {"mode": mode, "relu_mask_record": opt.relu_masks, "iters": iters,
            "ms_per_iter": e0.elapsed_time(e1) / iters,
            "loss_first": float(losses[0]), "loss_last": float(losses[-1]),
            "loss_every_10": [float(x) for x in losses[::10]],
            "best_iter": int(opt.best_iter[0].item()), "best_loss": float(opt.best_loss[0].item()),
            "skipped_steps": int(opt.skipped[0].item()),
            "rel_dist_to_target_start": 1.0,
            "rel_dist_to_target_final": float(np.linalg.norm(z - z_true) / np.linalg.norm(z_true)),
            "rel_dist_to_target_best": float(np.linalg.norm(zb - z_true) / np.linalg.norm(z_true))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--modes", default="fp16x3,bf16x3")
    ap.add_argument("--compare-record", action="store_true",
                    help="run the first mode with and without the ReLU-mask record")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = {}
    runs = [(m, "auto") for m in args.modes.split(",")]
    if args.compare_record:
        runs = [(runs[0][0], True), (runs[0][0], False)]
    for mode, rm in runs:
        key = f"{mode}/{rm}"
        out[key] = run(mode, args.iters, rm)
        print(json.dumps(out[key]), flush=True)
    if len(out) == 2:
        a, b = (np.asarray(v["loss_every_10"]) for v in out.values())
        print(json.dumps({"max_rel_loss_curve_difference": float(np.max(np.abs(a - b) / np.abs(a)))}))


if __name__ == "__main__":
    main()
