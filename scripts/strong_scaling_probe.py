"""Predict the strong-scaling curve of bench.py (C3 cut into pixel tiles dealt
over G ranks) on ONE GPU: for G in 1, 2, 4, 8 run every rank's shard of the
iterate in turn (the collectives replaced by identity -- their cost is
measured separately: two tiny all-reduces per iterate), time each rank's
iterate with CUDA events, and report max over ranks, the implied rays/s and
the efficiency vs G = 1.  The ranks' kernels never wait on each other, so a
rank's device time alone is what the G-GPU run would see per rank (plus the
collectives).  No numbers from here go into bench.py's JSON.

  python scripts/strong_scaling_probe.py [--tile 32] [--steps 4] [--warmup 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200 import shard as shard_mod  # noqa: E402
from paper_1911_13225_b200.shard import TileShard  # noqa: E402
from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tile", type=int, default=32)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--skew", type=int, default=None, help="shard.DEAL_SKEW (0: plain round-robin)")
args = ap.parse_args()
if args.skew is not None:
    shard_mod.DEAL_SKEW = args.skew

shard_mod.all_reduce_sum = lambda t, group=None, world=1: t
shard_mod.fixed_all_reduce = lambda b, group=None, world=1: b

field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
cfg = st.TraceConfig(k_samples=3)
views = ring_views(8, 512)
obs = render_depth_observations(field, target_code(1), views, cfg)
rays = 8 * 512 * 512
base = None
for G in [int(x) for x in args.worlds.split(",")]:
    per_rank = []
    for r in range(G):
        opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg,
                                 max_iters=args.warmup + args.steps + 2,
                                 shard=TileShard(r, G, args.tile, None))
        for _ in range(args.warmup):
            opt.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tr = []
        e0.record()
        for _ in range(args.steps):
            ev = opt.timing = []
            opt.step()
            opt.timing = None
            tr.append(ev)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        tms = float(np.mean([a.elapsed_time(b) for a, b, _ in tr]))
        per_rank.append((ms, tms, opt.last_trace.stats()["total_queries"]))
        del opt
    worst = max(p[0] for p in per_rank)
    val = rays / (worst * 1e-3)
    base = base or val
    print(json.dumps({"G": G, "tile": args.tile, "skew": shard_mod.DEAL_SKEW, "max_rank_ms": worst,
                      "rank_ms": [round(p[0], 2) for p in per_rank],
                      "rank_trace_ms": [round(p[1], 2) for p in per_rank],
                      "rank_queries": [p[2] for p in per_rank],
                      "rays_per_s": val, "efficiency": val / (G * base)}), flush=True)
