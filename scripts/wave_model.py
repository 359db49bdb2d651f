"""Wave-quantisation model of the tensor-core march for bench.py's C3 shards:
for world sizes G (rank 0's pixel tiles, scripts/strong_scaling_probe.py's
setup) trace once and, from the per-slot live rows, count
  stepped = sum_s ceil(tiles_s / pairs)   (one wave per partial wave: today)
  fluid   = max(sum_s tiles_s / pairs, slots)   (steps overlapping, the bound)
in tile-times (one 128-row tile through the 8x512 decoder on a CTA pair).

  python scripts/wave_model.py [--worlds 1,2,4,8]
"""
import argparse
import json
import math
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
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--tile", type=int, default=32)
args = ap.parse_args()
shard_mod.all_reduce_sum = lambda t, group=None, world=1: t
shard_mod.fixed_all_reduce = lambda b, group=None, world=1: b

field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
cfg = st.TraceConfig(k_samples=3)
views = ring_views(8, 512)
obs = render_depth_observations(field, target_code(1), views, cfg)
pairs = torch.cuda.get_device_properties(0).multi_processor_count // 2
for G in [int(x) for x in args.worlds.split(",")]:
    opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=4,
                             shard=TileShard(0, G, args.tile, None))
    opt.step()
    torch.cuda.synchronize()
    lc = opt.last_trace.live_counts_dev.cpu().numpy().sum(axis=0)
    lc = lc[lc > 0]
    tiles = np.ceil(lc / 128.0)
    stepped = float(np.sum(np.ceil(tiles / pairs)))
    fluid = max(float(np.sum(tiles) / pairs), float(len(lc)))
    print(json.dumps({"G": G, "slots": int(len(lc)), "rows": int(lc.sum()), "tiles": int(tiles.sum()),
                      "stepped_tile_times": stepped, "fluid_tile_times": fluid,
                      "fluid_over_stepped": fluid / stepped,
                      "slots_under_one_wave": int(np.sum(tiles < pairs))}), flush=True)
