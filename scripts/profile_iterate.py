"""One C3 latent-optimisation iterate (the bench's step: 8 ring views x 512^2,
fp16x3, ReLU-mask record) bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch list / per-kernel captures).

  python scripts/profile_iterate.py [--warmup 2]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warmup", type=int, default=2)
args = ap.parse_args()
field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
views = ring_views(8, 512)
cfg = st.TraceConfig(k_samples=3)
obs = render_depth_observations(field, target_code(1), views, cfg)
opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=8)
for _ in range(args.warmup):
    opt.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
opt.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("queries", opt.last_trace.stats()["total_queries"], "samples", int(opt.head_counts[1].item()))
