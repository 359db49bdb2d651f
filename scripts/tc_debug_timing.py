"""Decoder-evaluation timing under the kernel's DIST_TC_DEBUG experiments
(results invalid for debug != 0): which part of k_tc_mlp bounds a tile?
  DIST_TC_DEBUG=0 (product) 1 (no epilogue math) 2 (no MMAs) 4 (no weight TMA)
  python scripts/tc_debug_timing.py   # prints one JSON line for the current env
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_13225_b200 as st  # noqa: E402

field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
n = 148 * 64 * 40   # 40 tiles per CTA pair... per SM-row
pts = torch.from_numpy(np.random.default_rng(0).uniform(-0.8, 0.8, (n, 3))).cuda()
code = np.random.default_rng(1).normal(0, 0.1, 256)
for _ in range(3):
    field.evaluate_device(pts, code)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    field.evaluate_device(pts, code)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
tiles = n / 128
print(json.dumps({"debug": os.environ.get("DIST_TC_DEBUG", "0"), "n": n, "ms": ms,
                  "us_per_tile_round": ms * 1e3 / (tiles / 74),
                  "tflops_executed": n * 3 * 3.67e6 / (ms * 1e-3) / 1e12}))
