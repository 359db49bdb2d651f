"""reconstruct_multiview per-iterate wall time, device-resident loop vs the
per-view host loop (optimize._DEVICE_MULTIVIEW), on 8 ring views of the 8x512
decoder (fp16x3) with textured synthetic images.  One JSON line per setting.

  python scripts/multiview_timing.py [--res 128] [--iters 6]
"""
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
from paper_1911_13225_b200 import optimize  # noqa: E402
from paper_1911_13225_b200.workloads import ring_views, target_code  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--res", type=int, default=128)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--precision", default="fp16x3")
args = ap.parse_args()
field = st.NeuralField.geometric(256, (512,) * 8, 0, precision=args.precision)
views = ring_views(8, args.res)
rng = np.random.default_rng(0)
yy, xx = np.mgrid[0:args.res, 0:args.res] / args.res
images = [np.stack([0.5 + 0.5 * np.sin(9 * xx + k), 0.5 + 0.5 * np.cos(7 * yy - k), xx * yy], axis=2)
          for k in range(8)]
cfg = st.TraceConfig(k_samples=1)
for dev in (True, False, True):
    optimize._DEVICE_MULTIVIEW = dev
    st.reconstruct_multiview(field, images, views, code0=target_code(1) * 0.9, iters=1, views_per_iter=4,
                             cfg=cfg, seed=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    best, rep = st.reconstruct_multiview(field, images, views, code0=target_code(1) * 0.9, iters=args.iters,
                                         views_per_iter=4, cfg=cfg, seed=1)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / args.iters
    print(json.dumps({"loop": "device" if dev else "host", "res": args.res, "views": 8, "views_per_iter": 4,
                      "precision": args.precision, "ms_per_iter": round(ms, 2),
                      "losses": [round(x, 9) for x in rep.losses]}), flush=True)
