"""recover_pose per-iterate wall time, device objective (dist_pose_*) vs the
HeadBundle host path (optimize._DEVICE_POSE), 8x512 decoder, one view.
One JSON line per setting.

  python scripts/pose_timing.py [--res 128] [--iters 8] [--precision fp16x3]
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
from paper_1911_13225_b200.workloads import target_code  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--res", type=int, default=128)
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--precision", default="fp16x3")
args = ap.parse_args()
net = st.NeuralField.geometric(256, (512,) * 8, 0, precision=args.precision)
intr = st.Intrinsics(width=args.res, height=args.res)
pose = st.look_at((0.3, 0.4, -2.2))
cfg = st.TraceConfig(k_samples=3)
code = target_code(1)
m = st.render(net, code, intr, pose, cfg, with_normals=False)
obs = [st.Observation("depth", m.depth), st.Observation("silhouette", m.mask.astype(np.float64))]
p0 = st.Pose.from_params(pose.params() + np.array([0.02, 0.01, -0.01, 0.0, 0.03, 0.0]))
for dev in (True, False, True):
    optimize._DEVICE_POSE = dev
    st.recover_pose(net, code, obs, intr, p0, iters=1, cfg=cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    best, rep = st.recover_pose(net, code, obs, intr, p0, iters=args.iters, cfg=cfg)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / args.iters
    print(json.dumps({"objective": "device" if dev else "host", "res": args.res, "k_samples": 3,
                      "precision": args.precision, "ms_per_iter": round(ms, 2),
                      "losses": [round(x, 9) for x in rep.losses]}), flush=True)
