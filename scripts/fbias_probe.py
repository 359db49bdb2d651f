"""Diagnostic: signed error of the tensor-core decoder (f_tc - f_fp64) on the
query points of a real trace (the C3 ring view 0 sample record), and its
dependence on f -- the TMEM accumulator truncation bias."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200.workloads import ring_views, target_code  # noqa: E402

f64 = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp64")
z = target_code(1)
views = ring_views(8, 512)[:2]
dt = st.trace_views(f64, z, views, st.TraceConfig(k_samples=3))
# query points: every finite record sample (d_k along the ray) of the two views
from paper_1911_13225_b200.camera import generate_rays  # noqa: E402
pts = []
for v, (intr, pose) in enumerate(views):
    b = generate_rays(intr, pose, 1)
    n = intr.width * intr.height
    td = dt.topk_d[v * n:(v + 1) * n].cpu().numpy()
    ta = dt.topk_absf[v * n:(v + 1) * n].cpu().numpy()
    ok = np.isfinite(ta)
    r, k = np.nonzero(ok)
    pts.append(b.origin + td[r, k, None] * b.dirs[r])
pts = np.concatenate(pts)[:1 << 20]
P = torch.from_numpy(pts).cuda()
ref = f64.evaluate_device(P, z).cpu().numpy()
out = {"n": int(len(pts))}
for prec in ("fp16x3", "bf16x3", "fp32"):
    e = f64.with_precision(prec).evaluate_device(P, z).cpu().numpy() - ref
    near = np.abs(ref) < 1e-3
    A = np.stack([np.ones_like(ref), ref], 1)
    coef = np.linalg.lstsq(A, e, rcond=None)[0]
    out[prec] = {"mean": float(e.mean()), "median": float(np.median(e)), "std": float(e.std()),
                 "mean_near_surface": float(e[near].mean()), "std_near_surface": float(e[near].std()),
                 "maxabs": float(np.abs(e).max()), "fit_bias_slope": [float(c) for c in coef]}
for prec in ("fp16x3", "bf16x3"):
    out[prec]["head_gain"] = f64.with_precision(prec).head_gain()
print(json.dumps(out))
