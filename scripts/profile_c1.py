"""C1 (tiny 5-16-16-1 MLP, one 64^2 view, one completion iterate) broken
down: device ms per iterate eager and graph-replayed, trace vs objective,
host ms to issue one iterate, and our launches per iterate.  With --ncu the
third eager iterate is bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off` (launch list).

  python scripts/profile_c1.py [--precision fp64|fp32] [--ncu]
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
from paper_1911_13225_b200 import _lib  # noqa: E402
from paper_1911_13225_b200.shading import device_maps  # noqa: E402
from paper_1911_13225_b200.tracer import trace_views  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp64")
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()

rng = np.random.default_rng(7)
net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng, precision=args.precision)
code = rng.normal(0.0, 0.3, 2)
intr, pose = st.Intrinsics(width=64, height=64), st.look_at((0.0, 0.0, -2.0))
cfg = st.TraceConfig(k_samples=3)
obs = {"depth": device_maps(st.trace_views(net, code + 0.05, [(intr, pose)], cfg))[0]}
R = args.reps
opt = st.LatentOptimizer(net, [(intr, pose)], obs, code[None], cfg, max_iters=8 * R + 16)
lib = _lib.lib()
for _ in range(3):
    opt.step()
torch.cuda.synchronize()
if args.ncu:
    torch.cuda.profiler.start()
    opt.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


out = {"precision": args.precision}
# eager: device time, host issue time, launches
torch.cuda.synchronize()
n0 = lib.dist_launch_count()
h0 = time.perf_counter()
e0 = ev()
for _ in range(R):
    opt.step()
e1 = ev()
host_ms = (time.perf_counter() - h0) / R * 1e3
torch.cuda.synchronize()
out["eager_ms"] = e0.elapsed_time(e1) / R
out["eager_host_issue_ms"] = host_ms
out["launches_per_iter"] = (lib.dist_launch_count() - n0) / R
# split
tr, ob = [], []
for _ in range(R):
    a = ev()
    dt = trace_views(net, opt.code, opt.views, cfg, reuse=opt.last_trace, relu_masks=opt.relu_masks)
    opt.last_trace = dt
    b = ev()
    opt._objective_after_trace(dt)
    c = ev()
    opt._adam()
    tr.append((a, b))
    ob.append((b, c))
torch.cuda.synchronize()
out["trace_ms"] = float(np.mean([a.elapsed_time(b) for a, b in tr]))
out["objective_ms"] = float(np.mean([a.elapsed_time(b) for a, b in ob]))
out["queries"] = int(opt.last_trace.stats()["total_queries"])
# graph replay
opt.step_graph()
opt.step_graph()
torch.cuda.synchronize()
e0 = ev()
for _ in range(R):
    opt.step_graph()
e1 = ev()
torch.cuda.synchronize()
out["graph_ms"] = e0.elapsed_time(e1) / R
print(json.dumps(out))
