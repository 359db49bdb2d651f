"""Slot overlap of the fluid march (DIST_TC_TIMELINE=4): one C3 shard
iterate of rank 0 at world size G; prints, per slot, its grid's first CTA
start and last CTA end relative to the trace start, and how much of each
slot ran while the previous slot was still running.

  python scripts/fluid_timeline.py [--world 8]
"""
import argparse
import ctypes
import os
import sys

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200 import _lib, shard as shard_mod  # noqa: E402
from paper_1911_13225_b200.shard import TileShard  # noqa: E402
from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
args = ap.parse_args()
shard_mod.all_reduce_sum = lambda t, group=None, world=1: t
shard_mod.fixed_all_reduce = lambda b, group=None, world=1: b
field = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3")
cfg = st.TraceConfig(k_samples=3)
views = ring_views(8, 512)
obs = render_depth_observations(field, target_code(1), views, cfg)
opt = st.LatentOptimizer(field, views, {"depth": obs}, np.zeros((1, 256)), cfg, max_iters=4,
                         shard=TileShard(0, args.world, 32, None))
opt.step()
torch.cuda.synchronize()
os.environ["DIST_TC_TIMELINE"] = "4"   # the next iterate only (16384 CTA rows)
opt.step()
torch.cuda.synchronize()
os.environ.pop("DIST_TC_TIMELINE")

buf = (ctypes.c_ulonglong * (16384 * 4))()
_lib.lib().dist_debug_fluid_timeline(buf, 16384)
a = np.array(buf[:], dtype=np.uint64).reshape(16384, 4)
a = a[a[:, 1] > 0]
slot = (a[:, 0] & np.uint64(0xFFFFFFFF)).astype(int)
t0, t1 = a[:, 1].astype(np.int64), a[:, 2].astype(np.int64)
tiles = (a[:, 3] >> np.uint64(48)).astype(int)
trow = (a[:, 3] & np.uint64((1 << 48) - 1)).astype(np.int64)
order = np.argsort(t0)
slot, t0, t1, tiles, trow = slot[order], t0[order], t1[order], tiles[order], trow[order]
base = t0[0]
level = np.cumsum(np.r_[0, np.diff(slot) < 0])
print(f"CTA rows {len(slot)}; levels {level.max() + 1}")
prev_end = None
for (lv, sl) in sorted(set(zip(level.tolist(), slot.tolist()))):
    m = (level == lv) & (slot == sl)
    st_, en = (t0[m].min() - base) / 1e3, (t1[m].max() - base) / 1e3
    ov = "" if prev_end is None else f"  overlap with previous {max(0.0, prev_end - st_):7.1f} us"
    busy = m & (tiles > 0)
    if sl < 6 or sl % 10 == 0 or sl > 90:
        print(f"level {lv} slot {sl:3d}: CTAs {m.sum():4d} busy {busy.sum():4d} tiles/CTA max {tiles[m].max()}  "
              f"start {st_:9.1f}  end {en:9.1f}  dur {en - st_:7.1f} us{ov}")
    prev_end = en
