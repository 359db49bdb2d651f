"""Full-size parity report against the reference fixtures (tests/golden/c2_256.npz,
c3_512_v*.npz; oracle/make_fullsize.py) for every precision mode.

  python scripts/fullsize_parity.py [--out profiles/r02_fullsize_parity.jsonl]
      [--precisions fp64,fp32,bf16x3,fp16x3] [--c3-precisions fp16x3,fp32]

One JSON line per (config, view, precision) with the tests/parity_full.py
statistics, including every out-of-band ray with its trajectory margins.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import parity_full as pf  # noqa: E402
import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200.shading import device_maps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_fullsize_parity.jsonl"))
    ap.add_argument("--precisions", default="fp64,fp32,bf16x3,fp16x3")
    ap.add_argument("--c3-precisions", default="fp16x3,bf16x3,fp32,fp64")
    ap.add_argument("--band-f", type=float, default=pf.BAND_F)
    ap.add_argument("--band-esc", type=float, default=pf.BAND_ESC)
    args = ap.parse_args()
    code = np.random.default_rng(1).normal(0.0, 0.1, 256)
    base = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp64")
    lines = []
    g = pf.load("c2_256.npz")
    intr, pose = st.Intrinsics(width=256, height=256), st.Pose(g["omega"], g["t"])
    for prec in args.precisions.split(","):
        f = base.with_precision(prec)
        t0 = time.time()
        r = st.trace(f, code, intr, pose, st.TraceConfig())
        s = pf.compare_trace(g, r.state.status, r.state.steps, st.depth_map(r), r.live_counts,
                             normals=st.normal_map(r), band_f=args.band_f, band_esc=args.band_esc)
        s.update(config="C2 256^2 render", precision=prec, wall_s=time.time() - t0)
        lines.append(s)
        print(json.dumps({k: v for k, v in s.items() if k != "out_of_band_rays"}), flush=True)
    paths = sorted(glob.glob(os.path.join(pf.GOLDEN, "c3_512_v*.npz")))
    gs = [pf.load(os.path.basename(p)) for p in paths]
    if gs:
        views = [(st.Intrinsics(width=512, height=512), st.Pose(x["omega"], x["t"])) for x in gs]
        n = 512 * 512
        for prec in args.c3_precisions.split(","):
            f = base.with_precision(prec)
            t0 = time.time()
            dt = st.trace_views(f, code, views, st.TraceConfig(k_samples=3))
            depth, _, _ = device_maps(dt, True, False, False)
            status, steps = dt.status.cpu().numpy(), dt.steps.cpu().numpy()
            depth = depth.cpu().numpy().reshape(-1)
            per_view = dt.stats()["live_counts_per_view"]
            for v, x in enumerate(gs):
                sl = slice(v * n, (v + 1) * n)
                s = pf.compare_trace(x, status[sl], steps[sl], depth[sl], per_view[v],
                                     band_f=args.band_f, band_esc=args.band_esc)
                s.update(config="C3 512^2 ring view", view=int(x["view"]), precision=prec,
                         wall_s=time.time() - t0)
                lines.append(s)
                print(json.dumps({k: v for k, v in s.items() if k != "out_of_band_rays"}), flush=True)
            lc = np.asarray(dt.stats()["live_counts"])
            ref = np.zeros(max(len(x["live_counts"]) for x in gs), np.int64)
            for x in gs:
                ref[:len(x["live_counts"])] += x["live_counts"]
            m = min(len(lc), len(ref))
            summ = {"config": "C3 batched live counts", "precision": prec,
                    "steps_equal": int((lc[:m] == ref[:m]).sum()), "steps": int(max(len(lc), len(ref))),
                    "max_abs_diff": int(np.max(np.abs(lc[:m] - ref[:m]))),
                    "queries": int(lc.sum()), "queries_ref": int(ref.sum())}
            lines.append(summ)
            print(json.dumps(summ), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        for s in lines:
            fh.write(json.dumps(s) + "\n")


if __name__ == "__main__":
    main()
