"""Full-size trace parity (BASELINE config 3: 8 ring views x 512^2, the bench
workload): the tensor-core precisions against the fp64 SIMT trace (the
reference's own arithmetic, bit-exact on every golden) on the same decoder,
code and cameras.  Prints one JSON line per precision with the north_star's
parity terms:

* hit masks (status) and step counts, over all rays and over the rays outside
  the north_star band (final |SDF| of the fp64 trace within 1e-5 of epsilon);
* per-step live counts;
* depth relative error of rays converged in both traces.

  python scripts/c3_trace_parity_fp64.py [--res 512] [--views 8]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1911_13225_b200 as st  # noqa: E402
from paper_1911_13225_b200.shading import device_maps  # noqa: E402
from paper_1911_13225_b200.workloads import ring_views, target_code  # noqa: E402


def run(field, z, views, cfg):
    dt = st.trace_views(field, z, views, cfg)
    depth, _, _ = device_maps(dt, True, False, False)
    return {"status": dt.status.cpu().numpy(), "steps": dt.steps.cpu().numpy(),
            "b": dt.b.cpu().numpy(), "depth": depth.cpu().numpy().reshape(-1),
            "live": np.array(dt.stats()["live_counts"]), "queries": dt.stats()["total_queries"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, default=512)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--precisions", default="fp16x3,bf16x3,fp32")
    args = ap.parse_args()
    cfg = st.TraceConfig(k_samples=3)
    views = ring_views(args.views, args.res)
    z = target_code(1)
    f64 = st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp64")
    ref = run(f64, z, views, cfg)
    eps = cfg.epsilon
    band = np.abs(np.abs(ref["b"]) - eps) < 1e-5     # north_star: final |SDF| within 1e-5 of eps
    for prec in args.precisions.split(","):
        out = run(f64.with_precision(prec), z, views, cfg)
        st_diff = out["status"] != ref["status"]
        sp_diff = out["steps"] != ref["steps"]
        any_diff = st_diff | sp_diff
        conv = (ref["status"] == 1) & (out["status"] == 1)
        rel = np.abs(out["depth"][conv] - ref["depth"][conv]) / np.abs(ref["depth"][conv])
        same = conv & ~sp_diff
        rel_same = np.abs(out["depth"][same] - ref["depth"][same]) / np.abs(ref["depth"][same])
        # the band on either trace's final |SDF| (a ray that stops at a grazing
        # near-miss in one trace and marches on to a farther surface in the other
        # ends within 1e-5 of eps in the first)
        band2 = band | (np.abs(np.abs(out["b"]) - eps) < 1e-5)
        out2 = conv & ~band2[:]
        rel2 = np.abs(out["depth"][out2] - ref["depth"][out2]) / np.abs(ref["depth"][out2])
        nl = min(len(ref["live"]), len(out["live"]))
        live_diff = np.abs(out["live"][:nl] - ref["live"][:nl])
        line = {
            "workload": f"C3 trace: {args.views} ring views x {args.res}^2, geometric 8x512, z = target_code(1)",
            "precision": prec, "rays": int(ref["status"].size),
            "queries": [int(ref["queries"]), int(out["queries"])],
            "status_differ": int(st_diff.sum()), "status_differ_outside_band": int((st_diff & ~band).sum()),
            "steps_differ": int(sp_diff.sum()), "steps_differ_outside_band": int((sp_diff & ~band).sum()),
            "rays_in_band": int(band.sum()),
            "differ_outside_band_frac": float((any_diff & ~band).sum() / any_diff.size),
            "live_counts_max_abs_diff": int(live_diff.max()) if nl else 0,
            "live_counts_max_rel_diff": float((live_diff / np.maximum(ref["live"][:nl], 1)).max()) if nl else 0.0,
            "live_counts_equal_steps": int((live_diff == 0).sum()), "steps_total": int(nl),
            "depth_rel_err_converged": {"max": float(rel.max()), "p99": float(np.quantile(rel, 0.99)),
                                        "over_1e-4": int((rel > 1e-4).sum()), "n": int(rel.size)},
            "rays_in_band_either": int(band2.sum()),
            "status_differ_outside_band_either": int((st_diff & ~band2).sum()),
            "steps_differ_outside_band_either": int((sp_diff & ~band2).sum()),
            "depth_rel_err_converged_outside_band_either": {
                "max": float(rel2.max()), "p99": float(np.quantile(rel2, 0.99)),
                "over_1e-4": int((rel2 > 1e-4).sum()), "n": int(rel2.size)},
            "depth_rel_err_same_steps": {"max": float(rel_same.max()), "p99": float(np.quantile(rel_same, 0.99)),
                                         "over_1e-4": int((rel_same > 1e-4).sum()), "n": int(rel_same.size)},
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
