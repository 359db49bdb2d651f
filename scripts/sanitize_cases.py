"""Small trace + objective cases for compute-sanitizer (memcheck,
racecheck, synccheck on the parity configs).

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py tiny64 fp64
    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py geo64 fp16x3

Each case traces the golden view, renders maps + normals and runs one fused
objective (depth + silhouette) so every kernel of the iterate launches at
least once; the script prints the launch count and exits 0.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import cfg_from, golden_weights, load_golden  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny64"
    prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
    import torch
    import paper_1911_13225_b200 as st
    from paper_1911_13225_b200 import _lib
    g = load_golden(f"{name}.npz")
    res = int(g["res"])
    if name == "tiny64":
        net = st.NeuralField(golden_weights(g), latent_dim=2, precision=prec)
    else:
        net = st.NeuralField.geometric(256, (512,) * 8, int(g["seed"]), precision=prec)
    intr, pose = st.Intrinsics(width=res, height=res), st.Pose(g["omega"], g["t"])
    cfg = st.TraceConfig(**cfg_from(g["cfg"]))
    code = g["code"]
    r = st.trace(net, code, intr, pose, cfg)
    st.render(net, code, intr, pose, cfg)
    obs = [st.Observation("depth", g["obs_depth"])]
    sil = (np.isfinite(g["obs_depth"])).astype(np.float64)
    obs.append(st.Observation("silhouette", sil))
    tot, terms, grad, n_conv, q = st.completion_objective(net, code, obs, intr, pose, cfg,
                                                          st.LossWeights())
    # the batched optimiser path with the ReLU-mask record (tensor-core modes)
    if prec in ("fp16x3", "bf16x3"):
        views = [(intr, pose)]
        opt = st.LatentOptimizer(net, views, {"depth": g["obs_depth"][None]}, code[None], cfg,
                                 relu_masks=True, max_iters=2)
        opt.step()
        opt.step()
    torch.cuda.synchronize()
    print(f"{name} {prec}: queries {r.total_queries} loss {tot:.6g} |g| {np.linalg.norm(grad):.6g} "
          f"launches {_lib.lib().dist_launch_count()}")


if __name__ == "__main__":
    main()
