"""Synthetic workloads of BASELINE.json.

Standard decoder: `NeuralField.geometric(256, (512,)*8, seed=0)`; target code
z* = N(0, 0.1^2) from default_rng(1); views on the ring of
test_acceptance.py:297-302; observations are depth maps rendered from z* with
TraceConfig(k_samples=3); optimisation starts at z0 = 0.
"""

from __future__ import annotations

import numpy as np

from .camera import Intrinsics, look_at


def ring_eye(k: int, n: int, radius: float = 2.0) -> np.ndarray:
    th = 2.0 * np.pi * k / n
    eye = np.array([2.0 * np.sin(th), 0.6 * np.sin(2.0 * th + 0.4), -2.0 * np.cos(th)])
    return eye * (radius / np.linalg.norm(eye))


def ring_views(n_views: int, res: int, first: int = 0, total: int | None = None, stride: int = 1):
    """Views first, first+stride, ... (n_views of them) of a `total`-view ring at
    res x res.  stride = world size interleaves the ring over ranks, so every
    rank sees the whole ring (balanced per-rank cost)."""
    total = total or n_views * stride
    intr = Intrinsics(width=res, height=res)
    return [(intr, look_at(ring_eye(first + j * stride, total))) for j in range(n_views)]


def target_code(seed: int = 1, dim: int = 256) -> np.ndarray:
    return np.random.default_rng(seed).normal(0.0, 0.1, dim)


def render_depth_observations(field, code, views, cfg):
    """[V,H,W] depth maps of `code` from `views` (rendered on the device)."""
    from .shading import device_maps
    from .tracer import trace_views
    dt = trace_views(field, code, views, cfg)
    depth, _, _ = device_maps(dt, True, False, False)
    return depth
