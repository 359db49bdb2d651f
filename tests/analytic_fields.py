"""Closed-form fields for the plugin-seam tests (TEST INFRASTRUCTURE).

The reference keeps its analytic SDFs as test oracles (SURVEY 2.1 row 3:
out of scope for the product path).  These are independent minimal
restatements with the duck-typed field protocol (`latent_dim`, `evaluate`,
`spatial_gradient`; tracer.py:165, fields.py:45-88), plus the fakes of the
reference's tests (NanField, test_tracer.py:172-178; ConstField,
test_shading.py:20-29), and the closed-form sphere depth of oracles.py:25-44.
"""
from __future__ import annotations

import numpy as np


def _p(points):
    p = np.asarray(points, dtype=np.float64)
    return p[None, :] if p.ndim == 1 else p


class Sphere:
    latent_dim = 0

    def __init__(self, radius=0.5, center=(0.0, 0.0, 0.0)):
        self.r = float(radius)
        self.c = np.asarray(center, dtype=np.float64)

    def evaluate(self, points, code=None):
        return np.linalg.norm(_p(points) - self.c, axis=1) - self.r

    def spatial_gradient(self, points):
        q = _p(points) - self.c
        n = np.linalg.norm(q, axis=1, keepdims=True)
        return np.divide(q, n, out=np.zeros_like(q), where=n > 0)


class Plane:
    latent_dim = 0

    def __init__(self, normal=(0.0, 0.0, 1.0), offset=0.0):
        n = np.asarray(normal, dtype=np.float64)
        self.n = n / np.linalg.norm(n)
        self.off = float(offset)

    def evaluate(self, points, code=None):
        return _p(points) @ self.n - self.off

    def spatial_gradient(self, points):
        return np.broadcast_to(self.n, _p(points).shape).copy()


class NanField:
    """NaN everywhere, or only where x > x_nan (partial)."""
    latent_dim = 0

    def __init__(self, x_nan=None, base=None):
        self.x_nan, self.base = x_nan, base

    def evaluate(self, points, code=None):
        p = _p(points)
        if self.x_nan is None:
            return np.full(len(p), np.nan)
        f = self.base.evaluate(p)
        f[p[:, 0] > self.x_nan] = np.nan
        return f


def sphere_depth_image(intr, pose, radius=0.5):
    """Camera z of a centred sphere per pixel from the pinhole model, +inf on a
    miss (the quadratic of oracles.py:25-44, rebuilt independently)."""
    R, c = pose.rotation(), pose.center()
    cx, cy = intr.center
    i, j = np.meshgrid(np.arange(intr.width), np.arange(intr.height))
    hom = np.stack([(i + 0.5 - cx) / intr.fx, (j + 0.5 - cy) / intr.fy, np.ones(i.shape)], -1)
    nrm = np.linalg.norm(hom, axis=-1)
    v = (hom / nrm[..., None]).reshape(-1, 3) @ R
    b = v @ c
    disc = b * b - (float(c @ c) - radius * radius)
    t = np.where(disc >= 0.0, -b - np.sqrt(np.maximum(disc, 0.0)), np.inf)
    z = (t / nrm.ravel()).reshape(intr.height, intr.width)
    return np.where(np.isfinite(z), z, np.inf)
