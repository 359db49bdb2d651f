"""Loss terms -- drop-in for the reference losses.py:21-117.

`Observation` and `LossWeights` are the reference's value types.  The loss
functions below take a `HeadBundle` and return (value, seed) exactly like the
reference, for callers that drive the heads by hand.  The optimisation loop
itself never calls them: dist_objective computes the same seeds inside the
fused head kernel (csrc/heads.cu).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np


@dataclass
class Observation:
    """losses.py:21-42: depth / silhouette / normal image with an optional trust mask."""
    kind: str
    image: np.ndarray
    mask: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in ("depth", "silhouette", "normal", "color"):
            raise ValueError(f"unknown observation kind {self.kind!r}")
        self.image = np.asarray(self.image, dtype=np.float64)

    def valid(self) -> np.ndarray:
        ok = np.isfinite(self.image)
        if ok.ndim == 3:
            ok = ok.all(axis=2)
        return ok if self.mask is None else (ok & self.mask)


@dataclass
class LossWeights:
    """losses.py:45-51."""
    depth: float = 10.0
    silhouette: float = 1.0
    normal: float = 1.0
    photometric: float = 5.0
    latent: float = 1.0


def depth_loss(heads, obs: Observation):
    """Masked camera-z L1, each pixel's samples sharing one unit of weight (losses.py:54-75)."""
    m = heads.sample_d.shape[0]
    px = heads.pixels
    valid = heads.converged & obs.valid()[px[:, 1], px[:, 0]]
    n_px = int(valid.sum())
    if n_px == 0:
        warnings.warn("depth loss: no overlap between observation and render", RuntimeWarning)
        return 0.0, np.zeros(m)
    ok = valid[heads.sample_pixel]
    sp = px[heads.sample_pixel]
    r = np.where(ok, heads.depth_z - obs.image[sp[:, 1], sp[:, 0]], 0.0)
    w = np.where(ok, heads.sample_weight / n_px, 0.0)
    return float(np.sum(w * np.abs(r))), w * np.sign(r) * heads.scale[heads.sample_pixel]


def silhouette_loss(soft, target):
    """Hinge on the signed soft silhouette (losses.py:78-91)."""
    t = np.asarray(target, dtype=np.float64)
    if t.shape != soft.shape:
        raise ValueError("silhouette shapes differ")
    n = soft.size
    val = float(np.sum(t * np.maximum(soft, 0.0) + (1.0 - t) * np.maximum(-soft, 0.0))) / n
    return val, (t * (soft > 0.0) - (1.0 - t) * (soft < 0.0)) / n


def normal_loss(heads, obs: Observation):
    """Mean -n.n_obs over valid, non-degenerate pixels (losses.py:94-111)."""
    p = heads.pixels.shape[0]
    px = heads.pixels
    nob = obs.image[px[:, 1], px[:, 0]]
    valid = heads.converged & (np.linalg.norm(heads.normal_value, axis=1) > 0.0) & \
        obs.valid()[px[:, 1], px[:, 0]]
    n = int(valid.sum())
    seed = np.zeros((p, 3))
    if n == 0:
        return 0.0, seed
    seed[valid] = -nob[valid] / n
    return -float(np.einsum("ij,ij->", heads.normal_value[valid], nob[valid])) / n, seed


def latent_reg(code):
    """|z|^2 and its gradient (losses.py:114-117)."""
    z = np.asarray(code, dtype=np.float64)
    return float(z @ z), 2.0 * z
