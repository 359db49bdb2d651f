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


# === photometric consistency (losses.py:120-222) ============

def to_gray(img):
    """Channel mean of a colour image (losses.py:123-125)."""
    img = np.asarray(img, dtype=np.float64)
    return img.mean(axis=2) if img.ndim == 3 else img


def bilinear_sample(img, u, v):
    """Pixel-centre bilinear sample with border clamping, plus d/du and d/dv
    (losses.py:128-150).  Host utility; the warp itself runs on the device."""
    h, w = img.shape
    xs = np.clip(u - 0.5, 0.0, w - 1.0)
    ys = np.clip(v - 0.5, 0.0, h - 1.0)
    x0 = np.clip(np.floor(xs).astype(np.int64), 0, w - 2) if w > 1 else np.zeros_like(xs, np.int64)
    y0 = np.clip(np.floor(ys).astype(np.int64), 0, h - 2) if h > 1 else np.zeros_like(ys, np.int64)
    x1, y1 = np.minimum(x0 + 1, w - 1), np.minimum(y0 + 1, h - 1)
    fx, fy = xs - x0, ys - y0
    a, b, c, d = img[y0, x0], img[y0, x1], img[y1, x0], img[y1, x1]
    val = (a * (1 - fx) + b * fx) * (1 - fy) + (c * (1 - fx) + d * fx) * fy
    return val, (b - a) * (1 - fy) + (d - c) * fy, (c - a) * (1 - fx) + (d - b) * fx


def _photometric_device(z_i, gray_i, intr_i, pose_i, gray_j, intr_j, pose_j, z_j, thresh):
    import torch

    from . import _lib
    from .camera import camera_struct
    _lib.require_device()
    z_i = np.asarray(z_i, dtype=np.float64)
    h, w = z_i.shape
    hj, wj = np.asarray(z_j).shape
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()  # noqa: E731
    cams = _lib.cameras_to_device([camera_struct(intr_i, pose_i), camera_struct(intr_j, pose_j)])
    zi, gi, gj, zj = dev(z_i), dev(gray_i), dev(gray_j), dev(z_j)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    dz = torch.empty(h * w, dtype=torch.float64, device="cuda")
    vis = torch.empty(h * w, dtype=torch.uint8, device="cuda")
    lib = _lib.lib()
    ws = _lib.workspace(lib.dist_photometric_workspace_size(h, w))
    _lib.check(lib.dist_photometric(cams.data_ptr(), h, w, hj, wj, zi.data_ptr(), gi.data_ptr(),
                                    gj.data_ptr(), zj.data_ptr(), float(thresh), loss.data_ptr(),
                                    dz.data_ptr(), vis.data_ptr(), ws.data_ptr(), ws.numel(),
                                    _lib.stream_ptr()))
    lv = loss.cpu().numpy()
    return float(lv[0]), dz.cpu().numpy().reshape(h, w), vis.cpu().numpy().reshape(h, w).astype(bool)


def visibility_mask(z_i, intr_i, pose_i, z_j, intr_j, pose_j, thresh: float = 0.001):
    """Pixels of view i whose surface point view j also sees (losses.py:159-183)."""
    zeros = np.zeros_like(np.asarray(z_i, dtype=np.float64))
    zj = np.asarray(z_j, dtype=np.float64)
    return _photometric_device(z_i, zeros, intr_i, pose_i, np.zeros_like(zj), intr_j, pose_j,
                               zj, thresh)[2]


def photometric_loss(z_i, gray_i, intr_i, pose_i, gray_j, intr_j, pose_j, z_j,
                     thresh: float = 0.001):
    """Mean L1 between view i and view j warped through i's depth, and dL/dz_i
    (losses.py:186-222), computed by the dist_photometric kernels."""
    loss, dz, _ = _photometric_device(z_i, gray_i, intr_i, pose_i, gray_j, intr_j, pose_j, z_j,
                                      thresh)
    return loss, dz
