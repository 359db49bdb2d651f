"""Maps and differentiable heads -- drop-in for the reference shading.py.

Maps (depth, mask, soft silhouette, normals) are computed on the device from
the resident trace (dist_maps / dist_normals) and returned as numpy images of
the reference's shapes.  `HeadBundle` rebuilds the frozen sample record (the
reference's layout, for drop-in callers) and runs every taped re-evaluation
and reverse sweep on the GPU through dist_eval / dist_eval_vjp
(shading.py:156-281).  The optimisation loop uses the fused device-side
version instead (dist_objective, csrc/heads.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .tracer import CONVERGED, TraceResult, trace


def _view_slice(result: TraceResult):
    dt = result.device
    n = dt.W * dt.H
    return dt, slice(result.view * n, (result.view + 1) * n)


def device_maps(dt, want_depth=True, want_mask=True, want_sil=True):
    """All V views' depth [V,H,W] (+inf bg), mask, soft silhouette on the device."""
    import torch
    n = dt.V * dt.W * dt.H
    depth = torch.empty(n, dtype=torch.float64, device="cuda") if want_depth else None
    mask = torch.empty(n, dtype=torch.uint8, device="cuda") if want_mask else None
    sil = torch.empty(n, dtype=torch.float64, device="cuda") if want_sil else None
    c = _lib.config_struct(dt.cfg)
    st = dt.state_struct()
    _lib.check(_lib.lib().dist_maps(dt.cams.data_ptr(), dt.V, dt.W, dt.H, C.byref(c), C.byref(st),
                                    _lib.ptr(depth), _lib.ptr(mask), _lib.ptr(sil),
                                    _lib.stream_ptr()))
    shp = (dt.V, dt.H, dt.W)
    return (None if depth is None else depth.view(shp), None if mask is None else mask.view(shp),
            None if sil is None else sil.view(shp))


def device_normals(dt):
    """normal_map of all V views on the device: [V,H,W,3]."""
    import torch
    h = dt.field.handle()
    n = dt.V * dt.W * dt.H
    out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    S = 1 if dt.codes is None else dt.codes.shape[0]
    lib = _lib.lib()
    ws = _lib.workspace(lib.dist_normals_workspace_size(h, dt.V, dt.W, dt.H, S))
    c = _lib.config_struct(dt.cfg)
    st = dt.state_struct()
    _lib.check(lib.dist_normals(h, _lib.ptr(dt.codes), S, dt.cams.data_ptr(), dt.V, dt.W, dt.H,
                                C.byref(c), C.byref(st), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                _lib.stream_ptr()))
    return out.view(dt.V, dt.H, dt.W, 3)


def _host(result: TraceResult, idx: int):
    maps = getattr(result, "_maps_cache", None)
    if maps is None:
        d, m, s = device_maps(result.device)
        v = result.view
        maps = (d[v].cpu().numpy(), m[v].cpu().numpy().astype(bool), s[v].cpu().numpy())
        result._maps_cache = maps
    return maps[idx]


def ray_distance(state, i: int, alpha: float) -> float:
    """shading.py:29-33."""
    if state.status[i] != CONVERGED:
        raise ValueError(f"ray {i} has not converged (status {state.status[i]})")
    return float(state.d[i] + (1.0 - alpha) * state.b[i])


def hard_mask(result: TraceResult) -> np.ndarray:
    """shading.py:48-52."""
    return _host(result, 1).copy()


def depth_map(result: TraceResult) -> np.ndarray:
    """Camera-space z per pixel, +inf background (shading.py:55-61)."""
    return _host(result, 0).copy()


def soft_silhouette(result: TraceResult) -> np.ndarray:
    """Signed soft occupancy (shading.py:97-113)."""
    return _host(result, 2).copy()


def surface_points(result: TraceResult):
    """World-space converged hit points and their ray indices (shading.py:64-70)."""
    s = result.state
    idx = np.nonzero(s.status == CONVERGED)[0]
    d = (s.d + (1.0 - result.config.alpha) * s.b)[idx]
    return s.bundle.origin + d[:, None] * s.bundle.dirs[idx], idx


def normal_map(result: TraceResult, field=None, code=None) -> np.ndarray:
    """Unit normals by six-probe central differences (shading.py:73-94)."""
    dt = result.device
    if field is not None and field is not dt.field:
        raise ValueError("normal_map must use the field the trace was computed with")
    if dt.external:
        return _external_normals(result, dt.field, dt.codes if code is None else code)
    return device_normals(dt)[result.view].cpu().numpy()


def _external_normals(result: TraceResult, field, code):
    """normal_map for a caller-evaluated field (the plugin seam): the six
    probes around each converged surface point go through the field's own
    evaluate, once, as shading.py:84-87 queries it."""
    pts, idx = surface_points(result)
    st = result.state
    out = np.zeros((st.bundle.height, st.bundle.width, 3))
    if idx.size == 0:
        return out
    delta = result.config.normal_delta
    offs = np.concatenate([np.eye(3), -np.eye(3)], axis=0) * delta
    f = np.asarray(field.evaluate((pts[:, None, :] + offs[None]).reshape(-1, 3), code),
                   dtype=np.float64).reshape(-1, 6)
    raw = (f[:, :3] - f[:, 3:]) / (2.0 * delta)
    nrm = np.linalg.norm(raw, axis=1, keepdims=True)
    unit = np.where(nrm > 0.0, raw / np.where(nrm > 0.0, nrm, 1.0), 0.0)
    out[st.bundle.pixels[idx, 1], st.bundle.pixels[idx, 0]] = unit
    return out


def attribute_map(result: TraceResult, attr_field, code=None) -> np.ndarray:
    """Surface attributes (colour) per converged pixel, zero background
    (shading.py:116-126)."""
    pts, idx = surface_points(result)
    m = getattr(attr_field, "out_dim", 3)
    b = result.state.bundle
    img = np.zeros((b.height, b.width, m))
    if idx.size:
        img[b.pixels[idx, 1], b.pixels[idx, 0]] = attr_field.evaluate(pts, code)
    return img


@dataclass
class RenderMaps:
    """shading.py:129-135."""
    depth: np.ndarray
    normal: np.ndarray
    silhouette: np.ndarray
    mask: np.ndarray
    attribute: np.ndarray | None = None


def render(field, code, intr, pose, cfg=None, attr_field=None, attr_code=None,
           with_normals: bool = True) -> RenderMaps:
    """Trace and assemble every map (shading.py:138-150)."""
    result = trace(field, code, intr, pose, cfg)
    normal = normal_map(result) if with_normals else np.zeros((intr.height, intr.width, 3))
    attr = attribute_map(result, attr_field, attr_code) if attr_field is not None else None
    return RenderMaps(depth=depth_map(result), normal=normal, silhouette=soft_silhouette(result),
                      mask=hard_mask(result), attribute=attr)


# === differentiable heads (shading.py:156-288) ================================

class HeadBundle:
    """Taped surrogates over the frozen marching record of one traced view.

    Same attributes and `backward` contract as the reference HeadBundle:
    depth head d_k + f(p_k, z) per selected sample, silhouette head
    f(p_best, z) - eps per recorded pixel, normal head from six probes per
    converged pixel.  The sample bookkeeping mirrors the reference's record
    layout on the host; every decoder evaluation and the reverse sweep run on
    the GPU (NeuralField.vjp_device -> dist_eval_vjp).
    """

    def __init__(self, result: TraceResult, field, code=None, want_normals: bool = False,
                 want_weights: bool = False):
        if want_weights:
            raise ValueError("weight gradients are outside the B200 hot path")
        st, cfg = result.state, result.config
        self._field, self._code, self._cfg = field, code, cfg
        rec = np.flatnonzero(np.isfinite(st.topk_absf[:, 0]))
        self.ray_index = rec
        self.pixels = st.bundle.pixels[rec]
        self.converged = st.status[rec] == CONVERGED
        self.scale = st.bundle.scale[rec]
        finite = np.isfinite(st.topk_absf[rec])
        counts = finite.sum(axis=1)
        pix_of, slot_of = np.nonzero(finite)          # row-major: pixel order, then slot
        self.sample_pixel = pix_of
        self.sample_weight = 1.0 / counts[pix_of]
        self.sample_d = st.topk_d[rec[pix_of], slot_of]
        self.best_sample = np.searchsorted(pix_of, np.arange(rec.size))
        dirs = st.bundle.dirs[rec]
        self._origin = st.bundle.origin
        pts = self._origin + self.sample_d[:, None] * dirs[pix_of]
        self._m = pts.shape[0]
        self._conv_rows = np.flatnonzero(self.converged)
        self._want_normals = bool(want_normals and self._conv_rows.size)
        if self._want_normals:
            dsurf = (st.d + (1.0 - cfg.alpha) * st.b)[rec[self._conv_rows]]
            surf = self._origin + dsurf[:, None] * dirs[self._conv_rows]
            off = np.concatenate([np.eye(3), -np.eye(3)]) * cfg.normal_delta
            probes = (surf[:, None, :] + off[None]).reshape(-1, 3)
            pts = np.concatenate([pts, probes])
        self._pts = pts
        self._assemble(self._eval(code))

    def _eval(self, code) -> np.ndarray:
        if self._pts.shape[0] == 0:
            return np.zeros(0)
        return self._field.evaluate(self._pts, code)

    def _assemble(self, vals: np.ndarray) -> None:
        cfg = self._cfg
        m = self._m
        self.sample_f = vals[:m]
        self.depth_value = self.sample_d + self.sample_f
        self.depth_z = self.depth_value * self.scale[self.sample_pixel]
        self.sil_value = self.sample_f[self.best_sample] - cfg.epsilon
        self.normal_value = np.zeros((self.pixels.shape[0], 3))
        self._raw_norm = np.zeros(self._conv_rows.size)
        if self._want_normals:
            f6 = vals[m:].reshape(-1, 6)
            raw = (f6[:, :3] - f6[:, 3:]) / (2.0 * cfg.normal_delta)
            nrm = np.linalg.norm(raw, axis=1)
            unit = np.divide(raw, nrm[:, None], out=np.zeros_like(raw), where=nrm[:, None] > 0.0)
            self.normal_value[self._conv_rows] = unit
            self._raw_norm = nrm

    def depth_image(self, height: int, width: int) -> np.ndarray:
        img = np.full((height, width), np.inf)
        r = self._conv_rows
        img[self.pixels[r, 1], self.pixels[r, 0]] = self.depth_z[self.best_sample[r]]
        return img

    def evaluate_at(self, code):
        """Replay the surrogates at another code (frozen positions)."""
        fresh = HeadBundle.__new__(HeadBundle)
        fresh.__dict__.update(self.__dict__)
        fresh._assemble(self._eval(code))
        return fresh.depth_value, fresh.sil_value, fresh.normal_value

    def backward(self, depth_seed=None, sil_seed=None, normal_seed=None) -> dict:
        """Seeded gradients: {"code", "sample_point_grads", ["surface_point_grads"]}."""
        import torch
        m = self._m
        seed = np.zeros(self._pts.shape[0])
        if depth_seed is not None:
            seed[:m] += np.asarray(depth_seed, dtype=np.float64)
        if sil_seed is not None:
            np.add.at(seed, self.best_sample, np.asarray(sil_seed, dtype=np.float64))
        if normal_seed is not None and self._want_normals:
            ns = np.asarray(normal_seed, dtype=np.float64)[self._conv_rows]
            ok = self._raw_norm > 0.0
            u = self.normal_value[self._conv_rows]
            proj = ns - u * np.einsum("ij,ij->i", u, ns)[:, None]
            rs = np.where(ok[:, None], proj / np.where(ok, self._raw_norm, 1.0)[:, None], 0.0)
            pp = np.concatenate([rs, -rs], axis=1) / (2.0 * self._cfg.normal_delta)
            seed[m:] = pp.reshape(-1)
        D = getattr(self._field, "latent_dim", 0) if hasattr(self._field, "vjp_device") else 0
        if self._pts.shape[0] == 0:
            out = {"sample_point_grads": np.zeros((0, 3))}
            if D:
                out["code"] = np.zeros(D)
            return out
        if hasattr(self._field, "vjp_device"):
            _, gc, gp = self._field.vjp_device(torch.from_numpy(self._pts), self._code,
                                               torch.from_numpy(seed))
            gp = gp.cpu().numpy()
        else:
            # an analytic field through the plugin seam: the reference's custom
            # node, d/dp = seed * spatial_gradient (fields.py:362-373)
            gp = seed[:, None] * np.asarray(self._field.spatial_gradient(self._pts), dtype=np.float64)
        if not np.all(np.isfinite(gp)):
            raise FloatingPointError("non-finite gradient for leaf 'points'")
        out = {"sample_point_grads": gp[:m]}
        if self._want_normals:
            out["surface_point_grads"] = gp[m:].reshape(-1, 6, 3).sum(axis=1)
        if D:
            g = gc.cpu().numpy()[0]
            if not np.all(np.isfinite(g)):
                raise FloatingPointError("non-finite gradient for leaf 'code'")
            out["code"] = g
        return out


def diff_heads(result: TraceResult, field, code=None, want_normals: bool = False,
               want_weights: bool = False) -> HeadBundle:
    """shading.py:284-288."""
    return HeadBundle(result, field, code, want_normals=want_normals, want_weights=want_weights)
