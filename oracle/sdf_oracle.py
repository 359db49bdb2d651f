"""CPU oracle for the DIST sphere-tracing hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy float64 restatement of the reference `sdftrace`
algorithm for the hot path.  It exists so that the
parity tests, `__graft_entry__.smoke()` and the `cpu_baseline` leg of
`bench.py` have a checker that travels to the GPU box (the reference tree does
not).  Nothing in the product package imports it; the product path fails loudly
when the CUDA library is missing.

Parity status: PINNED.  `oracle/make_golden.py` runs the unmodified reference
(imported from /root/reference in the build container) on the cases committed
under `tests/golden/`, and `tests/test_oracle_cpu.py` checks this restatement
against those fixtures (bitwise for ray state and query counts, 1e-12 for
floating outputs).

Every function cites the reference lines it restates (paths relative to
/root/reference/pkg/src/sdftrace/).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dfield

import numpy as np

MARCHING, CONVERGED, ESCAPED, EXHAUSTED = 0, 1, 2, 3   # tracer.py:24


# --------------------------------------------------------------------------
# camera (camera.py:25-61, 104-166, 177-212)
# --------------------------------------------------------------------------

def rodrigues(omega) -> np.ndarray:
    """Axis-angle -> rotation (camera.py:104-113)."""
    w = np.asarray(omega, dtype=np.float64)
    th = np.linalg.norm(w)
    K = np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])
    if th < 1e-12:
        return np.eye(3) + K + 0.5 * (K @ K)
    return np.eye(3) + (np.sin(th) / th) * K + ((1.0 - np.cos(th)) / th**2) * (K @ K)


def rotation_log(R) -> np.ndarray:
    """Rotation -> axis-angle (camera.py:135-151)."""
    R = np.asarray(R, dtype=np.float64)
    th = np.arccos(np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0))
    vee = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if th < 1e-8:
        return 0.5 * vee
    if np.pi - th < 1e-6:
        A = (R + np.eye(3)) / 2.0
        ax = np.sqrt(np.clip(np.diag(A), 0.0, None))
        k = int(np.argmax(ax))
        ax = A[:, k] / ax[k]
        return th * ax / np.linalg.norm(ax)
    return th / (2.0 * np.sin(th)) * vee


@dataclass
class Cam:
    """Pinhole camera: fx = focal/sensor*W, centre W/2,H/2 (camera.py:25-61);
    world-to-camera p_c = R p + t, centre c = -R^T t (camera.py:157-172)."""
    width: int
    height: int
    omega: np.ndarray
    t: np.ndarray
    focal_mm: float = 60.0
    sensor_mm: float = 32.0

    @property
    def fx(self) -> float:
        return self.focal_mm / self.sensor_mm * self.width

    @property
    def R(self) -> np.ndarray:
        return rodrigues(self.omega)

    @property
    def origin(self) -> np.ndarray:
        return -self.R.T @ self.t


def cam_look_at(eye, width, height, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0),
                focal_mm=60.0, sensor_mm=32.0) -> Cam:
    """camera.py:183-195."""
    eye = np.asarray(eye, dtype=np.float64)
    z = np.asarray(target, dtype=np.float64) - eye
    z = z / np.linalg.norm(z)
    x = np.cross(z, np.asarray(up, dtype=np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z], axis=0)
    return Cam(width, height, rotation_log(R), -R @ eye, focal_mm, sensor_mm)


def ring_eye(k: int, n: int, radius: float = 2.0) -> np.ndarray:
    """The multi-view ring of test_acceptance.py:297-302."""
    th = 2.0 * np.pi * k / n
    eye = np.array([2.0 * np.sin(th), 0.6 * np.sin(2.0 * th + 0.4), -2.0 * np.cos(th)])
    return eye * (radius / np.linalg.norm(eye))


@dataclass
class Rays:
    origin: np.ndarray
    dirs: np.ndarray
    pixels: np.ndarray
    scale: np.ndarray
    width: int
    height: int


def cam_rays(cam: Cam, level: int = 1) -> Rays:
    """Pixel-centre rays of the 1/level grid, row-major (camera.py:190-212)."""
    w, h = cam.width // level, cam.height // level
    cx, cy = cam.width / 2.0, cam.height / 2.0
    jj, ii = np.divmod(np.arange(w * h), w)
    v = np.empty((w * h, 3))
    v[:, 0] = ((ii + 0.5) * level - cx) / cam.fx
    v[:, 1] = ((jj + 0.5) * level - cy) / cam.fx
    v[:, 2] = 1.0
    nrm = np.linalg.norm(v, axis=1)
    dirs = (v / nrm[:, None]) @ cam.R
    return Rays(cam.origin, dirs, np.stack([ii, jj], 1).astype(np.int64),
                1.0 / nrm, w, h)


# --------------------------------------------------------------------------
# decoder (fields.py:185-291)
# --------------------------------------------------------------------------

@dataclass
class Decoder:
    """Latent-conditioned MLP on concat(code, p) (fields.py:185-247).

    skip: index of the layer whose input is concat(h, code, p) (DeepSDF skip
    layout); -1 = the reference's plain stack.
    """
    weights: list
    latent_dim: int
    final: str = "tanh"
    skip: int = -1

    def _x(self, pts, code):
        pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
        if self.latent_dim == 0:
            return pts
        z = np.broadcast_to(np.asarray(code, dtype=np.float64), (pts.shape[0], self.latent_dim))
        return np.concatenate([z, pts], axis=1)

    def forward(self, pts, code, keep=False):
        """Plain forward; keep=True also returns pre-activations (fields.py:239-247)."""
        x = self._x(pts, code)
        h = x
        pre = []
        L = len(self.weights)
        for i, (W, b) in enumerate(self.weights):
            if i == self.skip:
                h = np.concatenate([h, x], axis=1)
            a = h @ W + b
            pre.append((h, a))
            if i < L - 1:
                h = np.maximum(a, 0.0)
            else:
                h = np.tanh(a) if self.final == "tanh" else a
        return (h[:, 0], pre) if keep else h[:, 0]

    def __call__(self, pts, code):
        return self.forward(pts, code)

    def backward(self, pts, code, seed):
        """VJP of sum(seed * f) w.r.t. code and points (autodiff.py:95-129,175-200,220-255)."""
        f, pre = self.forward(pts, code, keep=True)
        L = len(self.weights)
        g = np.asarray(seed, dtype=np.float64)[:, None]
        if self.final == "tanh":
            g = g * (1.0 - f[:, None] ** 2)
        gx = None
        for i in range(L - 1, -1, -1):
            W, _ = self.weights[i]
            h_in, a = pre[i]
            if i < L - 1:
                g = g * (a > 0.0)
            gin = g @ W.T
            if i == self.skip:
                d_in = gin.shape[1] - (self.latent_dim + 3)
                gx = gin[:, d_in:] if gx is None else gx + gin[:, d_in:]
                gin = gin[:, :d_in]
            g = gin
        gx = g if gx is None else gx + g
        D = self.latent_dim
        return {"code": gx[:, :D].sum(axis=0), "points": gx[:, D:], "f": f}


def he_init(latent_dim, hidden, seed):
    """NeuralField.init recipe (fields.py:209-219): He normal, last layer x0.1."""
    rng = np.random.default_rng(seed)
    dims = [latent_dim + 3, *hidden, 1]
    ws = []
    for i, (p, q) in enumerate(zip(dims[:-1], dims[1:])):
        s = np.sqrt(2.0 / p) * (0.1 if i == len(dims) - 2 else 1.0)
        ws.append((rng.standard_normal((p, q)) * s, np.zeros(q)))
    return ws


def geometric_init(latent_dim=256, hidden=(512,) * 8, seed=0, skip=-1):
    """The standard synthetic decoder of SURVEY.md 8(d): a seeded geometric
    (SAL-style) init that produces a real surface.  Hidden W ~ N(0, 2/out),
    zero bias; latent rows of W0 x0.1; last layer N(sqrt(pi)/sqrt(n), 1e-4),
    bias -0.5.  With skip >= 0 the skip layer consumes concat(h, code, p) and
    its predecessor narrows so the skip layer input stays `hidden` wide."""
    rng = np.random.default_rng(seed)
    D = latent_dim
    outs = list(hidden)
    if skip > 0:
        outs[skip - 1] = hidden[skip - 1] - (D + 3)
    ins = [D + 3] + list(hidden)
    ws = []
    for i, o in enumerate(outs):
        W = rng.standard_normal((ins[i], o)) * (np.sqrt(2.0) / np.sqrt(o))
        if i == 0:
            W[:D] *= 0.1                       # latent rows
        elif i == skip:
            W[ins[i] - (D + 3):ins[i] - 3] *= 0.1
        ws.append((W, np.zeros(o)))
    n = hidden[-1]
    W = rng.normal(np.sqrt(np.pi) / np.sqrt(n), 1e-4, (n, 1))
    ws.append((W, np.full(1, -0.5)))
    return ws


# --------------------------------------------------------------------------
# tracer (tracer.py:27-252)
# --------------------------------------------------------------------------

@dataclass
class Cfg:
    """TraceConfig defaults (tracer.py:27-50)."""
    alpha: float = 1.5
    epsilon: float = 5e-5
    max_steps: int = 100
    k_samples: int = 1
    coarse_start_scale: int = 4
    split_interval: int = 3
    normal_delta: float = 1e-3
    use_dynamic_mask: bool = True


@dataclass
class Trace:
    rays: Rays
    d: np.ndarray
    b: np.ndarray
    status: np.ndarray
    steps: np.ndarray
    tk_d: np.ndarray
    tk_f: np.ndarray
    tk_a: np.ndarray
    band: np.ndarray
    margin_f: np.ndarray = None     # min over own+inherited queries of ||b| - eps|
    margin_esc: np.ndarray = None   # min over escape tests of min(|p|^2-1|, |v.p|, |b|)
    live_counts: list = dfield(default_factory=list)
    total_queries: int = 0
    nan_count: int = 0


BAND_F = 1e-5      # |(|b| - eps)| margin for the trajectory band
BAND_ESC = 1e-6    # margin on the escape-test quantities


def _init(rays: Rays, K: int) -> Trace:
    """Near unit-sphere intersection; misses escape (tracer.py:88-119)."""
    n = rays.dirs.shape[0]
    c = rays.origin
    c2 = float(c @ c)
    d = np.zeros(n)
    st = np.zeros(n, np.uint8)
    if c2 > 1.0:
        m = rays.dirs @ c
        disc = m * m - (c2 - 1.0)
        hit = (disc >= 0.0) & (m < 0.0)
        d[hit] = -m[hit] - np.sqrt(disc[hit])
        st[~hit] = ESCAPED
    return Trace(rays, d, np.full(n, np.nan), st, np.zeros(n, np.int64),
                 np.zeros((n, K)), np.zeros((n, K)), np.full((n, K), np.inf),
                 np.zeros(n, bool), np.full(n, np.inf), np.full(n, np.inf))


def _step(T: Trace, fn, cfg: Cfg, band_f=BAND_F, band_esc=BAND_ESC):
    """One march step (tracer.py:132-193), plus the band flags of SURVEY 8c."""
    live = T.status == MARCHING
    rows = np.nonzero(live)[0] if cfg.use_dynamic_mask else np.arange(T.d.size)
    queried = rows.size
    p = T.rays.origin + T.d[rows, None] * T.rays.dirs[rows]
    f = np.asarray(fn(p), dtype=np.float64)
    if not cfg.use_dynamic_mask:
        rows, f = rows[live[rows]], f[live[rows]]
    bad = ~np.isfinite(f)
    T.status[rows[bad]] = EXHAUSTED
    T.b[rows[bad]] = np.nan
    T.steps[rows[bad]] += 1
    rows, f = rows[~bad], f[~bad]
    dk = T.d[rows]
    a = np.abs(f)
    # strict-< insertion into the sorted record; ties keep the earlier sample
    for r, fv, av, dv in zip(rows, f, a, dk):
        K = T.tk_a.shape[1]
        if av < T.tk_a[r, K - 1]:
            pos = int(np.searchsorted(T.tk_a[r, :K - 1], av, side="right"))
            T.tk_a[r, pos + 1:] = T.tk_a[r, pos:K - 1].copy()
            T.tk_f[r, pos + 1:] = T.tk_f[r, pos:K - 1].copy()
            T.tk_d[r, pos + 1:] = T.tk_d[r, pos:K - 1].copy()
            T.tk_a[r, pos], T.tk_f[r, pos], T.tk_d[r, pos] = av, fv, dv
    T.steps[rows] += 1
    T.b[rows] = f
    T.d[rows] = dk + cfg.alpha * f
    conv = a < cfg.epsilon
    T.band[rows] |= np.abs(a - cfg.epsilon) < band_f
    T.margin_f[rows] = np.minimum(T.margin_f[rows], np.abs(a - cfg.epsilon))
    T.status[rows[conv]] = CONVERGED
    mv = rows[~conv]
    if mv.size:
        pn = T.rays.origin + T.d[mv, None] * T.rays.dirs[mv]
        r2 = np.einsum("ij,ij->i", pn, pn) - 1.0
        vp = np.einsum("ij,ij->i", T.rays.dirs[mv], pn)
        fm = f[~conv]
        esc = (r2 > 0.0) & (fm > 0.0) & (vp > 0.0)
        T.band[mv] |= (np.abs(r2) < band_esc) | (np.abs(vp) < band_esc) | (np.abs(fm) < band_esc)
        T.margin_esc[mv] = np.minimum(T.margin_esc[mv], np.minimum(np.minimum(np.abs(r2), np.abs(vp)),
                                                                    np.abs(fm)))
        T.status[mv[esc]] = ESCAPED
    return queried, int(bad.sum())


def _split(T: Trace, fine: Rays) -> Trace:
    """4-way split; converged children re-arm (tracer.py:196-218)."""
    par = (fine.pixels[:, 1] // 2) * T.rays.width + fine.pixels[:, 0] // 2
    st = T.status[par].copy()
    st[st == CONVERGED] = MARCHING
    return Trace(fine, T.d[par].copy(), T.b[par].copy(), st, T.steps[par].copy(),
                 T.tk_d[par].copy(), T.tk_f[par].copy(), T.tk_a[par].copy(),
                 T.band[par].copy(), T.margin_f[par].copy(), T.margin_esc[par].copy(),
                 T.live_counts, T.total_queries, T.nan_count)


def trace(fn, cam: Cam, cfg: Cfg, band_f=BAND_F, band_esc=BAND_ESC) -> Trace:
    """Coarse-to-fine trace with the global step budget (tracer.py:221-252).

    `band` flags rays whose own or inherited trajectory made a decision within
    band_f of epsilon (|b| test) or band_esc of zero (escape test) -- the
    exclusion set for exact per-ray parity."""
    s = cfg.coarse_start_scale
    levels = [l for l in (4, 2, 1) if l <= s]
    T = _init(cam_rays(cam, levels[0]), cfg.k_samples)
    done = 0
    for li, lv in enumerate(levels):
        if li:
            T = _split(T, cam_rays(cam, lv))
        budget = cfg.split_interval if lv > 1 else cfg.max_steps - done
        for _ in range(budget):
            if done >= cfg.max_steps or not np.any(T.status == MARCHING):
                break
            q, nn = _step(T, fn, cfg, band_f, band_esc)
            T.live_counts.append(q)
            T.total_queries += q
            T.nan_count += nn
            done += 1
    T.status[T.status == MARCHING] = EXHAUSTED
    return T


# --------------------------------------------------------------------------
# maps (shading.py:29-113)
# --------------------------------------------------------------------------

def _grid(T: Trace, vals, fill, ch=0):
    shp = (T.rays.height, T.rays.width) + ((ch,) if ch else ())
    img = np.full(shp, fill, dtype=np.float64)
    img[T.rays.pixels[:, 1], T.rays.pixels[:, 0]] = vals
    return img


def surf_dist(T: Trace, alpha: float):
    """d* = d + (1-alpha) b (shading.py:36-37)."""
    return T.d + (1.0 - alpha) * T.b


def depth_map(T: Trace, cfg: Cfg):
    """shading.py:55-61."""
    conv = T.status == CONVERGED
    return _grid(T, np.where(conv, surf_dist(T, cfg.alpha) * T.rays.scale, np.inf), np.inf)


def hard_mask(T: Trace):
    """shading.py:48-52."""
    return _grid(T, T.status == CONVERGED, 0.0).astype(bool)


def soft_silhouette(T: Trace, cfg: Cfg):
    """shading.py:97-113."""
    rec = np.isfinite(T.tk_a[:, 0])
    c = T.rays.origin
    m = T.rays.dirs @ c
    perp = np.sqrt(np.maximum(float(c @ c) - m * m, 0.0))
    vals = np.where(rec, T.tk_a[:, 0] - cfg.epsilon, perp - 1.0)
    return _grid(T, vals, np.nan)


def normal_map(T: Trace, fn, cfg: Cfg):
    """Six-probe central differences, zero-norm -> 0 (shading.py:73-94)."""
    idx = np.nonzero(T.status == CONVERGED)[0]
    img = np.zeros((T.rays.height, T.rays.width, 3))
    if idx.size == 0:
        return img
    pts = T.rays.origin + surf_dist(T, cfg.alpha)[idx, None] * T.rays.dirs[idx]
    off = np.concatenate([np.eye(3), -np.eye(3)]) * cfg.normal_delta
    f = np.asarray(fn((pts[:, None, :] + off[None]).reshape(-1, 3))).reshape(-1, 6)
    raw = (f[:, :3] - f[:, 3:]) / (2.0 * cfg.normal_delta)
    nrm = np.linalg.norm(raw, axis=1)
    unit = np.zeros_like(raw)
    ok = nrm > 0.0
    unit[ok] = raw[ok] / nrm[ok, None]
    img[T.rays.pixels[idx, 1], T.rays.pixels[idx, 0]] = unit
    return img


# --------------------------------------------------------------------------
# heads, losses, backward (shading.py:156-281, losses.py:21-117)
# --------------------------------------------------------------------------

@dataclass
class Heads:
    ray_index: np.ndarray
    pixels: np.ndarray
    converged: np.ndarray
    scale: np.ndarray
    sample_pixel: np.ndarray
    sample_weight: np.ndarray
    sample_d: np.ndarray
    best_sample: np.ndarray
    sample_pts: np.ndarray
    sample_f: np.ndarray
    depth_value: np.ndarray
    depth_z: np.ndarray
    sil_value: np.ndarray
    conv_rows: np.ndarray
    normal_value: np.ndarray
    raw_norm: np.ndarray
    probe_pts: np.ndarray | None


def heads(T: Trace, fn, cfg: Cfg, want_normals=False) -> Heads:
    """Frozen-sample surrogates d_k + f(p_k) (shading.py:166-225)."""
    rec = np.nonzero(np.isfinite(T.tk_a[:, 0]))[0]
    cnt = np.isfinite(T.tk_a[rec]).sum(axis=1)
    sp = np.repeat(np.arange(rec.size), cnt)
    slot = (np.arange(sp.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)).astype(np.int64)
    sd = T.tk_d[rec[sp], slot]
    best = np.searchsorted(sp, np.arange(rec.size))
    dirs = T.rays.dirs[rec]
    pts = T.rays.origin + sd[:, None] * dirs[sp]
    conv = T.status[rec] == CONVERGED
    crow = np.nonzero(conv)[0]
    probe = None
    if want_normals and crow.size:
        surf = T.rays.origin + surf_dist(T, cfg.alpha)[rec[crow], None] * dirs[crow]
        off = np.concatenate([np.eye(3), -np.eye(3)]) * cfg.normal_delta
        probe = (surf[:, None, :] + off[None]).reshape(-1, 3)
    allp = pts if probe is None else np.concatenate([pts, probe])
    vals = np.asarray(fn(allp), dtype=np.float64) if allp.shape[0] else np.zeros(0)
    f = vals[:pts.shape[0]]
    scale = T.rays.scale[rec]
    nv = np.zeros((rec.size, 3))
    rn = np.zeros(crow.size)
    if probe is not None:
        f6 = vals[pts.shape[0]:].reshape(-1, 6)
        raw = (f6[:, :3] - f6[:, 3:]) / (2.0 * cfg.normal_delta)
        rn = np.linalg.norm(raw, axis=1)
        ok = rn > 0.0
        u = np.zeros_like(raw)
        u[ok] = raw[ok] / rn[ok, None]
        nv[crow] = u
    return Heads(rec, T.rays.pixels[rec], conv, scale, sp, 1.0 / cnt[sp], sd, best,
                 pts, f, sd + f, (sd + f) * scale[sp], f[best] - cfg.epsilon if rec.size else f[:0],
                 crow, nv, rn, probe)


def depth_loss(H: Heads, z_obs_img, valid_img):
    """Masked camera-z L1 with per-pixel 1/count weights (losses.py:54-75)."""
    m = H.sample_d.size
    vpx = H.converged & valid_img[H.pixels[:, 1], H.pixels[:, 0]]
    n = int(vpx.sum())
    if n == 0:
        return 0.0, np.zeros(m)
    ok = vpx[H.sample_pixel]
    zo = z_obs_img[H.pixels[H.sample_pixel, 1], H.pixels[H.sample_pixel, 0]]
    r = np.where(ok, H.depth_z - zo, 0.0)
    w = np.where(ok, H.sample_weight / n, 0.0)
    return float(np.sum(w * np.abs(r))), w * np.sign(r) * H.scale[H.sample_pixel]


def silhouette_loss(soft, target):
    """Hinge on the signed soft silhouette (losses.py:78-91)."""
    t = np.asarray(target, dtype=np.float64)
    n = soft.size
    loss = float(np.sum(t * np.maximum(soft, 0.0) + (1.0 - t) * np.maximum(-soft, 0.0))) / n
    return loss, (t * (soft > 0.0) - (1.0 - t) * (soft < 0.0)) / n


def normal_loss(H: Heads, n_obs_img, valid_img):
    """Mean -n.n_obs over valid, non-degenerate pixels (losses.py:94-111)."""
    p = H.pixels.shape[0]
    ok = np.linalg.norm(H.normal_value, axis=1) > 0.0
    nob = n_obs_img[H.pixels[:, 1], H.pixels[:, 0]]
    v = H.converged & ok & valid_img[H.pixels[:, 1], H.pixels[:, 0]]
    n = int(v.sum())
    seed = np.zeros((p, 3))
    if n == 0:
        return 0.0, seed
    seed[v] = -nob[v] / n
    return -float(np.einsum("ij,ij->", H.normal_value[v], nob[v])) / n, seed


def heads_backward(H: Heads, dec: Decoder, code, cfg: Cfg, d_seed=None, s_seed=None,
                   n_seed=None):
    """Seeded VJP over samples + probes (shading.py:244-281)."""
    m = H.sample_d.size
    npr = 0 if H.probe_pts is None else H.probe_pts.shape[0]
    seed = np.zeros(m + npr)
    if d_seed is not None:
        seed[:m] += d_seed
    if s_seed is not None:
        np.add.at(seed, H.best_sample, s_seed)
    if n_seed is not None and npr:
        ns = np.asarray(n_seed)[H.conv_rows]
        rs = np.zeros_like(ns)
        ok = H.raw_norm > 0.0
        u = H.normal_value[H.conv_rows][ok]
        rs[ok] = (ns[ok] - u * np.einsum("ij,ij->i", u, ns[ok])[:, None]) / H.raw_norm[ok, None]
        pp = np.concatenate([rs, -rs], axis=1) / (2.0 * cfg.normal_delta)
        seed[m:] = pp.reshape(-1)
    allp = H.sample_pts if npr == 0 else np.concatenate([H.sample_pts, H.probe_pts])
    if allp.shape[0] == 0:
        return {"code": np.zeros(dec.latent_dim), "sample_point_grads": np.zeros((0, 3))}
    g = dec.backward(allp, code, seed)
    out = {"code": g["code"], "sample_point_grads": g["points"][:m]}
    if npr:
        out["surface_point_grads"] = g["points"][m:].reshape(-1, 6, 3).sum(axis=1)
    return out


@dataclass
class Weights:
    """LossWeights (losses.py:45-51)."""
    depth: float = 10.0
    silhouette: float = 1.0
    normal: float = 1.0
    photometric: float = 5.0
    latent: float = 1.0


def objective(dec: Decoder, code, cam: Cam, cfg: Cfg, w: Weights, depth=None,
              depth_valid=None, silhouette=None, normals=None, normals_valid=None,
              implicit=False):
    """completion_objective (optimize.py:102-138).  implicit=True replaces the
    surrogate depth gradient by the implicit one;
    implicit="unit" uses the unit normal in the denominator."""
    T = trace(lambda p: dec(p, code), cam, cfg)
    H = heads(T, lambda p: dec(p, code), cfg, want_normals=(normals is not None) or implicit)
    terms = {}
    ds = ss = ns = None
    if depth is not None:
        dv = np.isfinite(depth) if depth_valid is None else depth_valid & np.isfinite(depth)
        l, s = depth_loss(H, depth, dv)
        terms["depth"] = l
        ds = w.depth * s
        if implicit:
            ds = implicit_depth_seeds(H, ds, T.rays.dirs[H.ray_index], unit_normal=implicit == "unit")
    if silhouette is not None:
        l, gi = silhouette_loss(soft_silhouette(T, cfg), silhouette)
        terms["silhouette"] = l
        ss = w.silhouette * gi[H.pixels[:, 1], H.pixels[:, 0]]
    if normals is not None:
        nvld = np.isfinite(normals).all(axis=2)
        if normals_valid is not None:
            nvld &= normals_valid
        l, s = normal_loss(H, normals, nvld)
        terms["normal"] = l
        ns = w.normal * s
    z = np.asarray(code, dtype=np.float64)
    terms["latent"] = float(z @ z)
    g = heads_backward(H, dec, code, cfg, ds, ss, ns)["code"] + w.latent * 2.0 * z
    total = w.depth * terms.get("depth", 0.0) + w.silhouette * terms.get("silhouette", 0.0) \
        + w.normal * terms.get("normal", 0.0) + w.latent * terms["latent"]
    return total, terms, g, int(H.converged.sum()), T.total_queries, T


@dataclass
class Adam:
    """AdamState + adam_step (optimize.py:35-63)."""
    lr: float = 1e-2
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8
    m: np.ndarray | None = None
    v: np.ndarray | None = None
    t: int = 0
    skipped: int = 0

    def step(self, x, g):
        g = np.asarray(g, dtype=np.float64)
        if not np.all(np.isfinite(g)):
            self.skipped += 1
            return x.copy()
        if self.m is None:
            self.m, self.v = np.zeros_like(x), np.zeros_like(x)
        self.t += 1
        self.m = self.b1 * self.m + (1.0 - self.b1) * g
        self.v = self.b2 * self.v + (1.0 - self.b2) * g * g
        mh = self.m / (1.0 - self.b1 ** self.t)
        vh = self.v / (1.0 - self.b2 ** self.t)
        return x - self.lr * mh / (np.sqrt(vh) + self.eps)


IMPLICIT_GRAZING = 0.1


def implicit_depth_seeds(H: Heads, d_seed, cam_dirs_rec, unit_normal=False):
    """Implicit-gradient variant: per-sample depth seeds
    scaled by -1/(grad f . v) at converged pixels, grad f = the raw Eq. 3
    difference vector (normal_value * raw_norm), grazing pixels (grad f . v >=
    -IMPLICIT_GRAZING, factor > 10) excluded -- the rule of csrc/heads.cuh."""
    s = np.zeros_like(d_seed)
    if H.conv_rows.size == 0:
        return s
    gradf = H.normal_value[H.conv_rows] * (1.0 if unit_normal else H.raw_norm[:, None])
    gv = np.einsum("ij,ij->i", gradf, cam_dirs_rec[H.conv_rows])
    fac = np.zeros(H.pixels.shape[0])
    ok = gv < -IMPLICIT_GRAZING
    fac[H.conv_rows[ok]] = -1.0 / gv[ok]
    return d_seed * fac[H.sample_pixel]


def min_steps(d, alpha, theta, eps):
    """Eq. 9 bound (tracer.py:258-273) -- used only by oracle self-tests."""
    r = abs(1.0 - alpha * math.sin(theta))
    return max(1, math.ceil((math.log(eps) - math.log(d)) / math.log(r)))


# --------------------------------------------------------------------------
# camera pose gradient and recovery (camera.py:85-103,
# 215-278; optimize.py:185-266)
# --------------------------------------------------------------------------

def _hat(w):
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def rotation_partials(omega):
    """R and dR/d omega_i of the exponential map (camera.py:85-103)."""
    w = np.asarray(omega, dtype=np.float64)
    R = rodrigues(w)
    t2 = float(w @ w)
    if t2 < 1e-16:
        return R, [_hat(e) for e in np.eye(3)]
    I = np.eye(3)
    return R, [_hat((w[i] * w + np.cross(w, (I - R) @ I[:, i])) / t2) @ R for i in range(3)]


def pose_grad(cam: Cam, pixels, dist, grads, level=1):
    """Chain dL/dp_m into (dL/d omega, dL/d t) with frozen distances (camera.py:255-278)."""
    g = np.atleast_2d(np.asarray(grads, dtype=np.float64))
    d = np.asarray(dist, dtype=np.float64).reshape(-1)
    px = np.asarray(pixels, dtype=np.float64)
    cx, cy = cam.width / 2.0, cam.height / 2.0
    u = np.stack([((px[:, 0] + 0.5) * level - cx) / cam.fx,
                  ((px[:, 1] + 0.5) * level - cy) / cam.fx, np.ones(len(px))], axis=1)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    R, dR = rotation_partials(cam.omega)
    gs = g.sum(axis=0)
    gw = np.array([gs @ (-(dRi.T @ cam.t)) + np.einsum("m,mk,mk->", d, g, u @ dRi) for dRi in dR])
    return gw, -(R @ gs)


def pose_objective(dec: Decoder, code, cam: Cam, cfg: Cfg, w: Weights, depth=None, silhouette=None):
    """Loss and 6-vector gradient of one pose iterate (optimize.py:185-233)."""
    fn = lambda p: dec(p, code)  # noqa: E731
    T = trace(fn, cam, cfg)
    H = heads(T, fn, cfg)
    terms, ds, ss, gimg = {}, None, None, None
    if depth is not None:
        l, s = depth_loss(H, depth, np.isfinite(depth))
        terms["depth"] = l
        ds = w.depth * s
    if silhouette is not None:
        l, gimg = silhouette_loss(soft_silhouette(T, cfg), silhouette)
        terms["silhouette"] = l
        ss = w.silhouette * gimg[H.pixels[:, 1], H.pixels[:, 0]]
    b = heads_backward(H, dec, code, cfg, ds, ss)
    pix, dist, pg = H.pixels[H.sample_pixel], H.sample_d, b["sample_point_grads"]
    if gimg is not None:
        miss = np.nonzero(~np.isfinite(T.tk_a[:, 0]))[0]
        if miss.size:
            sd = w.silhouette * gimg[T.rays.pixels[miss, 1], T.rays.pixels[miss, 0]]
            dirs = T.rays.dirs[miss]
            dstar = -(dirs @ T.rays.origin)
            pstar = T.rays.origin + dstar[:, None] * dirs
            nrm = np.linalg.norm(pstar, axis=1, keepdims=True)
            gm = sd[:, None] * np.divide(pstar, nrm, out=np.zeros_like(pstar), where=nrm > 0)
            pix = np.concatenate([pix, T.rays.pixels[miss]])
            dist = np.concatenate([dist, dstar])
            pg = np.concatenate([pg, gm])
    gw, gt = pose_grad(cam, pix, dist, pg)
    total = w.depth * terms.get("depth", 0.0) + w.silhouette * terms.get("silhouette", 0.0)
    return total, terms, np.concatenate([gw, gt]), T.total_queries
