"""Sphere tracing on the B200 -- drop-in for the reference tracer.py.

`trace(field, code, intr, pose, cfg)` has the reference signature and returns
a `TraceResult` whose `state` is a `RayState` of numpy arrays
(tracer.py:53-82), so the reference's own map, loss and test code can read it.
Underneath, `trace_views` runs the whole coarse-to-fine march of V views on
the device in one C-ABI call (dist_trace) with no host synchronisation per
step, and keeps the state resident in HBM (`DeviceTrace`) for the heads,
losses and optimiser that follow.
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass, field as dfield

import numpy as np

from . import _lib
from .camera import Intrinsics, Pose, RayBundle, camera_struct, generate_rays

MARCHING, CONVERGED, ESCAPED, EXHAUSTED = 0, 1, 2, 3


@dataclass
class TraceConfig:
    """tracer.py:27-50 (same defaults and validation)."""
    alpha: float = 1.5
    epsilon: float = 5e-5
    max_steps: int = 100
    k_samples: int = 1
    coarse_start_scale: int = 4
    split_interval: int = 3
    normal_delta: float = 1e-3
    use_dynamic_mask: bool = True

    def __post_init__(self):
        if not (0.0 < self.alpha < 2.0):
            raise ValueError("alpha must be in (0, 2)")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.max_steps < 1:
            raise ValueError("max_steps must be at least 1")
        if self.k_samples < 1:
            raise ValueError("k_samples must be at least 1")
        if self.coarse_start_scale not in (1, 2, 4):
            raise ValueError("coarse_start_scale must be 1, 2, or 4")
        if self.split_interval < 1:
            raise ValueError("split_interval must be at least 1")


@dataclass
class RayState:
    """Host view of one view's final-level state (tracer.py:53-73)."""
    bundle: RayBundle
    d: np.ndarray
    b: np.ndarray
    status: np.ndarray
    steps: np.ndarray
    topk_d: np.ndarray
    topk_f: np.ndarray
    topk_absf: np.ndarray

    @property
    def n(self) -> int:
        return self.d.shape[0]

    def live(self) -> np.ndarray:
        return self.status == MARCHING


class DeviceTrace:
    """Device-resident result of tracing V views (all tensors on cuda)."""

    def __init__(self, field, codes, cams, intrs, poses, cfg: TraceConfig, W: int, H: int,
                 relu_masks: bool = False):
        import torch
        self.field, self.codes, self.cfg = field, codes, cfg
        self.external = False   # traced through the plugin seam (trace_external)
        self.cams, self.intrs, self.poses = cams, intrs, poses
        self.V, self.W, self.H = len(intrs), W, H
        n = self.V * W * H
        K = cfg.k_samples
        dev = "cuda"
        self.d = torch.empty(n, dtype=torch.float64, device=dev)
        self.b = torch.empty(n, dtype=torch.float64, device=dev)
        self.status = torch.empty(n, dtype=torch.uint8, device=dev)
        self.steps = torch.empty(n, dtype=torch.int32, device=dev)
        self.topk_d = torch.empty((n, K), dtype=torch.float64, device=dev)
        self.topk_f = torch.empty((n, K), dtype=torch.float64, device=dev)
        self.topk_absf = torch.empty((n, K), dtype=torch.float64, device=dev)
        # per view: its own query count per own step (include/dist.h dist_trace)
        self.live_counts_dev = torch.zeros((self.V, cfg.max_steps), dtype=torch.int64, device=dev)
        self.stats_dev = torch.zeros(4, dtype=torch.int64, device=dev)
        # ReLU masks of the recorded samples (include/dist.h dist_ray_state):
        # lets dist_objective skip the taped forward for them
        self.relu_masks = self.topk_slot = None
        if relu_masks:
            nm = len(field.weights) - 1
            self.relu_masks = torch.empty(n * (K + 1) * nm * 16, dtype=torch.int32, device=dev)
            self.topk_slot = torch.empty((n, K + 1), dtype=torch.uint8, device=dev)

    def state_struct(self) -> _lib.dist_ray_state:
        return _lib.dist_ray_state(self.d.data_ptr(), self.b.data_ptr(), self.status.data_ptr(),
                                   self.steps.data_ptr(), self.topk_d.data_ptr(),
                                   self.topk_f.data_ptr(), self.topk_absf.data_ptr(),
                                   _lib.ptr(self.relu_masks), _lib.ptr(self.topk_slot))

    def stats(self) -> dict:
        """Audit counters (TraceResult fields).  live_counts: the views' own
        per-step query counts summed by step index; live_counts_per_view: each
        view's list (tracer.py:247-249)."""
        s = self.stats_dev.cpu().numpy()
        lc = self.live_counts_dev.cpu().numpy()
        per = [[int(x) for x in row[: int(np.count_nonzero(row))]] for row in lc]
        return {"total_queries": int(s[0]), "nan_count": int(s[1]), "steps": int(s[2]),
                "warnings": int(s[3]), "live_counts": [int(x) for x in lc.sum(axis=0)[: int(s[2])]],
                "live_counts_per_view": per}


def _code_tensor(field, codes):
    import torch
    if field.latent_dim == 0:
        return None, 1
    if codes is None:
        raise ValueError("field expects a latent code")
    if isinstance(codes, torch.Tensor):
        z = codes.to(device="cuda", dtype=torch.float64)
    else:
        z = torch.from_numpy(np.asarray(codes, dtype=np.float64).copy()).cuda()
    z = z.reshape(-1, field.latent_dim).contiguous()
    return z, z.shape[0]


def relu_mask_bytes(field, n_rays: int, k_samples: int) -> int:
    """Device bytes of the optional ReLU-mask record of n_rays rays."""
    return n_rays * (k_samples + 1) * (len(field.weights) - 1) * 64 + n_rays * (k_samples + 1)


def trace_views(field, codes, views, cfg: TraceConfig | None = None,
                shape_of_view=None, reuse: DeviceTrace | None = None,
                relu_masks: bool = False) -> DeviceTrace:
    """Trace V views (list of (Intrinsics, Pose)) of one resolution in one call.

    codes: [D] or [S, D]; shape_of_view[v] picks the code row of view v.
    reuse: a DeviceTrace of the same views/config whose buffers (and uploaded
    cameras) are overwritten in place -- the optimisation loop's fast path.
    relu_masks: also record the ReLU masks of every recorded sample (tensor-core
    precisions; the objective then runs only the backward sweep for them).
    """
    import torch
    cfg = cfg or TraceConfig()
    _lib.require_device()
    intrs = [v[0] for v in views]
    poses = [v[1] for v in views]
    W, H = intrs[0].width, intrs[0].height
    if any(i.width != W or i.height != H for i in intrs):
        raise ValueError("all views of one trace call must share a resolution")
    if W % cfg.coarse_start_scale or H % cfg.coarse_start_scale:
        raise ValueError(f"resolution {W}x{H} not divisible by coarse_start_scale "
                         f"{cfg.coarse_start_scale}")
    h = field.handle()
    z, S = _code_tensor(field, codes)
    if reuse is not None:
        dt = reuse
        dt.codes = z
    else:
        sv = [0] * len(views) if shape_of_view is None else [int(s) for s in shape_of_view]
        cams = _lib.cameras_to_device([camera_struct(i, p, s) for i, p, s in zip(intrs, poses, sv)])
        dt = DeviceTrace(field, z, cams, intrs, poses, cfg, W, H, relu_masks=relu_masks)
    cams = dt.cams
    lib = _lib.lib()
    c = _lib.config_struct(cfg)
    nbytes = lib.dist_trace_workspace_size(h, C.byref(c), len(views), W, H, S)
    ws = _lib.workspace(nbytes)
    st = dt.state_struct()
    _lib.check(lib.dist_trace(h, _lib.ptr(z), S, cams.data_ptr(), len(views), W, H, C.byref(c),
                              C.byref(st), dt.live_counts_dev.data_ptr(), dt.stats_dev.data_ptr(),
                              ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
    dt._ws_keep = ws
    return dt


@dataclass
class TraceResult:
    """tracer.py:76-82, plus `device` (the resident DeviceTrace)."""
    state: RayState
    config: TraceConfig
    intrinsics: Intrinsics
    pose: Pose
    live_counts: list = dfield(default_factory=list)
    total_queries: int = 0
    nan_count: int = 0
    device: DeviceTrace | None = None
    view: int = 0


def host_result(dt: DeviceTrace, view: int = 0) -> TraceResult:
    """Copy one view's state to numpy in the reference's RayState layout."""
    n = dt.W * dt.H
    sl = slice(view * n, (view + 1) * n)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        bundle = generate_rays(dt.intrs[view], dt.poses[view], 1)
    st = RayState(bundle=bundle, d=dt.d[sl].cpu().numpy(), b=dt.b[sl].cpu().numpy(),
                  status=dt.status[sl].cpu().numpy(),
                  steps=dt.steps[sl].cpu().numpy().astype(np.int64),
                  topk_d=dt.topk_d[sl].cpu().numpy(), topk_f=dt.topk_f[sl].cpu().numpy(),
                  topk_absf=dt.topk_absf[sl].cpu().numpy())
    s = dt.stats()
    lc = s["live_counts_per_view"][view]
    # per-view audit (tracer.py:80-82); NaN queries are counted for the whole batch
    return TraceResult(state=st, config=dt.cfg, intrinsics=dt.intrs[view], pose=dt.poses[view],
                       live_counts=lc, total_queries=int(sum(lc)),
                       nan_count=s["nan_count"] if dt.V == 1 else int(np.isnan(st.b).sum()),
                       device=dt, view=view)


def trace_external(field, code, views, cfg: TraceConfig | None = None) -> DeviceTrace:
    """The reference's plugin seam (tracer.py:165): trace V views of ANY field
    with `evaluate(points[n,3], code) -> f[n]` -- analytic SDFs, the
    reference's own fields, test fakes.  The march (init, dynamic mask, top-K
    record, update, splits, audit counters) runs on the device
    (dist_trace_external); the field is called once per step on that step's
    query points, as the reference's march_step calls it."""
    cfg = cfg or TraceConfig()
    _lib.require_device()
    intrs = [v[0] for v in views]
    poses = [v[1] for v in views]
    W, H = intrs[0].width, intrs[0].height
    if any(i.width != W or i.height != H for i in intrs):
        raise ValueError("all views of one trace call must share a resolution")
    if W % cfg.coarse_start_scale or H % cfg.coarse_start_scale:
        raise ValueError(f"resolution {W}x{H} not divisible by coarse_start_scale "
                         f"{cfg.coarse_start_scale}")
    cams = _lib.cameras_to_device([camera_struct(i, p, 0) for i, p in zip(intrs, poses)])
    dt = DeviceTrace(field, code, cams, intrs, poses, cfg, W, H)
    n = len(views) * W * H
    pts = np.empty(n * 3, dtype=np.float64)
    vals = np.empty(n, dtype=np.float64)
    err = []

    def evaluate(p_ptr, m, f_ptr, _user):
        try:
            p = np.ctypeslib.as_array(p_ptr, shape=(m, 3)).copy()
            f = np.asarray(field.evaluate(p, code), dtype=np.float64).reshape(-1)
            if f.shape[0] != m:
                raise ValueError(f"field returned {f.shape[0]} values for {m} points")
            np.ctypeslib.as_array(f_ptr, shape=(m,))[:] = f
            return 0
        except BaseException as ex:   # re-raised below, after the C call unwinds
            err.append(ex)
            return 1

    fn = _lib.FIELD_FN(evaluate)
    lib = _lib.lib()
    c = _lib.config_struct(cfg)
    ws = _lib.workspace(lib.dist_trace_external_workspace_size(C.byref(c), len(views), W, H))
    st = dt.state_struct()
    rc = lib.dist_trace_external(fn, None, cams.data_ptr(), len(views), W, H, C.byref(c), C.byref(st),
                                 dt.live_counts_dev.data_ptr(), dt.stats_dev.data_ptr(),
                                 pts.ctypes.data, vals.ctypes.data, ws.data_ptr(), ws.numel(),
                                 _lib.stream_ptr())
    if err:
        raise err[0]
    _lib.check(rc)
    dt.external = True
    return dt


def trace(field, code, intr: Intrinsics, pose: Pose, cfg: TraceConfig | None = None) -> TraceResult:
    """Full render-tracing pass (tracer.py:221-252) on the GPU.  Any object
    with `evaluate(points, code)` is accepted (the reference's duck-typed
    field protocol); NeuralField runs its decoder on the device as well."""
    cfg = cfg or TraceConfig()
    if intr.width % cfg.coarse_start_scale or intr.height % cfg.coarse_start_scale:
        raise ValueError(f"resolution {intr.width}x{intr.height} not divisible by "
                         f"coarse_start_scale {cfg.coarse_start_scale}")
    if not hasattr(field, "handle"):
        if not hasattr(field, "evaluate"):
            raise TypeError("field must provide evaluate(points, code)")
        dt = trace_external(field, code, [(intr, pose)], cfg)
    else:
        dt = trace_views(field, code, [(intr, pose)], cfg)
    res = host_result(dt, 0)
    if dt.stats()["warnings"] & 1:
        warnings.warn("camera center inside the unit sphere; rays start at d=0", RuntimeWarning)
    return res
