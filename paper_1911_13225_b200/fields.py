"""Latent-conditioned neural SDF on the device -- the drop-in `NeuralField`.

Same constructor, attributes and validation as the reference
(fields.py:185-219): a list of (W[in,out], b[out]) float64 pairs applied to
concat(code, p), ReLU hidden layers, a tanh (or linear) head.  The weights are
packed once into an immutable device decoder (dist_decoder_create) per
arithmetic mode; `evaluate` (the reference's field protocol used by the
tracer, tracer.py:165) runs on the GPU through dist_eval.  Extensions:
`precision` selects fp64 / fp32 / bf16x3 decoder arithmetic, and `skip`
selects the DeepSDF layout where layer `skip` consumes concat(h, code, p).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

PRECISIONS = ("fp64", "fp32", "bf16x3", "fp16x3")


def _pts(points) -> np.ndarray:
    p = np.asarray(points, dtype=np.float64)
    if p.ndim == 1:
        p = p[None, :]
    if p.ndim != 2 or p.shape[1] != 3:
        raise ValueError(f"points must be [n,3], got {p.shape}")
    return p


class NeuralField:
    """MLP SDF on concat(code, p) evaluated by libdist_b200 (fields.py:185-247)."""

    def __init__(self, weights, latent_dim: int = 0, hidden_activation: str = "relu",
                 final_activation: str = "tanh", precision: str = "fp64", skip: int = -1):
        self.weights = [(np.asarray(W, dtype=np.float64), np.asarray(b, dtype=np.float64))
                        for W, b in weights]
        self.latent_dim = int(latent_dim)
        if hidden_activation not in ("relu", "tanh"):
            raise ValueError(f"unknown hidden activation {hidden_activation!r}")
        if final_activation not in ("tanh", "linear", "sigmoid"):
            raise ValueError(f"unknown final activation {final_activation!r}")
        if hidden_activation != "relu":
            raise ValueError("the B200 decoder implements ReLU hidden layers only")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        self.hidden_activation = hidden_activation
        self.final_activation = final_activation
        self.precision = precision
        self.skip = int(skip)
        if self.skip < 0 and self.weights[0][0].shape[0] != self.latent_dim + 3:
            raise ValueError("first layer width must be latent_dim + 3")
        if self.weights[-1][0].shape[1] != 1:
            raise ValueError("final layer must map to one output")
        self._handles: dict[str, int] = {}

    # --- construction helpers -------------------------------------------------
    @classmethod
    def init(cls, latent_dim: int = 0, hidden=(64, 64, 64, 64), rng=None, **kw):
        """He-normal init with a x0.1 last layer (fields.py:209-219); same RNG draws."""
        rng = np.random.default_rng(rng)
        dims = [latent_dim + 3, *hidden, 1]
        weights = []
        for i, (p, q) in enumerate(zip(dims[:-1], dims[1:])):
            scale = np.sqrt(2.0 / p)
            if i == len(dims) - 2:
                scale *= 0.1
            weights.append((rng.standard_normal((p, q)) * scale, np.zeros(q)))
        return cls(weights, latent_dim=latent_dim, **kw)

    @classmethod
    def geometric(cls, latent_dim: int = 256, hidden=(512,) * 8, seed: int = 0, skip: int = -1,
                  **kw):
        """The standard synthetic DeepSDF decoder of SURVEY.md 8(d): seeded
        geometric init that yields a real surface (hidden W ~ N(0, 2/out),
        latent rows x0.1, head N(sqrt(pi/n), 1e-4), bias -0.5)."""
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
                W[:D] *= 0.1
            elif i == skip:
                W[ins[i] - (D + 3):ins[i] - 3] *= 0.1
            ws.append((W, np.zeros(o)))
        n = hidden[-1]
        ws.append((rng.normal(np.sqrt(np.pi) / np.sqrt(n), 1e-4, (n, 1)), np.full(1, -0.5)))
        return cls(ws, latent_dim=latent_dim, skip=skip, **kw)

    def with_precision(self, precision: str) -> "NeuralField":
        f = NeuralField.__new__(NeuralField)
        f.__dict__.update(self.__dict__)
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        f.precision = precision
        f._handles = self._handles   # packs are per precision; share the cache
        f._owner = False
        return f

    # --- device decoder ---------------------------------------------------------
    def handle(self) -> int:
        """The immutable device decoder for self.precision (created on first use)."""
        h = self._handles.get(self.precision)
        if h:
            return h
        _lib.require_device()
        L = len(self.weights)
        dims = [self.weights[0][0].shape[0] if self.skip < 0 else self.latent_dim + 3]
        for i, (W, _) in enumerate(self.weights):
            dims.append(W.shape[1])
        if self.skip > 0:
            dims[0] = self.latent_dim + 3
        self._keep = [(np.ascontiguousarray(W), np.ascontiguousarray(b)) for W, b in self.weights]
        Wp = (C.c_void_p * L)(*[W.ctypes.data for W, _ in self._keep])
        bp = (C.c_void_p * L)(*[b.ctypes.data for _, b in self._keep])
        dims_c = (C.c_int32 * (L + 1))(*dims)
        out = C.c_void_p()
        _lib.check(_lib.lib().dist_decoder_create(
            Wp, bp, L, dims_c, self.latent_dim, self.skip,
            {"tanh": 0, "linear": 1, "sigmoid": 2}[self.final_activation], _lib.PREC[self.precision],
            C.byref(out)))
        self._handles[self.precision] = out.value
        return out.value

    def head_gain(self) -> tuple:
        """The calibrated accumulator-bias gain of the tensor-core head
        (include/dist.h dist_decoder_head_gain): (march/eval, fp16 probes)."""
        g = (C.c_double * 2)()
        _lib.check(_lib.lib().dist_decoder_head_gain(self.handle(), g))
        return float(g[0]), float(g[1])

    def __del__(self):
        try:
            lib = _lib._lib
            if lib is not None and getattr(self, "_owner", True):
                for h in list(self._handles.values()):
                    lib.dist_decoder_destroy(h)
                self._handles.clear()
        except Exception:
            pass

    def _codes_dev(self, code, torch):
        if self.latent_dim == 0:
            return None, 1
        if code is None:
            raise ValueError("field expects a latent code")
        if isinstance(code, torch.Tensor):
            z = code.to(device="cuda", dtype=torch.float64).reshape(-1, self.latent_dim)
            return z.contiguous(), z.shape[0]
        code = np.asarray(code, dtype=np.float64)
        if code.shape != (self.latent_dim,):
            raise ValueError(f"code shape {code.shape} != ({self.latent_dim},)")
        return torch.from_numpy(code.copy()).cuda(), 1

    # --- field protocol -----------------------------------------------------------
    def evaluate(self, points, code=None):
        """f(points, code) on the GPU; numpy in -> numpy out (fields.py:233-247)."""
        import torch
        p = points if isinstance(points, torch.Tensor) else _pts(points)
        out = self.evaluate_device(p, code)
        return out if isinstance(points, torch.Tensor) else out.cpu().numpy()

    def evaluate_device(self, points, code=None, shape_ids=None):
        import torch
        h = self.handle()
        z, S = self._codes_dev(code, torch)
        P = points if isinstance(points, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(points))
        P = P.to(device="cuda", dtype=torch.float64).reshape(-1, 3).contiguous()
        n = P.shape[0]
        f = torch.empty(n, dtype=torch.float64, device="cuda")
        if n == 0:
            return f
        sid = None if shape_ids is None else shape_ids.to(device="cuda", dtype=torch.int32).contiguous()
        lib = _lib.lib()
        nbytes = lib.dist_eval_workspace_size(h, n, S)
        ws = _lib.workspace(nbytes)
        _lib.check(lib.dist_eval(h, _lib.ptr(z), S, P.data_ptr(), _lib.ptr(sid), n, f.data_ptr(),
                                 ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
        return f

    def vjp_device(self, points, code, seed, shape_ids=None, want_points=True):
        """Taped evaluation + reverse sweep (fields.py:260-291): returns
        (f[n], d(seed.f)/dcode [S,D], d(seed.f)/dp [n,3] or None)."""
        import torch
        h = self.handle()
        z, S = self._codes_dev(code, torch)
        P = points.to(device="cuda", dtype=torch.float64).reshape(-1, 3).contiguous()
        n = P.shape[0]
        sd = seed.to(device="cuda", dtype=torch.float64).reshape(-1).contiguous()
        f = torch.empty(n, dtype=torch.float64, device="cuda")
        gc = torch.zeros((S, max(self.latent_dim, 1)), dtype=torch.float64, device="cuda")
        gp = torch.zeros((n, 3), dtype=torch.float64, device="cuda") if want_points else None
        if n == 0:
            return f, gc[:, :self.latent_dim], gp
        sid = None if shape_ids is None else shape_ids.to(device="cuda", dtype=torch.int32).contiguous()
        lib = _lib.lib()
        ws = _lib.workspace(lib.dist_eval_workspace_size(h, n, S))
        _lib.check(lib.dist_eval_vjp(h, _lib.ptr(z), S, P.data_ptr(), _lib.ptr(sid), n,
                                     sd.data_ptr(), f.data_ptr(),
                                     gc.data_ptr() if self.latent_dim else None, _lib.ptr(gp),
                                     ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
        return f, gc[:, :self.latent_dim], gp


class AttributeField:
    """MLP from concat(shape code, attribute code, p) to an m-vector in [0, 1]
    (fields.py:294-338).  Held on the device as m
    single-output sigmoid-head decoders over the same hidden stack;
    `dist_eval_channels` runs that stack once per point and then the m heads
    (SIMT precisions, m <= 8; otherwise each channel is evaluated in turn)."""

    def __init__(self, weights, shape_dim: int = 0, attr_dim: int = 0,
                 hidden_activation: str = "relu", precision: str = "fp64"):
        self.weights = [(np.asarray(W, dtype=np.float64), np.asarray(b, dtype=np.float64))
                        for W, b in weights]
        self.shape_dim, self.attr_dim = int(shape_dim), int(attr_dim)
        self.hidden_activation = hidden_activation
        if self.weights[0][0].shape[0] != self.shape_dim + self.attr_dim + 3:
            raise ValueError("first layer width must be shape_dim + attr_dim + 3")
        self.out_dim = self.weights[-1][0].shape[1]
        W, b = self.weights[-1]
        self._channels = [NeuralField(self.weights[:-1] + [(W[:, c:c + 1], b[c:c + 1])],
                                      latent_dim=self.shape_dim + self.attr_dim,
                                      hidden_activation=hidden_activation,
                                      final_activation="sigmoid", precision=precision)
                          for c in range(self.out_dim)]

    @classmethod
    def init(cls, shape_dim: int = 0, attr_dim: int = 0, hidden=(32, 32, 32), out_dim: int = 3,
             rng=None, **kw):
        """He-normal init (fields.py:312-319), same RNG draws as the reference."""
        rng = np.random.default_rng(rng)
        dims = [shape_dim + attr_dim + 3, *hidden, out_dim]
        weights = [(rng.standard_normal((p, q)) * np.sqrt(2.0 / p), np.zeros(q))
                   for p, q in zip(dims[:-1], dims[1:])]
        return cls(weights, shape_dim=shape_dim, attr_dim=attr_dim, **kw)

    def evaluate(self, points, code=None):
        d = self.shape_dim + self.attr_dim
        if d:
            code = np.asarray(code, dtype=np.float64)
            if code.shape != (d,):
                raise ValueError(f"attribute code shape {code.shape} != ({d},)")
        p = _pts(points)
        if self.out_dim <= 8 and self._channels[0].precision in ("fp64", "fp32"):
            return self.evaluate_device(p, code if d else None).cpu().numpy()
        return np.stack([ch.evaluate(p, code if d else None) for ch in self._channels], axis=1)

    def evaluate_device(self, points, code=None):
        """[n, m] on the device: the hidden stack once, then the m heads."""
        import torch
        ch0 = self._channels[0]
        z, S = ch0._codes_dev(code, torch)
        P = points if isinstance(points, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(points))
        P = P.to(device="cuda", dtype=torch.float64).reshape(-1, 3).contiguous()
        n = P.shape[0]
        out = torch.empty((n, self.out_dim), dtype=torch.float64, device="cuda")
        if n == 0:
            return out
        lib = _lib.lib()
        handles = (C.c_void_p * self.out_dim)(*[ch.handle() for ch in self._channels])
        ws = _lib.workspace(lib.dist_eval_workspace_size(ch0.handle(), n, S))
        _lib.check(lib.dist_eval_channels(C.cast(handles, C.c_void_p), self.out_dim, _lib.ptr(z), S,
                                          P.data_ptr(), None, n, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                          _lib.stream_ptr()))
        return out


def eval_field(field, points, code=None):
    """fields.py:350-352."""
    return field.evaluate(points, code)
