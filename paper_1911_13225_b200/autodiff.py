"""The taped-evaluation seam of the reference, backed by the device.

The reference records a field evaluation on a general reverse-mode tape
(autodiff.py:49-255) and differentiates it with `backward(tape, output,
seed)`; `eval_field_taped(field, points, code)` is the entry point its heads
and pose chain use (fields.py:344-373).  On the hot path the only taped
program is the decoder itself, so the tape here is a record of one
evaluation -- field, frozen points, code -- and `backward` runs the decoder's
reverse sweep on the GPU (dist_eval_vjp: the fused tcgen05 head kernel or the
SIMT fp64/fp32 sweep).  Leaves and error behaviour follow the reference:
gradients for "points" [n,3] and, for latent-conditioned fields, "code" [D];
a seed of the wrong shape raises ValueError, a non-finite gradient
FloatingPointError (autodiff.py:229-254).  Network-weight leaves
(want_weights=True) are outside the hot path and raise ValueError.

Analytic / duck-typed fields (anything with evaluate and spatial_gradient)
get the reference's single custom node: d/dp = seed * spatial_gradient
(fields.py:362-373).
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np


class Tape:
    """One recorded evaluation (the leaves the reference's tape would hold)."""

    def __init__(self, field, points: np.ndarray, code):
        self.field = field
        self._leaf_values = {"points": points}
        if getattr(field, "latent_dim", 0) > 0 and hasattr(field, "handle"):
            self._leaf_values["code"] = np.asarray(code, dtype=np.float64)
        self.code = code


class Tensor(NamedTuple):
    """The output node of a Tape: its value [n] and the tape it belongs to."""
    value: np.ndarray
    tape: Tape


class TapedEval(NamedTuple):
    values: np.ndarray
    tape: Tape
    output: Tensor


def eval_field_taped(field, points, code=None, want_weights: bool = False) -> TapedEval:
    """fields.py:355-373: evaluate and record for backward()."""
    if want_weights:
        raise ValueError("weight gradients are outside the B200 hot path")
    from .fields import _pts
    p = _pts(points)
    vals = np.asarray(field.evaluate(p, code), dtype=np.float64).reshape(-1)
    tape = Tape(field, p, code)
    return TapedEval(vals, tape, Tensor(vals, tape))


def backward(tape: Tape, output: Tensor, seed) -> dict:
    """Gradient of seed . output w.r.t. the tape's leaves (autodiff.py:220-255)."""
    if output.tape is not tape:
        raise ValueError("output node is not on this tape")
    seed = np.asarray(seed, dtype=np.float64)
    if seed.shape != output.value.shape:
        raise ValueError(f"seed shape {seed.shape} != output {output.value.shape}")
    field, p = tape.field, tape._leaf_values["points"]
    out = {}
    if hasattr(field, "vjp_device"):
        import torch
        P = torch.from_numpy(np.ascontiguousarray(p)).cuda()
        S = torch.from_numpy(np.ascontiguousarray(seed)).cuda()
        _, gc, gp = field.vjp_device(P, tape.code, S)
        out["points"] = gp.cpu().numpy()
        if "code" in tape._leaf_values:
            out["code"] = gc.cpu().numpy().reshape(-1)
    elif hasattr(field, "spatial_gradient"):
        out["points"] = seed[:, None] * np.asarray(field.spatial_gradient(p), dtype=np.float64)
    else:
        raise ValueError("field provides neither a device decoder nor spatial_gradient")
    for name, g in out.items():
        if not np.all(np.isfinite(g)):
            raise FloatingPointError(f"non-finite gradient for leaf {name!r}")
    return out
