"""ctypes binding of libdist_b200.so (include/dist.h).

This is the reference-side binding INTEGRATION.md describes: the reference is
Python, so the C ABI is bound with ctypes and device buffers are PyTorch
tensors whose raw pointers cross the boundary.  There is no CPU fallback:
importing a compute entry point on a machine without the built library or
without an sm_100 GPU raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DIST_LIB_PATH") or os.path.join(_HERE, "libdist_b200.so")  # override: A/B timing only

DIST_OK, DIST_ERR_CONFIG, DIST_ERR_NUMERIC, DIST_ERR_CUDA = 0, 2, 3, 4
PREC = {"fp64": 0, "fp32": 1, "bf16x3": 2, "fp16x3": 3}


class dist_camera(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("origin", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("shape", C.c_int32),
                ("reserved", C.c_int32)]


class dist_trace_config(C.Structure):
    _fields_ = [("alpha", C.c_double), ("epsilon", C.c_double), ("normal_delta", C.c_double),
                ("max_steps", C.c_int32), ("k_samples", C.c_int32),
                ("coarse_start_scale", C.c_int32), ("split_interval", C.c_int32),
                ("use_dynamic_mask", C.c_int32), ("reserved", C.c_int32)]


class dist_ray_state(C.Structure):
    _fields_ = [("d", C.c_void_p), ("b", C.c_void_p), ("status", C.c_void_p),
                ("steps", C.c_void_p), ("topk_d", C.c_void_p), ("topk_f", C.c_void_p),
                ("topk_absf", C.c_void_p), ("relu_masks", C.c_void_p), ("topk_slot", C.c_void_p)]


class dist_objective_io(C.Structure):
    _fields_ = [("obs_depth", C.c_void_p), ("obs_depth_mask", C.c_void_p),
                ("obs_sil", C.c_void_p), ("w_depth", C.c_double), ("w_sil", C.c_double),
                ("w_latent", C.c_double), ("grad", C.c_void_p), ("view_terms", C.c_void_p),
                ("shape_terms", C.c_void_p), ("grad_mode", C.c_int32), ("reserved", C.c_int32),
                ("counts_out", C.c_void_p), ("obs_normal", C.c_void_p),
                ("obs_normal_mask", C.c_void_p), ("w_normal", C.c_double), ("phase", C.c_int32),
                ("reserved2", C.c_int32), ("view_norm", C.c_void_p), ("colsum_fixed", C.c_void_p)]


VIEW_TERMS = 6   # dist_objective_io.view_terms columns (include/dist.h)


class dist_adam_config(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double)]


FIELD_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double), C.c_void_p)

_SIGS = {
    "dist_last_error": (C.c_char_p, []),
    "dist_device_info": (C.c_int, [C.POINTER(C.c_int)] * 3),
    "dist_launch_count": (C.c_int64, []),
    "dist_debug_mlp_timeline": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    "dist_debug_fluid_timeline": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    "dist_debug_heads_timeline": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    "dist_decoder_create": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int,
                                      C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "dist_decoder_destroy": (C.c_int, [C.c_void_p]),
    "dist_decoder_precision": (C.c_int, [C.c_void_p]),
    "dist_eval_workspace_size": (C.c_size_t, [C.c_void_p, C.c_int64, C.c_int]),
    "dist_eval": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64,
                            C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_eval_vjp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_trace_workspace_size": (C.c_size_t, [C.c_void_p, C.POINTER(dist_trace_config), C.c_int,
                                               C.c_int, C.c_int, C.c_int]),
    "dist_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                             C.c_int, C.POINTER(dist_trace_config), C.POINTER(dist_ray_state),
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_trace_external_workspace_size": (C.c_size_t, [C.POINTER(dist_trace_config), C.c_int,
                                                        C.c_int, C.c_int]),
    "dist_trace_external": (C.c_int, [FIELD_FN, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(dist_trace_config), C.POINTER(dist_ray_state),
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_size_t, C.c_void_p]),
    "dist_maps": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(dist_trace_config),
                            C.POINTER(dist_ray_state), C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_void_p]),
    "dist_normals_workspace_size": (C.c_size_t, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    "dist_normals": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                               C.c_int, C.POINTER(dist_trace_config), C.POINTER(dist_ray_state),
                               C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_objective_workspace_size": (C.c_size_t, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                   C.c_int, C.c_int, C.c_int]),
    "dist_code_grad_fixed": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_double,
                                       C.c_void_p, C.c_void_p]),
    "dist_decoder_colsum_width": (C.c_int, [C.c_void_p]),
    "dist_decoder_head_gain": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "dist_objective": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                 C.c_int, C.POINTER(dist_trace_config), C.POINTER(dist_ray_state),
                                 C.POINTER(dist_objective_io), C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_eval_channels": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_photometric_workspace_size": (C.c_size_t, [C.c_int, C.c_int]),
    "dist_photometric": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dist_photo_heads": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(dist_ray_state), C.c_void_p, C.c_void_p, C.c_void_p]),
    "dist_photo_depth": (C.c_int, [C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    "dist_photo_seeds": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                   C.c_void_p]),
    "dist_pose_samples": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(dist_ray_state),
                                    C.c_void_p, C.c_void_p]),
    "dist_pose_seeds": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(dist_ray_state),
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dist_pose_grad": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(dist_ray_state),
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    "dist_adam_step": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_int, C.c_void_p, C.POINTER(dist_adam_config),
                                 C.c_void_p, C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def exported_symbols() -> list[str]:
    """Names the header declares (checked against the .so by the CPU tests)."""
    return sorted(_SIGS)


def load_library(path: str = LIB_PATH):
    """dlopen the library and attach signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class DistError(RuntimeError):
    pass


def check(rc: int):
    if rc == DIST_OK:
        return
    msg = (lib().dist_last_error() or b"").decode()
    if rc == DIST_ERR_CONFIG:
        raise ValueError(msg)
    if rc == DIST_ERR_NUMERIC:
        raise FloatingPointError(msg)
    raise DistError(msg or f"libdist_b200 error {rc}")


def lib():
    return load_library()


_device_checked = False


def require_device():
    """The product path runs only on a CUDA sm_100 device."""
    global _device_checked
    import torch
    if _device_checked:
        return
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1911_13225_b200 needs a CUDA (B200, sm_100a) device; "
                           "there is no CPU fallback")
    major, _ = torch.cuda.get_device_capability()
    if major != 10:
        raise RuntimeError("libdist_b200 is built for sm_100a (B200) only")
    load_library()
    _device_checked = True


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


_ws_cache: dict = {}


def workspace(nbytes: int):
    """A cached device scratch buffer per (device, stream), grown on demand.

    Calls on one stream are ordered, so they may share it; a different stream
    gets its own buffer (the C ABI itself takes per-call workspaces)."""
    import torch
    nbytes = max(int(nbytes), 256)
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    with _lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            _ws_cache[key] = buf
    return buf


def cameras_to_device(cams: list[dist_camera]):
    import torch
    arr = (dist_camera * len(cams))(*cams)
    raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
    return torch.from_numpy(raw).cuda(non_blocking=False)


def config_struct(cfg) -> dist_trace_config:
    return dist_trace_config(cfg.alpha, cfg.epsilon, cfg.normal_delta, cfg.max_steps,
                             cfg.k_samples, cfg.coarse_start_scale, cfg.split_interval,
                             1 if cfg.use_dynamic_mask else 0, 0)
