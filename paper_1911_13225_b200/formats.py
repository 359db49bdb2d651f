"""On-disk formats shared with the reference.

Files written by the reference load here and vice versa, so weights, cameras
and maps move between the two implementations bit-exactly:

* ``sdftrace-field/1`` JSON for neural fields (fields.py:376-459): floats are
  written with repr, so a load/save/load cycle is bit-exact;
* ``sdftrace-camera/1`` JSON (camera.py:284-312): focal/sensor in mm,
  resolution, principal point and the 3x4 world-to-camera extrinsic;
* ``sdftrace-report/1`` JSON for optimisation reports (cli.py:29, 55-70):
  the command name plus the ``OptimizeReport`` fields the reference writes;
* grayscale PFM for depth (float32, bottom-up rows, little-endian scale -1,
  +inf background stored as 0) and 8-bit binary PGM for masks
  (imageio.py:17-78).

Host-side I/O only: nothing here is on the compute path.
"""

from __future__ import annotations

import json

import numpy as np

from .camera import Intrinsics, Pose, log_rotation
from .fields import NeuralField

FIELD_FORMAT = "sdftrace-field/1"
CAMERA_FORMAT = "sdftrace-camera/1"
REPORT_FORMAT = "sdftrace-report/1"
_REPORT_KEYS = ("losses", "grad_norms", "best_iter", "best_loss", "total_queries", "elapsed",
                "skipped_steps", "non_identifiable")


def save_field(field: NeuralField, path, codes=None) -> None:
    doc = {"format": FIELD_FORMAT, "kind": "neural", "latent_dim": field.latent_dim,
           "hidden_activation": field.hidden_activation,
           "final_activation": field.final_activation,
           "weights": [[W.tolist(), b.tolist()] for W, b in field.weights]}
    if codes is not None:
        doc["codes"] = np.asarray(codes, dtype=np.float64).tolist()
    with open(path, "w") as fh:
        json.dump(doc, fh)


def load_field(path, precision: str = "fp64"):
    """Returns (NeuralField, codes or None); only neural fields are on the path."""
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != FIELD_FORMAT:
        raise ValueError(f"not a field file: format={doc.get('format')!r}")
    if doc.get("kind") != "neural":
        raise ValueError(f"field kind {doc.get('kind')!r} is not a neural decoder")
    f = NeuralField(doc["weights"], latent_dim=doc["latent_dim"],
                    hidden_activation=doc["hidden_activation"],
                    final_activation=doc["final_activation"], precision=precision)
    codes = doc.get("codes")
    return f, (None if codes is None else np.asarray(codes, dtype=np.float64))


def save_camera(intr: Intrinsics, pose: Pose, path) -> None:
    R = pose.rotation()
    cx, cy = intr.center
    doc = {"format": CAMERA_FORMAT, "focal_mm": intr.focal_mm, "sensor_mm": intr.sensor_mm,
           "resolution": [intr.width, intr.height], "principal": [cx, cy],
           "extrinsic": np.concatenate([R, pose.t[:, None]], axis=1).tolist()}
    with open(path, "w") as fh:
        json.dump(doc, fh)


def load_camera(path):
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != CAMERA_FORMAT:
        raise ValueError(f"not a camera file: format={doc.get('format')!r}")
    w, h = doc["resolution"]
    cx, cy = doc["principal"]
    ext = np.asarray(doc["extrinsic"], dtype=np.float64)
    if ext.shape != (3, 4):
        raise ValueError("extrinsic must be 3x4")
    return Intrinsics(doc["focal_mm"], doc["sensor_mm"], w, h, cx=cx, cy=cy), \
        Pose(log_rotation(ext[:, :3]), ext[:, 3])


def save_report(report, path, command: str) -> None:
    """cli.py:55-70: {"format", "command", losses, grad_norms, best_iter, best_loss,
    total_queries, elapsed, skipped_steps, non_identifiable}, indent 2, trailing newline."""
    payload = {}
    for k in _REPORT_KEYS:
        v = getattr(report, k)
        if isinstance(v, (list, tuple)):
            v = [float(x) for x in v]
        elif isinstance(v, (bool, np.bool_)):
            v = bool(v)
        elif isinstance(v, (int, np.integer)):
            v = int(v)
        elif isinstance(v, (float, np.floating)):
            v = float(v)
        payload[k] = v
    doc = {"format": REPORT_FORMAT, "command": command, **payload}
    with open(path, "w") as fh:
        fh.write(json.dumps(doc, indent=2) + "\n")


def load_report(path):
    """Returns (command, OptimizeReport) from an sdftrace-report/1 file."""
    from .optimize import OptimizeReport
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != REPORT_FORMAT:
        raise ValueError(f"not a report file: format={doc.get('format')!r}")
    rep = OptimizeReport()
    for k in _REPORT_KEYS:
        if k in doc:
            setattr(rep, k, doc[k])
    return doc.get("command"), rep


def write_pfm(path, img) -> None:
    a = np.asarray(img, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("PFM writer takes a single-channel image")
    a = a.astype(np.float32)
    a[np.isposinf(a)] = 0.0
    h, w = a.shape
    with open(path, "wb") as fh:
        fh.write(b"Pf\n" + f"{w} {h}\n".encode() + b"-1.0\n")
        fh.write(np.ascontiguousarray(a[::-1]).astype("<f4").tobytes())


def read_pfm(path):
    with open(path, "rb") as fh:
        if fh.readline().strip() != b"Pf":
            raise ValueError("not a grayscale PFM file")
        dims = fh.readline().split()
        if len(dims) != 2:
            raise ValueError("malformed PFM dimension line")
        w, h = int(dims[0]), int(dims[1])
        scale = float(fh.readline())
        raw = fh.read(w * h * 4)
    if len(raw) != w * h * 4:
        raise ValueError("PFM payload truncated")
    a = np.frombuffer(raw, dtype="<f4" if scale < 0 else ">f4").reshape(h, w)[::-1]
    a = a.astype(np.float64)
    a[a == 0.0] = np.inf
    return a


def write_pgm(path, img) -> None:
    a = np.asarray(img)
    data = np.where(a, 255, 0).astype(np.uint8) if a.dtype == bool else \
        np.round(np.clip(np.asarray(a, dtype=np.float64), 0.0, 1.0) * 255.0).astype(np.uint8)
    h, w = data.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{w} {h}\n255\n".encode() + data.tobytes())


def read_pgm(path):
    """8-bit binary PGM as uint8 (imageio.py:63-78)."""
    with open(path, "rb") as fh:
        if fh.readline().strip() != b"P5":
            raise ValueError("not a binary PGM file")
        line = fh.readline()
        while line.startswith(b"#"):
            line = fh.readline()
        w, h = (int(x) for x in line.split()[:2])
        maxval = int(fh.readline())
        if maxval != 255:
            raise ValueError(f"only maxval 255 supported, got {maxval}")
        raw = fh.read(w * h)
    if len(raw) != w * h:
        raise ValueError("PGM payload truncated")
    return np.frombuffer(raw, dtype=np.uint8).reshape(h, w).copy()
