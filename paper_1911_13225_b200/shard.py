"""Views sharded over ranks as pixel tiles -- SURVEY 8(e), strong scaling of C3.

The reference sums per-view gradients on one host (optimize.py:309-351,
`g += hg["code"]` at :340, the regulariser once at :341).  Here every view is
cut into `tile` x `tile` pixel tiles (a multiple of the coarse-to-fine block,
so the split tree tracer.py:196-218 never crosses a tile) and the tiles of all
views are dealt round-robin (skewed per tile row) over the ranks, so every rank marches rays of
every view and the per-view cost skew averages out.

A tile is traced as a view of its own: same rotation, centre and focal
length, principal point shifted by the tile origin.  Its pixel rays are
bit-identical to the parent view's (camera.py:190-212 evaluates
((i + .5) L - cx) / fx; with cx' = cx - x0 both differences are exact), so a
tile's march equals the same pixels of the whole view.

One iterate on a rank = trace(its tiles) -> dist_objective phase 1 (per-tile
counts) -> all-reduce of the per-view counts (n_px, n_normal: the
normalisers of losses.py:61-111 are whole-view quantities) -> phase 2 (seeds
and the fused backward with the whole views' normalisers) -> an exact
all-reduce of the fixed-point gradient column sums and a fixed-order sum of the
per-tile loss terms -> dist_code_grad_fixed -> Adam.  Integer sums are
associative, so the iterates are bit-identical for any number of ranks.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .camera import Intrinsics


@dataclass(frozen=True)
class TileIntrinsics(Intrinsics):
    """A pixel tile of a parent view: fx/fy of the parent, principal point
    shifted by the tile origin (camera.py:25-61 derives fx from the width,
    which a tile must not change)."""
    fx_parent: float = 0.0

    @property
    def fx(self) -> float:
        return self.fx_parent


@dataclass
class TileShard:
    """rank/world of the split, the tile size and the torch.distributed group
    (None: the default group; world 1 needs no process group at all)."""
    rank: int = 0
    world: int = 1
    tile: int = 32
    group: object = None


@dataclass
class Tile:
    index: int          # global tile index (view-major, row-major within the view)
    view: int           # parent view
    x0: int
    y0: int
    intr: TileIntrinsics
    pose: object


# Tile (tx, ty) of view v goes to rank (tx + DEAL_SKEW * ty + v) % world: each
# row of tiles is dealt round-robin, shifted by DEAL_SKEW per row, so a rank's
# tiles form diagonal stripes a few tiles apart instead of whole tile columns
# (a centred object made the column deal uneven).  0: plain round-robin over
# the global tile order.
DEAL_SKEW = 3


def _owner(t: int, tx: int, ty: int, v: int, world: int) -> int:
    if DEAL_SKEW == 0:
        return t % world
    return (tx + DEAL_SKEW * ty + v) % world


def tile_split(views, tile: int, rank: int, world: int, coarse: int = 4):
    """The tiles of `rank` (row-skewed round-robin, DEAL_SKEW) and the
    total tile count."""
    if tile % coarse:
        raise ValueError(f"tile {tile} must be a multiple of coarse_start_scale {coarse}")
    if not (0 <= rank < world):
        raise ValueError("rank must be in [0, world)")
    out, t = [], 0
    for v, (intr, pose) in enumerate(views):
        if intr.width % tile or intr.height % tile:
            raise ValueError(f"view {v}: {intr.width}x{intr.height} is not a multiple of tile {tile}")
        cx, cy = intr.center
        for y0 in range(0, intr.height, tile):
            for x0 in range(0, intr.width, tile):
                if _owner(t, x0 // tile, y0 // tile, v, world) == rank:
                    ti = TileIntrinsics(intr.focal_mm, intr.sensor_mm, tile, tile, cx - x0, cy - y0,
                                        fx_parent=intr.fx)
                    out.append(Tile(t, v, x0, y0, ti, pose))
                t += 1
    return out, t


# --- exact collectives --------------------------------------------------------

def _backend(group):
    import torch.distributed as dist
    try:
        return dist.get_backend(group)
    except Exception:
        return "gloo"


def all_reduce_sum(t, group=None, world: int = 1):
    """In-place SUM over ranks (NCCL on device tensors; gloo through host copies)."""
    if world <= 1:
        return t
    import torch
    import torch.distributed as dist
    if _backend(group) == "nccl" or t.device.type == "cpu":
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t
    h = t.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    t.copy_(h.to(t.device))
    return t


def fixed_all_reduce(buf, group=None, world: int = 1):
    """Exact SUM over ranks of 128-bit two's-complement integers (the
    fixed-point column sums of dist_objective_io.colsum_fixed, stored as
    [..., 2] int64 = (low word, high word)): split into four 32-bit limbs held
    in int64 (sums of up to 2^31 ranks cannot overflow them), all-reduce, then
    propagate the carries; modulo 2^128 this is the exact integer sum."""
    if world <= 1:
        return buf
    import torch
    u32 = buf.contiguous().view(torch.int32).reshape(-1, 4)
    limbs = u32.to(torch.int64) & 0xFFFFFFFF
    all_reduce_sum(limbs, group, world)
    out = torch.empty_like(limbs)
    carry = torch.zeros_like(limbs[:, 0])
    for k in range(4):
        s = limbs[:, k] + carry
        out[:, k] = s & 0xFFFFFFFF
        carry = s >> 32
    # back to int32 limbs (two's complement reinterpretation of 0..2^32-1)
    res = torch.where(out >= 2 ** 31, out - 2 ** 32, out).to(torch.int32)
    buf.view(torch.int32).reshape(-1, 4).copy_(res)
    return buf


def view_totals(tile_terms_global, n_views: int):
    """[T, k] per-tile terms (tiles view-major, equal count per view) -> [V, k]
    per-view sums, in a fixed order (the same on every rank and for any
    world size: the input is the same array everywhere)."""
    T, k = tile_terms_global.shape
    return tile_terms_global.reshape(n_views, T // n_views, k).sum(dim=1)


def int128_from_limbs(limbs: np.ndarray) -> list:
    """Host helper (tests): [n, 4] int32 limbs -> Python ints (signed 128-bit)."""
    out = []
    for row in np.asarray(limbs, dtype=np.int64):
        v = 0
        for k in range(4):
            v |= (int(row[k]) & 0xFFFFFFFF) << (32 * k)
        if v >= 1 << 127:
            v -= 1 << 128
        out.append(v)
    return out
