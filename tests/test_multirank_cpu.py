"""World-size-2 gloo test of the multi-GPU decomposition used by bench.py /
LatentOptimizer.step(reduce_fn): each rank owns a shard of the views, computes
its partial latent gradient (depth terms normalised per view, latent
regulariser on rank 0 only), the gradient and loss are all-reduced, and every
rank takes the same Adam step.  Checked against a single-process computation
over all views (optimize.py:309-351 pattern), with the oracle as the math."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_weights, load_golden

import sdf_oracle as orc

V, RES = 4, 16


def _problem():
    g = load_golden("tiny64.npz")
    dec = orc.Decoder(golden_weights(g), 2)
    cams = [orc.cam_look_at(orc.ring_eye(k, V), RES, RES) for k in range(V)]
    cfg = orc.Cfg(k_samples=3, coarse_start_scale=1)
    obs = [orc.depth_map(orc.trace(lambda p: dec(p, g["code"] + 0.05), c, cfg), cfg) for c in cams]
    return dec, cams, cfg, obs, np.asarray(g["code"], dtype=np.float64)


def _partial(dec, cams, cfg, obs, z, views, with_reg):
    w = orc.Weights(latent=1.0 if with_reg else 0.0)
    tot, grad = 0.0, np.zeros_like(z)
    for v in views:
        t, _, gr, _, _, _ = orc.objective(dec, z, cams[v], cfg, w, depth=obs[v])
        tot += t
        grad += gr
        w = orc.Weights(latent=0.0)   # regulariser only once per rank-0 partial
    return tot, grad


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dec, cams, cfg, obs, z = _problem()
    mine = list(range(rank, V, world))
    adam = orc.Adam()
    for _ in range(2):
        tot, grad = _partial(dec, cams, cfg, obs, z, mine, with_reg=(rank == 0))
        t = torch.tensor(np.concatenate([[tot], grad]))
        dist.all_reduce(t)
        z = adam.step(z, t[1:].numpy())
    out[rank] = z.tolist()
    dist.destroy_process_group()


def test_two_rank_allreduce_matches_single_process():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    dec, cams, cfg, obs, z = _problem()
    adam = orc.Adam()
    for _ in range(2):
        _, grad = _partial(dec, cams, cfg, obs, z, list(range(V)), with_reg=True)
        z = adam.step(z, grad)
    np.testing.assert_allclose(out[0], z, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(out[1], out[0], rtol=0, atol=0)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_interleaved_view_sharding_partitions_the_ring(world):
    """bench.py's weak-scaling shard: rank r traces ring views r, r+N, ..., r+7N
    of an 8N-view ring; together the ranks cover every view exactly once, and
    N=1 is the plain 8-view ring."""
    from paper_1911_13225_b200.workloads import ring_eye, ring_views
    total = 8 * world
    seen = []
    for r in range(world):
        views = ring_views(8, 16, first=r, total=total, stride=world)
        assert len(views) == 8
        for j, (_, pose) in enumerate(views):
            k = r + j * world
            np.testing.assert_allclose(pose.center(), ring_eye(k, total), rtol=0, atol=1e-8)
            seen.append(k)
    assert sorted(seen) == list(range(total))
    if world == 1:
        plain = ring_views(8, 16)
        for (_, a), (_, b) in zip(plain, ring_views(8, 16, first=0, total=8, stride=1)):
            np.testing.assert_array_equal(a.params(), b.params())


# --- pixel-tile sharding of the product path (paper_1911_13225_b200/shard.py) ----

@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_tile_split_partitions_every_pixel_once(world):
    from paper_1911_13225_b200.shard import tile_split
    from paper_1911_13225_b200.workloads import ring_views
    views = ring_views(3, 64)
    seen = np.zeros((3, 64, 64), np.int64)
    total = None
    for r in range(world):
        tiles, total = tile_split(views, 16, r, world)
        for t in tiles:
            # skewed deal: row ty of view v shifted by 3 ty + v (shard.DEAL_SKEW)
            assert (t.x0 // 16 + 3 * (t.y0 // 16) + t.view) % world == r
            seen[t.view, t.y0:t.y0 + 16, t.x0:t.x0 + 16] += 1
        if world in (1, 2):   # 4 tiles per row: every rank gets the same count
            assert len(tiles) == 3 * 16 // world
    assert total == 3 * 16 and np.all(seen == 1)
    with pytest.raises(ValueError):
        tile_split(views, 6, 0, world)   # not a multiple of the coarse block


def test_tile_rays_are_bit_identical_to_the_parent_view():
    """camera.py:190-212 on a tile (principal point shifted, parent focal
    length) reproduces the parent's camera-space ray of every pixel exactly, at
    every coarse-to-fine level."""
    from paper_1911_13225_b200.camera import Intrinsics
    from paper_1911_13225_b200.shard import tile_split
    from paper_1911_13225_b200.workloads import ring_views
    for cx in (None, 250.3):
        intr = Intrinsics(width=128, height=128, cx=cx, cy=None if cx is None else 61.7)
        views = [(intr, ring_views(1, 128)[0][1])]
        tiles, _ = tile_split(views, 32, 0, 1)
        pcx, pcy = intr.center
        for t in tiles:
            for L in (1, 2, 4):
                w = 32 // L
                j, i = np.divmod(np.arange(w * w), w)
                tcx, tcy = t.intr.center
                vt = np.stack([((i + 0.5) * L - tcx) / t.intr.fx, ((j + 0.5) * L - tcy) / t.intr.fy], 1)
                ip, jp = i + t.x0 // L, j + t.y0 // L
                vp = np.stack([((ip + 0.5) * L - pcx) / intr.fx, ((jp + 0.5) * L - pcy) / intr.fy], 1)
                assert np.array_equal(vt, vp)


def _fixed_worker(rank, world, port, out):
    from paper_1911_13225_b200.shard import fixed_all_reduce
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    vals = [int(x) for x in rng.integers(-2 ** 62, 2 ** 62, 64)]
    vals = [v * (1 << int(s)) for v, s in zip(vals, rng.integers(0, 60, 64))]   # up to 2^122
    buf = torch.zeros((64, 2), dtype=torch.int64)
    for k, v in enumerate(vals):
        u = v % (1 << 128)
        buf[k, 0] = (u & ((1 << 64) - 1)) - (1 << 64 if u & (1 << 63) else 0)
        hi = u >> 64
        buf[k, 1] = hi - (1 << 64 if hi & (1 << 63) else 0)
    fixed_all_reduce(buf, None, world)
    out[rank] = (vals, buf.view(torch.int32).reshape(-1, 4).numpy().tolist())
    dist.destroy_process_group()


def test_fixed_point_all_reduce_is_exact():
    """The 128-bit column sums of dist_objective_io.colsum_fixed reduce over two
    gloo ranks to the exact integer sum (limb carries across all 128 bits)."""
    from paper_1911_13225_b200.shard import int128_from_limbs
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_fixed_worker, args=(2, port, out), nprocs=2, join=True)
    exact = [a + b for a, b in zip(out[0][0], out[1][0])]
    for r in range(2):
        assert int128_from_limbs(np.asarray(out[r][1])) == exact


def _terms_worker(rank, world, port, out):
    from paper_1911_13225_b200.shard import all_reduce_sum, tile_split, view_totals
    from paper_1911_13225_b200.workloads import ring_views
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = ring_views(4, 64)
    tiles, T = tile_split(views, 16, rank, world)
    rng = np.random.default_rng(11)
    per_tile = rng.standard_normal((T, 6)) * 10.0 ** rng.integers(-8, 3, (T, 6))
    g = torch.zeros((T, 6), dtype=torch.float64)
    idx = torch.tensor([t.index for t in tiles])
    g[idx] = torch.from_numpy(per_tile[idx.numpy()])
    all_reduce_sum(g, None, world)
    out[rank] = view_totals(g, 4).numpy().tolist()
    dist.destroy_process_group()


def test_per_view_loss_totals_identical_for_any_world_size():
    """Each tile's loss row is written by exactly one rank, so the all-reduced
    [T, 6] array is the same bits for world 1 and 2, and so is its per-view sum."""
    from paper_1911_13225_b200.shard import view_totals
    import socket
    res = {}
    for world in (1, 2):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        out = mp.Manager().dict()
        mp.spawn(_terms_worker, args=(world, port, out), nprocs=world, join=True)
        res[world] = [out[r] for r in range(world)]
    assert res[1][0] == res[2][0] == res[2][1]
