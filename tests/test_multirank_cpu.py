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
