"""Multi-rank latent optimisation on the product path, run as two
ranks on the one available GPU: each rank is a process that drives
LatentOptimizer.step() on its skewed round-robin share of the pixel tiles of every
view (paper_1911_13225_b200/shard.py), with gloo carrying the two tiny
per-iterate collectives.  The ranks' kernels never wait on each other (the
collectives are host-side), so sharing one GPU changes timing only.

Checked: the iterates (codes after every Adam step) and the loss history are
bit-identical for world sizes 1 and 2, and the codes are bit-identical to the
unsharded single-process optimiser over the whole views (the exact fixed-point
column sums make the gradient independent of the partition).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ITERS = 3


def _problem(st, skip=-1):
    from paper_1911_13225_b200.workloads import render_depth_observations, ring_views, target_code
    field = (st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3", skip=skip) if skip >= 0
             else st.NeuralField.geometric(256, (512,) * 8, 0, precision="fp16x3"))
    views = ring_views(2, 128)
    cfg = st.TraceConfig(k_samples=3)
    obs = render_depth_observations(field, target_code(1), views, cfg).cpu().numpy()
    sil = np.isfinite(obs).astype(np.float64)
    return field, views, cfg, {"depth": obs, "silhouette": sil}


def _run(st, shard=None, skip=-1):
    field, views, cfg, obs = _problem(st, skip)
    opt = st.LatentOptimizer(field, views, obs, np.zeros((1, 256)), cfg, max_iters=ITERS,
                             shard=shard)
    codes = []
    for _ in range(ITERS):
        opt.step()
        codes.append(opt.code.cpu().numpy().copy())
    return np.stack(codes), opt.losses()[:, 0]


def _worker(rank, world, port, out, skip=-1):
    import torch
    import torch.distributed as dist
    import paper_1911_13225_b200 as st
    from paper_1911_13225_b200.shard import TileShard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    codes, losses = _run(st, TileShard(rank, world, 32), skip)
    out[rank] = (codes.tolist(), losses.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("skip", [-1, 4])
def test_two_ranks_one_gpu_bit_identical_iterates(skip):
    """skip=4: the DeepSDF decoder, whose exact column sums carry the skip
    layer's code rows as a second block."""
    import torch.multiprocessing as mp
    import paper_1911_13225_b200 as st
    from paper_1911_13225_b200.shard import TileShard
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(_worker, args=(2, port, out, skip), nprocs=2, join=True)
    c1, l1 = _run(st, TileShard(0, 1, 32), skip)      # one rank, the same tiles
    c0, l0 = _run(st, None, skip)                      # unsharded whole views
    for r in range(2):
        assert np.array_equal(np.asarray(out[r][0]), c1), f"rank {r} iterates differ from world 1"
        assert np.array_equal(np.asarray(out[r][1]), l1), f"rank {r} losses differ from world 1"
    assert np.array_equal(c1, c0), "tiled iterates differ from the unsharded optimiser"
    np.testing.assert_allclose(l1, l0, rtol=1e-12)
    assert np.linalg.norm(c1[-1]) > 0
