"""CPU, world size 2 over gloo: the multi-GPU host logic.

* view sharding covers every view exactly once, balanced;
* tile sharding is a partition;
* the fitting config's only collective (gradient all-reduce) sums the ranks'
  per-kernel gradients exactly once, in one flat bucket.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_15401_b200.distributed import allreduce_gradients, shard_tiles, shard_views


@pytest.mark.parametrize("views,world", [(64, 1), (64, 2), (64, 8), (7, 4), (3, 8)])
def test_shard_views_partition(views, world):
    got = [shard_views(views, r, world) for r in range(world)]
    flat = sorted(v for part in got for v in part)
    assert flat == list(range(views))
    sizes = [len(p) for p in got]
    assert max(sizes) - min(sizes) <= 1


def test_shard_tiles_partition():
    parts = [shard_tiles(4096, r, 8) for r in range(8)]
    assert sorted(np.concatenate(parts).tolist()) == list(range(4096))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k = 11
    rng = np.random.default_rng(rank)
    d_center = torch.tensor(rng.normal(size=(k, 3)))
    d_attr = torch.tensor(rng.normal(size=(k, 3)))
    mine = (d_center.clone(), d_attr.clone())
    allreduce_gradients([d_center, d_attr])
    out[rank] = (mine[0].numpy(), mine[1].numpy(), d_center.numpy(), d_attr.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gradient_allreduce_gloo_world2():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    want_c = out[0][0] + out[1][0]
    want_a = out[0][1] + out[1][1]
    for r in range(world):
        np.testing.assert_allclose(out[r][2], want_c, rtol=0, atol=1e-15)
        np.testing.assert_allclose(out[r][3], want_a, rtol=0, atol=1e-15)
