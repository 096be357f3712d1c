"""world_size-2 gloo test of the theta-batch sharding host logic (CPU, no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import workloads as W
from paper_2205_10091_b200.dist import allreduce_loss_grad, row_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, E_all, G_all, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = row_block(E_all.shape[0], world, rank)
    red = allreduce_loss_grad(torch.as_tensor(E_all[a:b]), torch.as_tensor(G_all[a:b]))
    out[rank] = red.numpy().copy()
    dist.destroy_process_group()


def test_row_blocks_partition():
    for B in (1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            blocks = [row_block(B, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == B
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2])
def test_allreduce_loss_grad_gloo(world):
    from oracle import oracle as orc
    c, H = W.hea(5, 2), W.heisenberg(5)
    th = W.thetas(6, c.n_params, 3)
    E, G = orc.value_grad_batch(c, H, th)          # stand-in per-row results
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, E, G, out), nprocs=world, join=True)
    want = np.concatenate([[E.sum()], G.sum(0)])
    for r in range(world):
        np.testing.assert_allclose(out[r], want, rtol=1e-13, atol=1e-13)
