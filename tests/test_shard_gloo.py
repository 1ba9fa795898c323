"""View sharding on CPU with the gloo backend, world size 2 and 3 (no GPU).

The per-rank renderer is replaced by a stand-in whose gradient contribution
is a known function of the view index, so the test checks exactly what the
sharding layer owns: the round-robin partition (coverage, disjointness,
balance) and the wiring of the single all-reduce of the gradient planes and
the loss."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_23040_b200.shard import local_views, reduce_gradients


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_views, shape, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = local_views(n_views, rank, world)
    grad = torch.zeros(shape, dtype=torch.float32)
    loss = torch.zeros(1, dtype=torch.float64)
    for v in views:   # stand-in render_backward: view v adds (v + 1) * pattern
        grad += (v + 1) * torch.arange(grad.numel(), dtype=torch.float32).reshape(shape) / grad.numel()
        loss += float(v * v)
    reduce_gradients(grad, loss, world)
    out[rank] = (views, grad.clone(), float(loss.item()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_views", [(2, 64), (3, 55), (2, 1)])
def test_round_robin_allreduce(world, n_views):
    if n_views < world:
        # a rank without views is a configuration error the stepper rejects
        assert local_views(n_views, 1, world) == []
        return
    port = _free_port()
    shape = (4, 3, 5)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, n_views, shape, out), nprocs=world, join=True)
    all_views = sorted(v for r in range(world) for v in out[r][0])
    assert all_views == list(range(n_views))                                   # coverage + disjointness
    sizes = [len(out[r][0]) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1                                        # balance
    pattern = torch.arange(60, dtype=torch.float32).reshape(shape) / 60
    expect = sum(v + 1 for v in range(n_views)) * pattern
    for r in range(world):
        torch.testing.assert_close(out[r][1], expect, rtol=1e-6, atol=1e-5)   # every rank holds the sum
        assert out[r][2] == float(sum(v * v for v in range(n_views)))


def test_single_rank_is_identity():
    g = torch.ones(2, 2)
    loss = torch.ones(1, dtype=torch.float64)
    reduce_gradients(g, loss, 1)
    assert torch.equal(g, torch.ones(2, 2)) and loss.item() == 1.0
    assert local_views(5, 0, 1) == [0, 1, 2, 3, 4]
