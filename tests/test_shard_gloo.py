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

from paper_2602_23040_b200.shard import local_pairs, local_views, reduce_frame_gradients, reduce_gradients


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


def _frame_worker(rank, world, port, F, D, HA, WA, out):
    """C4 exchange: every rank holds per-frame gradients that are zero on the static texels (frozen);
    the compacted exchange over the dynamic texels must equal the full all-reduce."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(5)
    dyn_mask = torch.rand((HA, WA), generator=g) < 0.25
    gr = torch.Generator().manual_seed(100 + rank)
    grads = torch.randn((F, D, HA, WA), generator=gr) * dyn_mask
    full = grads.clone()
    loss = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dyn = torch.nonzero(dyn_mask.reshape(-1)).reshape(-1)
    reduce_frame_gradients(grads, loss, world, dyn)
    dist.all_reduce(full)
    out[rank] = (torch.equal(grads, full), float(loss.item()), int(dyn.numel()))
    dist.destroy_process_group()


def test_frame_exchange_compacted_equals_full():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_frame_worker, args=(2, port, 3, 5, 8, 12, out), nprocs=2, join=True)
    for r in range(2):
        assert out[r][0] and out[r][1] == 3.0 and 0 < out[r][2] < 96


@pytest.mark.parametrize("F,V,world", [(30, 55, 8), (30, 55, 3), (2, 3, 4), (1, 5, 2)])
def test_frame_view_pairs_round_robin(F, V, world):
    allp = sorted(p for r in range(world) for p in local_pairs(F, V, r, world))
    assert allp == [(f, v) for f in range(F) for v in range(V)]                  # coverage + disjointness
    sizes = [len(local_pairs(F, V, r, world)) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1                                           # balance (C4: 207 max at 8)
