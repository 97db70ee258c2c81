"""World-size-2 gloo test of the multi-GPU host logic (batch sharding, the grad_c
all-reduce and the max-over-ranks timing) on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_18377_b200.parallel import allreduce_coeff_grad, max_over_ranks, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, cnt = shard(total, rank, world)
    g = torch.Generator().manual_seed(1234)
    full = torch.randn(total, 7, 50, generator=g)          # per-PDE grad_c of the whole batch
    local = full[start:start + cnt].sum(0)                  # what mpde_batch_sum gives per rank
    allreduce_coeff_grad(local)
    m = max_over_ranks(float(rank + 1))
    out[rank] = (start, cnt, float((local - full.sum(0)).abs().max()), m)
    dist.destroy_process_group()


def test_shard_covers_batch():
    for total in (1, 7, 32, 256):
        for world in (1, 2, 3, 8):
            spans = [shard(total, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == total
            assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


@pytest.mark.timeout(120)
def test_allreduce_equals_sum_of_local_gradients():
    world, total = 2, 9
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    assert sorted(out.keys()) == [0, 1]
    assert out[0][:2] == (0, 5) and out[1][:2] == (5, 4)
    for r in range(world):
        assert out[r][2] < 1e-5      # all-reduced batch sum == sum over the full batch
        assert out[r][3] == 2.0      # max over ranks


def _theta_worker(rank, world, port, total, out):
    import numpy as np

    from oracle.template import template_grad
    from paper_2502_18377_b200.parallel import allreduce_theta_grad
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, cnt = shard(total, rank, world)
    rng = np.random.default_rng(77)
    th = rng.normal(size=(6, 6))
    feat = rng.normal(size=(total, 2, 40))
    gc = rng.normal(size=(total, 5, 40))
    gb = rng.normal(size=(total, 40))
    local, _ = template_grad(th, feat[start:start + cnt], 2, gc[start:start + cnt],
                             gb[start:start + cnt])
    t = torch.from_numpy(local)
    allreduce_theta_grad(t)
    full, _ = template_grad(th, feat, 2, gc, gb)
    out[rank] = float(np.abs(t.numpy() - full).max() / np.abs(full).max())
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_theta_grad_allreduce_equals_full_batch():
    """The discovery step's collective (N2): theta is shared by the global batch, so the
    all-reduced per-rank dl/dtheta equals dl/dtheta of the whole batch."""
    world, total = 2, 5
    out = mp.Manager().dict()
    mp.spawn(_theta_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    assert sorted(out.keys()) == [0, 1]
    assert max(out.values()) < 1e-12
