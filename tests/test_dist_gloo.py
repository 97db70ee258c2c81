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
