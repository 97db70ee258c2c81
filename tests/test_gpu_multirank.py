"""Sharded solve == unsharded solve: two ranks each solve their shard
of a batch through the CUDA path and all-reduce the batch-summed grad_c; the per-PDE outputs
must equal, bit for bit, the same PDEs solved as one batch in one process, and the all-reduced
sum must equal the sum over the whole batch.

Only one GPU is available to the tests, so both ranks run on cuda:0 and the collective goes
over gloo (host-mediated): no rank's kernels wait on another rank's kernels, so this is two
independent solves plus a host all-reduce -- the same host logic bench.py runs over NCCL."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_RANK_SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import synth
from paper_2502_18377_b200 import mpde
from paper_2502_18377_b200.parallel import allreduce_coeff_grad, shard
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
cfg_name, total, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
dist.init_process_group("gloo")
torch.cuda.set_device(0)
start, cnt = shard(total, rank, world)
cfg = synth.CONFIGS[cfg_name]
bt = synth.make_batch(cfg_name, cnt, start=start)
g = synth.make_g(cfg_name, cnt, start=start)
dev = lambda a: torch.from_numpy(a).cuda()
s = mpde.Solver(cfg.shape, cfg.h, dev(bt["c"]))
z = s.forward(dev(bt["b"]), dev(bt["omega"]))
gc, gb, gw, _ = s.backward(dev(bt["b"]), z, dev(g))
gsum = torch.empty(gc.shape[1:], dtype=torch.float32, device="cuda")
mpde.mpde_batch_sum(gc, gsum)
torch.cuda.synchronize()
red = gsum.cpu()
allreduce_coeff_grad(red)   # gloo on the host copy (the bench all-reduces the device tensor over NCCL)
np.savez(out, z=z.cpu().numpy(), gc=gc.cpu().numpy(), gb=gb.cpu().numpy(), gw=gw.cpu().numpy(),
         red=red.numpy(), start=start, cnt=cnt)
s.close()
dist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cfg_name,total", [("C3", 4), ("C2", 5)])
def test_two_rank_shards_match_single_batch(cfg_name, total, tmp_path):
    import torch

    import synth
    from paper_2502_18377_b200 import mpde
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", _RANK_SCRIPT, cfg_name, str(total),
                                       str(tmp_path / f"r{r}.npz")], env=env, cwd=root))
    for p in procs:
        assert p.wait(timeout=600) == 0
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]

    cfg = synth.CONFIGS[cfg_name]
    bt = synth.make_batch(cfg_name, total)
    g = synth.make_g(cfg_name, total)
    dev = lambda a: torch.from_numpy(a).cuda()
    s = mpde.Solver(cfg.shape, cfg.h, dev(bt["c"]))
    z = s.forward(dev(bt["b"]), dev(bt["omega"]))
    gc, gb, gw, _ = s.backward(dev(bt["b"]), z, dev(g))
    torch.cuda.synchronize()
    full = {"z": z.cpu().numpy(), "gc": gc.cpu().numpy(), "gb": gb.cpu().numpy(), "gw": gw.cpu().numpy()}
    s.close()
    for p in parts:
        a, n = int(p["start"]), int(p["cnt"])
        for k in ("z", "gc", "gb", "gw"):
            assert np.array_equal(p[k], full[k][a:a + n]), f"{k} of PDEs {a}..{a + n - 1} differs"
    total_sum = full["gc"].astype(np.float64).sum(axis=0)
    for p in parts:
        err = np.abs(p["red"] - total_sum).max() / np.abs(total_sum).max()
        assert err < 1e-6, err
    assert np.array_equal(parts[0]["red"], parts[1]["red"])
