"""Helpers for the GPU parity tests: run the CUDA path through the C-ABI binding and the
oracle on the same seeded inputs."""
import numpy as np
import torch

from paper_2502_18377_b200 import mpde


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def gpu_solve(shape, h, c, b, om, g=None, weights=(1.0, 1.0, 1.0, 1.0), opts=None, want_dz=True):
    """c [B][M][P], b/om [B][P] (numpy float32).  Returns dict of numpy arrays."""
    s = mpde.Solver(shape, h, to_dev(c), opts=opts, weights=weights)
    bd, od = to_dev(b), to_dev(om)
    z = s.forward(bd, od)
    out = {"z": z}
    torch.cuda.synchronize()
    out["stats_fwd"] = s.stats_list()
    if g is not None:
        gc, gb, gw, dz = s.backward(bd, z, to_dev(g), want_dz=want_dz)
        torch.cuda.synchronize()
        out.update(grad_c=gc, grad_b=gb, grad_omega=gw, dz=dz, stats_bwd=s.stats_list())
    s.close()
    return {k: (v.cpu().numpy().astype(np.float64) if torch.is_tensor(v) else v)
            for k, v in out.items()}


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
