"""Small fwd+bwd solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 heat (dense-path and multigrid), a 16^3 3D problem and, with MPDE_MARCH=2, the t-marching
kernel.  python tools/sanitize_case.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2502_18377_b200 import mpde
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
bt = synth.make_batch("C1"); g = synth.make_g("C1"); cfg = bt["cfg"]
for opts in (None, mpde.mpde_default_options(levels_max=1)):
    s = mpde.Solver(cfg.shape, cfg.h, dev(bt["c"]), opts=opts)
    z = s.forward(dev(bt["b"]), dev(bt["omega"])); s.backward(dev(bt["b"]), z, dev(g)); torch.cuda.synchronize(); s.close()
rng = np.random.default_rng(1)
shape, B = (16, 16, 32), 2
P = int(np.prod(shape))
c = rng.normal(0, 0.5, (B, 7, P)); c[:, 1] += 1
s = mpde.Solver(shape, (0.05, 0.06, 0.07), dev(c), opts=mpde.mpde_default_options(max_iters=6, max_refine=2),
                bc=(("D", "-"), ("N", "D"), ("D", "N")))
z = s.forward(dev(rng.normal(size=(B, P))), dev(rng.normal(size=(B, P))), omega_n=dev(rng.normal(size=(B, 3, P))))
s.backward(dev(rng.normal(size=(B, P))), z, dev(rng.normal(size=(B, 7, P))), want_grad_omega_n=True)
torch.cuda.synchronize(); s.close()
print("ok")
