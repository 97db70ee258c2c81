import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu
from test_gpu_parity import _rand_problem
from paper_2502_18377_b200 import mpde
shape, h, B = (16, 16), (1/15, 1/15), 2
c, b, om, g = _rand_problem(shape, B, 31)
s = mpde.Solver(shape, h, gu.to_dev(c), weights=(1.25, 2.0, 0.75, 0.875))
for l in range(2):
    shp = mpde.mpde_hierarchy_query(s.h_, l, 0, None); Pl = shp[0] * shp[1]
    d = torch.empty((B, Pl), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 1, d)
    lm = torch.empty((B,), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 2, lm)
    print(l, shp, "dinv min/max per pde", d.min(1).values.tolist(), d.max(1).values.tolist(), "lmax", lm.tolist())
np.savez("gpurun_out/d1616.npz", c=c)
si = torch.empty((B, 64, 64), device="cuda"); mpde.mpde_hierarchy_query(s.h_, 1, 4, si)
print("sinv finite per pde", [bool(torch.isfinite(si[i]).all()) for i in range(B)], si.abs().amax((1, 2)).tolist())
r = torch.randn((B, 256), device="cuda"); z = torch.empty_like(r)
mpde.mpde_apply_precond(s.h_, r, z); print("precond finite", [bool(torch.isfinite(z[i]).all()) for i in range(B)], (r * z).sum(1).tolist())
np.save("gpurun_out/sinv1616.npy", si.cpu().numpy())
