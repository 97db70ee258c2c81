import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu
from paper_2502_18377_b200 import mpde
shape, h, B = (20, 26), (0.05, 0.04), 3
rng = np.random.default_rng(31)
c = rng.normal(0.0, 0.5, (B, 5, 520)); c[:, 1] += 1.0
c = c.astype(np.float32)
s = mpde.Solver(shape, h, gu.to_dev(c), weights=(1.25, 2.0, 0.75, 0.875))
L = mpde.mpde_hierarchy_query(s.h_, 0, 0, None)[3]
for l in range(L):
    shp = mpde.mpde_hierarchy_query(s.h_, l, 0, None); Pl = shp[0] * shp[1]
    d = torch.empty((B, Pl), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 1, d)
    lm = torch.empty((B,), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 2, lm)
    cc = torch.empty((B, 5, Pl), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 3, cc)
    print(l, shp, "dinv finite", bool(torch.isfinite(d).all()), "min/max", d.min().item(), d.max().item(), "lmax", lm.tolist(), "c finite", bool(torch.isfinite(cc).all()))
Pc = shp[0] * shp[1]
si = torch.empty((B, Pc, Pc), device="cuda"); mpde.mpde_hierarchy_query(s.h_, L - 1, 4, si)
print("sinv finite", bool(torch.isfinite(si).all()), si.abs().max().item())
r = torch.randn((B, 520), device="cuda"); z = torch.empty_like(r)
mpde.mpde_apply_precond(s.h_, r, z); print("precond finite", bool(torch.isfinite(z).all()), (r * z).sum(1).tolist())
