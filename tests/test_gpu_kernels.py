"""GPU unit tests of the condensed operator paths at sizes that select each kernel variant
(scalar, 4-points-per-thread, 2x2-blocked, fused single-kernel) against the Schur complement
built from the oracle's A, and symmetry / positivity of the V-cycle preconditioner."""
import numpy as np
import pytest
import torch

from oracle import Problem, assemble

pytestmark = pytest.mark.gpu


def _dense_schur(pr, c):
    A, _, _ = assemble(pr, c, np.zeros(pr.P), np.zeros(pr.P))
    N = (A.T @ A).toarray()
    P = pr.P
    return N[:P, :P] - N[:P, P:] @ np.linalg.solve(N[P:, P:], N[P:, :P])


@pytest.mark.parametrize("shape,h", [((9, 10, 12), (0.1, 0.08, 0.05)),    # v4 (n_y % 4 == 0)
                                     ((15, 17, 16), (0.05, 0.06, 0.07)),  # 2x2 blocked, odd t/x
                                     ((16, 18, 20), (0.05, 0.06, 0.07)),  # 2x2 blocked, interior
                                     ((8, 9, 11), (0.1, 0.1, 0.1)),       # scalar path
                                     ((20, 24), (0.05, 0.04))])           # 2D v4
def test_schur_variants_match_dense(shape, h):
    from paper_2502_18377_b200 import mpde
    rng = np.random.default_rng(5)
    D = len(shape)
    M, P, B = 1 + 2 * D, int(np.prod(shape)), 2
    c = rng.normal(0.0, 0.5, (B, M, P))
    c[:, 1] += 1.0
    c = c.astype(np.float32)
    w = (1.25, 2.0, 0.75, 0.875)
    s = mpde.Solver(shape, h, torch.from_numpy(c).cuda(), weights=w,
                    opts=mpde.mpde_default_options(levels_max=2))
    x = rng.normal(size=(B, P)).astype(np.float32)
    y = torch.empty((B, P), dtype=torch.float32, device="cuda")
    mpde.mpde_apply_schur(s.h_, 0, torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    pr = Problem(shape, h, *w)
    for i in range(B):
        S = _dense_schur(pr, c[i].astype(np.float64))
        ref = S @ x[i]
        assert np.linalg.norm(y[i].cpu().numpy() - ref) <= 1e-4 * np.linalg.norm(ref)
    s.close()


def _sparse_schur_apply(pr, c, x):
    """S x = N_pp x - N_pd N_dd^-1 N_dp x with sparse N = A^T A (N_dd block-diagonal)."""
    import scipy.sparse.linalg as sla
    A, _, _ = assemble(pr, c, np.zeros(pr.P), np.zeros(pr.P))
    N = (A.T @ A).tocsc()
    P = pr.P
    Npp, Npd, Ndp, Ndd = N[:P, :P], N[:P, P:], N[P:, :P], N[P:, P:]
    return Npp @ x - Npd @ sla.splu(Ndd.tocsc()).solve(Ndp @ x)


_APPLY_SCRIPT = r"""
import sys, numpy as np, torch
from paper_2502_18377_b200 import mpde
d = np.load(sys.argv[1])
shape, h, w = tuple(int(v) for v in d["shape"]), tuple(d["h"]), tuple(d["w"])
s = mpde.Solver(shape, h, torch.from_numpy(d["c"]).cuda(), weights=w)
y = torch.empty(d["x"].shape, dtype=torch.float32, device="cuda")
mpde.mpde_apply_schur(s.h_, 0, torch.from_numpy(d["x"]).cuda(), y)
torch.cuda.synchronize()
np.save(sys.argv[2], y.cpu().numpy())
np.save(sys.argv[3], np.array(mpde.mpde_hierarchy_query(s.h_, 0, 5, None)))
"""


# (shape, h, env, expected [pass 1, pass 2] kernel codes of mpde_hierarchy_query(what=5)):
# levels above MPDE_SMALLP = 16384 points per vector select the production kernels; below it
# the 64-thread v4 kernels run whatever the switches say, so the variant cases set
# MPDE_SMALLP=0 and every case asserts the kernel that actually ran.
_NOSMALL = {"MPDE_SMALLP": "0", "MPDE_MARCH": "0", "MPDE_SMALL_FUSED": "0", "MPDE_SLAB": "0"}
_NOMARCH = {"MPDE_MARCH": "0"}
_MARCH = {"MPDE_MARCH": "2"}  # the march on every eligible level, whatever the grid size
@pytest.mark.parametrize("shape,h,env,kinds,B", [
    # production: the one-kernel t-marching apply (code 9, march.cu) on launches with >= 148 CTAs
    ((6, 64, 64), (0.01, 1 / 64, 1 / 64), {"MPDE_MARCH": "1"}, (9, 9), 19),  # C4 level-0 geometry, 152 CTAs
    ((6, 64, 64), (0.01, 1 / 64, 1 / 64), {}, (1, 4), 19),     # default: two-pass <64,64>
    ((20, 32, 32), (0.02, 1 / 32, 1 / 32), {"MPDE_SLAB": "1"}, (11, 11), 2),    # mid-size level: t-slab clusters (5 CTAs)
    ((16, 32, 32), (0.02, 1 / 32, 1 / 32), {"MPDE_SLAB": "1"}, (11, 11), 3),    # C4 level-1 geometry (4-CTA clusters)
    ((32, 32, 32), (0.05, 0.3125, 0.3125), {"MPDE_SLAB": "1"}, (11, 11), 2),    # C3 level-0 geometry (8-CTA clusters)
    ((12, 24, 40), (0.03, 0.04, 0.02), {"MPDE_SLAB": "1"}, (11, 11), 2),        # 3 slabs, 960-point planes
    ((20, 32, 32), (0.02, 1 / 32, 1 / 32), {}, (1, 4), 2),      # default: two-pass <32,32>
    ((20, 32, 32), (0.02, 1 / 32, 1 / 32), _MARCH, (9, 9), 2),  # NY 32, 4 strips
    ((7, 16, 64), (0.05, 0.06, 0.07), _MARCH, (9, 9), 2),       # 2 strips, both edge strips
    ((9, 24, 32), (0.05, 0.06, 0.07), _MARCH, (9, 9), 2),       # 3 strips, one interior strip
    ((11, 40, 64), (0.03, 0.04, 0.02), _MARCH, (9, 9), 2),      # 5 strips, t extent 11
    ((8, 64, 128), (0.02, 0.03, 0.01), _MARCH, (9, 9), 2),      # NY 128 (512-thread CTAs)
    # the two-pass kernels the march replaces (and where it does not apply)
    ((6, 64, 64), (0.01, 1 / 64, 1 / 64), _NOMARCH, (1, 4), 2), # t-blocked pass 2 <64,64>
    ((6, 128, 128), (0.005, 1 / 128, 1 / 128), {}, (1, 4), 2),  # C5 level 0: 16 strips > 8, <128,128>
    ((17, 24, 48), (0.05, 0.06, 0.07), {}, (1, 3), 2),          # runtime extents (NY4 = 12, no remap)
    ((6, 16, 16), (0.05, 0.06, 0.07), {"MPDE_SMALL_FUSED": "1"}, (10, 10), 3),  # small level, one CTA per PDE
    ((7, 16, 32), (0.05, 0.06, 0.07), {"MPDE_SMALL_FUSED": "1"}, (10, 10), 2),  # P = 3584 (opt-in kernel)
    ((8, 16, 16), (0.05, 0.06, 0.07), {"MPDE_SLAB": "1"}, (11, 11), 3),         # C4 level-2 geometry: 2-CTA t-slab clusters
    ((7, 16, 32), (0.05, 0.06, 0.07), {"MPDE_FUSED": "1", **_NOSMALL}, (7, 7), 2),  # fused, 2 x-tiles
    ((9, 24, 36), (0.04, 0.03, 0.05), {"MPDE_FUSED": "1", **_NOSMALL}, (7, 7), 2),  # fused, interior tile
    ((7, 16, 64), (0.05, 0.06, 0.07), _NOSMALL, (1, 3), 2),      # t-blocked, natural quad mapping (NY4=16)
    ((7, 16, 64), (0.05, 0.06, 0.07), {"MPDE_REMAP": "1", **_NOSMALL}, (1, 3), 2),  # warp-specialised y quads
    ((8, 10, 32), (0.05, 0.06, 0.07), {"MPDE_REMAP": "1", **_NOSMALL}, (1, 3), 2),  # NY4=8 (4 interior / 4 edge)
    ((7, 16, 64), (0.05, 0.06, 0.07), {"MPDE_HY": "1", "MPDE_REMAP": "1", **_NOSMALL}, (8, 3), 2),  # y part in pass 1
    ((9, 12, 32), (0.05, 0.06, 0.07), {"MPDE_HY": "1", "MPDE_REMAP": "1", **_NOSMALL}, (8, 3), 2),
    ((7, 16, 64), (0.05, 0.06, 0.07), {"MPDE_TILE": "1", **_NOSMALL}, (1, 6), 2),   # smem-tiled pass 2
    ((13, 12, 32), (0.05, 0.06, 0.07), {"MPDE_TILE": "1", **_NOSMALL}, (1, 6), 2),  # partial last t tile
    ((9, 16, 64), (0.05, 0.06, 0.07), {"MPDE_B22_TP": "4", "MPDE_REMAP": "1", **_NOSMALL}, (1, 3), 2),  # t-pair CTA tiling
    ((9, 16, 64), (0.05, 0.06, 0.07), {"MPDE_SCHUR_BLOCK": "2", **_NOSMALL}, (1, 5), 2)])  # 2x2 blocking
def test_large_schur_matches_sparse(shape, h, env, kinds, B, tmp_path):
    """S apply through every 3D kernel variant, incl. the production instantiations the
    bench runs (the selection switches are read once per process, so the apply runs in a child
    process), against S applied through the oracle's sparse A (no dense N at these sizes)."""
    import os
    import subprocess
    import sys
    rng = np.random.default_rng(7)
    M, P = 7, int(np.prod(shape))
    c = rng.normal(0.0, 0.5, (B, M, P))
    c[:, 1] += 1.0
    c = c.astype(np.float32)
    w = (1.25, 2.0, 0.75, 0.875)
    x = rng.normal(size=(B, P)).astype(np.float32)
    np.savez(tmp_path / "in.npz", shape=np.array(shape), h=np.array(h), w=np.array(w), c=c, x=x)
    env = dict(os.environ, **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", _APPLY_SCRIPT, str(tmp_path / "in.npz"),
                    str(tmp_path / "y.npy"), str(tmp_path / "v.npy")], check=True, env=env, cwd=root)
    y = np.load(tmp_path / "y.npy")
    v = np.load(tmp_path / "v.npy")
    assert (int(v[0]), int(v[1])) == kinds, f"kernel variants {v.tolist()} != expected {kinds}"
    pr = Problem(shape, h, *w)
    for i in sorted({0, 1, B - 1}):  # first, second and last PDE of the launch
        ref = _sparse_schur_apply(pr, c[i].astype(np.float64), x[i].astype(np.float64))
        assert np.linalg.norm(y[i] - ref) <= 1e-4 * np.linalg.norm(ref)


@pytest.mark.parametrize("shape,h,B", [((16, 18, 20), (0.05, 0.06, 0.07), 2), ((20, 24), (0.05, 0.04), 2),
                                       ((20, 32, 32), (0.05, 0.03, 0.03), 2),
                                       ((6, 64, 64), (0.01, 1 / 64, 1 / 64), 19),
                                       ((64, 96), (0.05, 0.02), 2)])
def test_vcycle_symmetric_positive(shape, h, B):
    """The V-cycle is a fixed SPD linear map (needed by PCG): <Ma, b> = <a, Mb>, <Ma, a> > 0.
    (20,32,32) and (6,64,64) run the level-0 V-cycle applies through the bf16-coefficient
    t-blocked kernels <32,32> / <64,64> the bench uses (asserted); the t-marching variant's
    V-cycle applies are checked against these in tools/march_check.py and by
    test_march_vcycle_symmetric_positive."""
    from paper_2502_18377_b200 import mpde
    rng = np.random.default_rng(6)
    D = len(shape)
    M, P = 1 + 2 * D, int(np.prod(shape))
    c = rng.normal(0.0, 0.5, (B, M, P))
    c[:, 1] += 1.0
    s = mpde.Solver(shape, h, torch.from_numpy(c.astype(np.float32)).cuda())
    if P > 16384 and D == 3:
        v = mpde.mpde_hierarchy_query(s.h_, 0, 5, None)
        want = 4  # t-blocked <n,n> (the t-slab and t-marching applies are opt-in)
        assert v[2] == want and v[3] == 1, v  # reading bf16 coefficients
    a = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
    ma, mb = torch.empty_like(a), torch.empty_like(b)
    mpde.mpde_apply_precond(s.h_, a, ma)
    mpde.mpde_apply_precond(s.h_, b, mb)
    torch.cuda.synchronize()
    for i in range(B):
        l = float((ma[i].double() * b[i].double()).sum())
        r = float((a[i].double() * mb[i].double()).sum())
        assert abs(l - r) <= 1e-4 * (abs(l) + abs(r))
        assert float((ma[i].double() * a[i].double()).sum()) > 0
    s.close()


_PRECOND_SCRIPT = r"""
import sys, numpy as np, torch
from paper_2502_18377_b200 import mpde
rng = np.random.default_rng(6)
shape, B = (16, 18, 20), 2
P = int(np.prod(shape))
c = rng.normal(0.0, 0.5, (B, 7, P)); c[:, 1] += 1.0
s = mpde.Solver(shape, (0.05, 0.06, 0.07), torch.from_numpy(c.astype(np.float32)).cuda())
a = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
b = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
ma, mb = torch.empty_like(a), torch.empty_like(b)
mpde.mpde_apply_precond(s.h_, a, ma); mpde.mpde_apply_precond(s.h_, b, mb)
torch.cuda.synchronize()
for i in range(B):
    l = float((ma[i].double() * b[i].double()).sum()); r = float((a[i].double() * mb[i].double()).sum())
    assert abs(l - r) <= 1e-4 * (abs(l) + abs(r)), (l, r)
    assert float((ma[i].double() * a[i].double()).sum()) > 0
print("ok")
"""


def test_wcycle_symmetric_positive():
    """The W-cycle option (MPDE_WCYCLE=1: gamma = 2 below level 0) is still a fixed SPD map."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _PRECOND_SCRIPT], check=True, cwd=root,
                         env=dict(os.environ, MPDE_WCYCLE="1"), capture_output=True, text=True)
    assert "ok" in out.stdout


_MARCH_PRECOND = r"""
import sys, numpy as np, torch
from paper_2502_18377_b200 import mpde
rng = np.random.default_rng(6)
shape, B = (6, 64, 64), 19
P = int(np.prod(shape))
c = rng.normal(0.0, 0.5, (B, 7, P)); c[:, 1] += 1.0
s = mpde.Solver(shape, (0.01, 1 / 64, 1 / 64), torch.from_numpy(c.astype(np.float32)).cuda())
v = mpde.mpde_hierarchy_query(s.h_, 0, 5, None)
assert v[2] == 9 and v[3] == 1, v
a = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
b = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
ma, mb = torch.empty_like(a), torch.empty_like(b)
mpde.mpde_apply_precond(s.h_, a, ma); mpde.mpde_apply_precond(s.h_, b, mb)
torch.cuda.synchronize()
for i in range(B):
    l = float((ma[i].double() * b[i].double()).sum()); r = float((a[i].double() * mb[i].double()).sum())
    assert abs(l - r) <= 1e-4 * (abs(l) + abs(r)), (l, r)
    assert float((ma[i].double() * a[i].double()).sum()) > 0
print("ok")
"""


def test_march_vcycle_symmetric_positive():
    """The V-cycle with the t-marching S apply (MPDE_MARCH=1, bf16 coefficients on level 0,
    152 CTAs per launch) is still a fixed SPD map."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _MARCH_PRECOND], check=True, cwd=root,
                         env=dict(os.environ, MPDE_MARCH="1"), capture_output=True, text=True)
    assert "ok" in out.stdout
