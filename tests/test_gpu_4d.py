"""GPU parity on 4D grids (t + three space dims; P:84-88 define the method for a grid of any
dimension: "D-dimensional grid", the derivative variables and Taylor rows per dim, Eqs. 3-8).
The CUDA path takes ndim 2..4 (mpde.h); this file runs the 4D kernels through the C ABI
against the oracle, which is dimension-generic (tests/test_oracle_4d.py pins it in 4D):
  - the normal operator N = A^T A (several ragged shapes, mixed weights);
  - the condensed operator S on level 0 against the oracle's N blocks (sparse elimination);
  - fwd + bwd with mixed boundary types against the oracle's converged t-slab PCG: z*, d_z,
    grad_c, grad_b, grad_omega, grad_omega_n, the step gradient dl/dh and the duals lambda*;
  - a manufactured solution on a grid whose hierarchy coarsens every axis (4D restriction /
    prolongation and the 4096-point coarsest inverse)."""
import numpy as np
import pytest
import torch
import scipy.sparse.linalg as spla

from oracle import Problem, assemble, solve_backward, solve_forward, step_gradient
from oracle.neurlp import face_points, field_index

pytestmark = pytest.mark.gpu

E_Z, E_G = 1e-4, 1e-3
W = (1.25, 2.0, 0.75, 0.875)  # exactly representable in fp32 (the ABI takes float weights)
MIXED4 = (("D", "-"), ("N", "D"), ("D", "N"), ("N", "N"))


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _problem(shape, B, seed):
    rng = np.random.default_rng(seed)
    D = len(shape)
    M, P = 1 + 2 * D, int(np.prod(shape))
    c = rng.normal(0.0, 0.5, (B, M, P))
    c[:, 1] += 1.0
    f32 = lambda a: a.astype(np.float32)
    return (f32(c), f32(rng.normal(size=(B, P))), f32(rng.normal(size=(B, P))),
            f32(rng.normal(size=(B, D, P))), f32(rng.normal(size=(B, M, P))))


@pytest.mark.parametrize("shape,h,bc", [((6, 7, 6, 8), (0.1, 0.12, 0.09, 0.11), None),
                                        ((7, 6, 9, 6), (0.2, 0.1, 0.15, 0.3), MIXED4)])
def test_normal_apply_4d(shape, h, bc):
    """N p = A^T (A p) against the oracle's explicit CSR (fp64)."""
    from paper_2502_18377_b200 import mpde
    B = 2
    c, _, _, _, _ = _problem(shape, B, 11)
    rng = np.random.default_rng(12)
    z = rng.normal(size=c.shape).astype(np.float32)
    prob = mpde.make_problem(shape, h, B, *W, bc=bc)
    q = torch.empty_like(_dev(z))
    mpde.mpde_apply_normal(prob, _dev(c), _dev(z), q)
    q = q.cpu().numpy().astype(np.float64)
    pr = Problem(shape, h, *W, bc=bc)
    for i in range(B):
        A, _, _ = assemble(pr, c[i], np.zeros(pr.P), np.zeros(pr.P))
        ref = A.T @ (A @ z[i].reshape(-1).astype(np.float64))
        assert _rel(q[i], ref) <= 1e-6


@pytest.mark.parametrize("shape,h,bc", [((6, 7, 6, 8), (0.1, 0.12, 0.09, 0.11), None),
                                        ((7, 6, 9, 6), (0.2, 0.1, 0.15, 0.3), MIXED4)])
def test_schur_apply_4d(shape, h, bc):
    """S x = (N_pp - N_pd N_dd^-1 N_dp) x (block elimination of the derivative variables) against
    the oracle's N, the N_dd solve by SuperLU (N_dd is block diagonal over the points)."""
    from paper_2502_18377_b200 import mpde
    B = 2
    c, _, _, _, _ = _problem(shape, B, 21)
    s = mpde.Solver(shape, h, _dev(c), opts=mpde.mpde_default_options(levels_max=1), weights=W, bc=bc)
    rng = np.random.default_rng(22)
    x = rng.normal(size=(B, s.P)).astype(np.float32)
    y = torch.empty((B, s.P), dtype=torch.float32, device="cuda")
    mpde.mpde_apply_schur(s.h_, 0, _dev(x), y)
    torch.cuda.synchronize()
    s.close()
    pr = Problem(shape, h, *W, bc=bc)
    P = pr.P
    for i in range(B):
        A, _, _ = assemble(pr, c[i].astype(np.float64), np.zeros(P), np.zeros(P))
        N = (A.T @ A).tocsc()
        Npp, Npd, Ndd = N[:P, :P], N[:P, P:], N[P:, P:]
        xi = x[i].astype(np.float64)
        ref = Npp @ xi - Npd @ spla.splu(Ndd.tocsc()).solve(Npd.T @ xi)
        assert _rel(y[i].cpu().numpy(), ref) <= 1e-4


@pytest.fixture(scope="module")
def run4d():
    """One 4D batch (2 levels: the t axis halves 12 -> 6) solved on the GPU with every export,
    and PDE 0 by the oracle (t-slab PCG, converged to a true normal residual <= 1e-10)."""
    from paper_2502_18377_b200 import mpde
    shape, h, bc = (12, 6, 6, 6), (0.1, 0.12, 0.09, 0.11), MIXED4
    B = 2
    c, b, om, omn, g = _problem(shape, B, 4)
    s = mpde.Solver(shape, h, _dev(c), weights=W, bc=bc, opts=mpde.mpde_default_options(grad_steps=1))
    levels = [mpde.mpde_hierarchy_query(s.h_, l, 6, None) for l in range(2)]
    bd = _dev(b)
    z, lam = s.forward(bd, _dev(om), omega_n=_dev(omn), want_lambda=True)
    torch.cuda.synchronize()
    sf = s.stats_list()
    gc, gb, gw, dz, gwn = s.backward(bd, z, _dev(g), want_dz=True, want_grad_omega_n=True)
    gh = s.step_gradient(z)
    torch.cuda.synchronize()
    sb = s.stats_list()
    s.close()
    pr = Problem(shape, h, *W, bc=bc)
    f = solve_forward(pr, c[0], b[0], om[0], method="slab", omega_n=omn[0])
    bw = solve_backward(pr, f, g[0].reshape(-1).astype(np.float64), method="slab")
    gpu = {k: v[0].cpu().numpy().astype(np.float64) for k, v in
           dict(z=z, lam=lam, grad_c=gc, grad_b=gb, grad_omega=gw, dz=dz, gwn=gwn, gh=gh).items()}
    return dict(shape=shape, bc=bc, pr=pr, f=f, bw=bw, gpu=gpu, sf=sf, sb=sb, levels=levels)


def test_fwd_bwd_4d_matches_oracle(run4d):
    r = run4d
    g, f, bw = r["gpu"], r["f"], r["bw"]
    assert r["levels"] == [[12, 6, 6, 6, 2], [6, 6, 6, 6, 2]]
    assert all(s["status"] == "converged" for s in r["sf"] + r["sb"]), (r["sf"], r["sb"])
    assert _rel(g["z"], f["z"]) <= E_Z
    assert _rel(g["dz"], bw["dz"]) <= E_G
    for k in ("grad_c", "grad_b", "grad_omega"):
        assert _rel(g[k], bw[k]) <= E_G, k
    assert _rel(g["gwn"], bw["grad_omega_n"]) <= E_G
    pr, shape, bc = r["pr"], r["shape"], r["bc"]
    on = np.zeros((4, pr.P), bool)
    for d in range(4):
        for sd in (0, 1):
            if bc[d][sd] == "N":
                on[d][face_points(shape, d, sd)] = True
    assert np.all(g["gwn"][~on] == 0.0)


def test_step_gradient_and_duals_4d(run4d):
    """dl/dh_d (four step sizes) and lambda* = d - A z* in the structured [2 + 5D][P] layout."""
    from test_gpu_bc import _oracle_lambda_structured
    r = run4d
    pr, f, bw, g = r["pr"], r["f"], r["bw"], r["gpu"]
    assert _rel(g["gh"], step_gradient(pr, f, bw)) <= E_G
    ref = _oracle_lambda_structured(pr, f["lam"], f["info"])
    assert np.linalg.norm(g["lam"] - ref) <= 1e-4 * np.linalg.norm(f["d"])


def _quad_fields4(shape, h, rng):
    """u = sum_e a_e prod_d s_d^e_d (degree <= 2 per dim, s_d = x_d / L_d) and its pure
    derivatives in field order (phi, then (d, 1), (d, 2) per dim)."""
    D = len(shape)
    L = [(n - 1) * h[d] for d, n in enumerate(shape)]
    s = [np.arange(n) * h[d] / L[d] for d, n in enumerate(shape)]
    a = rng.normal(size=(3,) * D)
    tab = []  # per dim: [k][e] -> values along the axis
    for d in range(D):
        v = [np.ones_like(s[d]), s[d], s[d] ** 2]
        d1 = [0 * s[d], np.ones_like(s[d]) / L[d], 2 * s[d] / L[d]]
        d2 = [0 * s[d], 0 * s[d], np.full_like(s[d], 2 / L[d] ** 2)]
        tab.append((v, d1, d2))
    out = []
    for which in [None] + [(d, k) for d in range(D) for k in (1, 2)]:
        f = np.zeros(shape)
        for e in np.ndindex(*(3,) * D):
            t = a[e]
            for d in range(D):
                k = which[1] if which is not None and which[0] == d else 0
                sh = [1] * D
                sh[d] = -1
                t = t * tab[d][k][e[d]].reshape(sh)
            f = f + t
        out.append(f.reshape(-1))
    return np.stack(out)


@pytest.mark.parametrize("bc", [None, MIXED4])
def test_manufactured_4d_multilevel(bc):
    """P2 in 4D on a grid whose hierarchy coarsens every axis ((12,16,16,20) -> (6,8,8,10), a
    3840-point coarsest level): z* = (u, du) exactly for u per-dim quadratic with omega = u and
    omega_n[d] = du/dx_d; recovered within the north_star 1e-4."""
    from paper_2502_18377_b200 import mpde
    shape, h, B = (12, 16, 16, 20), (0.05, 1 / 15, 1 / 15, 1 / 19), 2
    rng = np.random.default_rng(31)
    D, P = 4, int(np.prod(shape))
    c = rng.normal(0.0, 0.3, (B, 1 + 2 * D, P))
    c[:, 1] += 1.0
    c = c.astype(np.float32)
    zs = np.stack([_quad_fields4(shape, h, rng) for _ in range(B)])
    b = (c.astype(np.float64) * zs).sum(axis=1).astype(np.float32)
    om = zs[:, 0].astype(np.float32)
    omn = np.stack([zs[:, field_index(d, 1)] for d in range(D)], axis=1).astype(np.float32)
    s = mpde.Solver(shape, h, _dev(c), bc=bc)
    assert mpde.mpde_hierarchy_query(s.h_, 0, 6, None) == [12, 16, 16, 20, 2]
    assert mpde.mpde_hierarchy_query(s.h_, 1, 6, None) == [6, 8, 8, 10, 2]
    z = s.forward(_dev(b), _dev(om), omega_n=_dev(omn))
    torch.cuda.synchronize()
    st = s.stats_list()
    s.close()
    for i in range(B):
        assert st[i]["status"] == "converged", st[i]
        assert _rel(z[i].cpu().numpy(), zs[i]) <= E_Z
