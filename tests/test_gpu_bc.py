"""GPU parity for the boundary-type extension ("Dirichlet ...,
Neumann ... or mixed types"; reading B1 in DESIGN.md): per-face Dirichlet / Neumann / none
rows through the C ABI (mpde_problem.bc, mpde_solve_fwd_bc / _bwd_bc) against the oracle on
the same inputs -- the normal operator, the condensed operator S, fwd + bwd with every
gradient including dl/domega_n, and manufactured solutions with Neumann data at grid sizes
that run the production kernels on several levels, and the exported duals lambda*."""
import numpy as np
import pytest
import torch

from oracle import Problem, assemble, solve_backward, solve_forward
from oracle.neurlp import face_points, field_index

pytestmark = pytest.mark.gpu

E_Z, E_G = 1e-4, 1e-3
W = (1.25, 2.0, 0.75, 0.875)
MIXED2 = (("D", "-"), ("N", "N"))
MIXED3 = (("D", "-"), ("N", "D"), ("D", "N"))
ALLN3 = (("D", "N"), ("N", "N"), ("N", "N"))


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


@pytest.mark.parametrize("shape,h,bc", [((12, 14), (0.1, 0.07), MIXED2), ((8, 9, 10), (0.1, 0.07, 0.05), MIXED3)])
def test_normal_apply_with_boundary_types(shape, h, bc):
    from paper_2502_18377_b200 import mpde
    B = 2
    c, _, _, _, z = _problem(shape, B, 1)
    prob = mpde.make_problem(shape, h, B, *W, bc=bc)
    q = torch.empty_like(_dev(z))
    mpde.mpde_apply_normal(prob, _dev(c), _dev(z), q)
    q = q.cpu().numpy()
    pr = Problem(shape, h, *W, bc=bc)
    for i in range(B):
        A, _, _ = assemble(pr, c[i], np.zeros(pr.P), np.zeros(pr.P))
        assert _rel(q[i], A.T @ (A @ z[i].reshape(-1).astype(np.float64))) <= 1e-6


@pytest.mark.parametrize("shape,h,bc", [((12, 10), (0.1, 0.05), MIXED2), ((7, 8, 9), (0.1, 0.2, 0.15), MIXED3),
                                        ((8, 8, 8), (0.1, 0.1, 0.1), ALLN3)])
def test_schur_apply_with_boundary_types(shape, h, bc):
    from paper_2502_18377_b200 import mpde
    B = 2
    c, _, _, _, _ = _problem(shape, B, 2)
    s = mpde.Solver(shape, h, _dev(c), opts=mpde.mpde_default_options(levels_max=1), weights=W, bc=bc)
    x = np.random.default_rng(3).normal(size=(B, s.P)).astype(np.float32)
    y = torch.empty((B, s.P), dtype=torch.float32, device="cuda")
    mpde.mpde_apply_schur(s.h_, 0, _dev(x), y)
    dinv = torch.empty_like(y)
    mpde.mpde_hierarchy_query(s.h_, 0, 1, dinv)
    torch.cuda.synchronize()
    pr = Problem(shape, h, *W, bc=bc)
    for i in range(B):
        A, _, _ = assemble(pr, c[i].astype(np.float64), np.zeros(pr.P), np.zeros(pr.P))
        N = (A.T @ A).toarray()
        P = pr.P
        S = N[:P, :P] - N[:P, P:] @ np.linalg.solve(N[P:, P:], N[P:, :P])
        assert _rel(y[i].cpu().numpy(), S @ x[i]) <= 1e-4
        assert _rel(1.0 / dinv[i].cpu().numpy(), np.diag(S)) <= 1e-5
    s.close()


@pytest.mark.parametrize("shape,h,bc", [((16, 16), (1 / 15, 1 / 15), MIXED2), ((20, 26), (0.05, 0.04), MIXED2),
                                        ((10, 12, 14), (0.1, 0.08, 0.07), MIXED3),
                                        ((10, 12, 14), (0.1, 0.08, 0.07), ALLN3)])
def test_fwd_bwd_with_boundary_types(shape, h, bc):
    """z*, grad_c, grad_b, grad_omega, grad_omega_n, d_z against the oracle (dense / LU)."""
    from paper_2502_18377_b200 import mpde
    B = 2
    c, b, om, omn, g = _problem(shape, B, 4)
    s = mpde.Solver(shape, h, _dev(c), weights=W, bc=bc)
    z = s.forward(_dev(b), _dev(om), omega_n=_dev(omn))
    torch.cuda.synchronize()
    sf = s.stats_list()
    gc, gb, gw, dz, gwn = s.backward(_dev(b), z, _dev(g), want_dz=True, want_grad_omega_n=True)
    torch.cuda.synchronize()
    s.close()
    pr = Problem(shape, h, *W, bc=bc)
    meth = "dense" if pr.n_v <= 5000 else "lu"
    D = len(shape)
    for i in range(B):
        assert sf[i]["status"] == "converged", sf[i]
        f = solve_forward(pr, c[i], b[i], om[i], method=meth, omega_n=omn[i])
        bw = solve_backward(pr, f, g[i].reshape(-1).astype(np.float64), method=meth)
        assert _rel(z[i].cpu().numpy(), f["z"]) <= E_Z
        assert _rel(dz[i].cpu().numpy(), bw["dz"]) <= E_G
        for k, v in (("grad_c", gc), ("grad_b", gb), ("grad_omega", gw)):
            assert _rel(v[i].cpu().numpy(), bw[k]) <= E_G, k
        assert _rel(gwn[i].cpu().numpy(), bw["grad_omega_n"]) <= E_G
        # zero off the Neumann faces of each dim
        on = np.zeros((D, pr.P), bool)
        for d in range(D):
            for sd in (0, 1):
                if bc[d][sd] == "N":
                    on[d][face_points(shape, d, sd)] = True
        assert np.all(gwn[i].cpu().numpy()[~on] == 0.0)


def _quad_fields(shape, h, rng):
    D = len(shape)
    axes = [np.arange(n) * h[d] for d, n in enumerate(shape)]
    X = np.meshgrid(*axes, indexing="ij")
    L = [(n - 1) * h[d] for d, n in enumerate(shape)]
    a = rng.normal(size=(3,) * D)
    fields = []
    for which in [None] + [(d, k) for d in range(D) for k in (1, 2)]:
        out = np.zeros(shape)
        for e in np.ndindex(*(3,) * D):
            term = np.full(shape, a[e])
            for d in range(D):
                s = X[d] / L[d]
                p = e[d]
                if which is not None and which[0] == d:
                    f = (p * s ** (p - 1) / L[d] if p >= 1 else 0 * s) if which[1] == 1 else \
                        (p * (p - 1) * s ** (p - 2) / L[d] ** 2 if p >= 2 else 0 * s)
                else:
                    f = s ** p
                term = term * f
            out = out + term
        fields.append(out.reshape(-1))
    return np.stack(fields)


@pytest.mark.parametrize("shape,h,bc,B", [((32, 64, 64), (0.01, 1 / 64, 1 / 64), MIXED3, 19),
                                          ((101, 256), (0.1, 1 / 16), MIXED2, 2)])
def test_manufactured_neumann_full_size(shape, h, bc, B):
    """P2 with Neumann data at C4 / C2 grid sizes (multigrid on every level, the production
    level-0 kernels <64,64> / 2D v4): u per-dim quadratic, omega = u,
    omega_n[d] = du/dx_d, so z* = (u, du) exactly.  Tolerance: the north_star 1e-4 (the
    fp32 rounding of the inputs bounds the floor)."""
    import synth
    from paper_2502_18377_b200 import mpde
    rng = np.random.default_rng(9)
    cfg_name = "C4" if len(shape) == 3 else "C2"
    c = synth.make_batch(cfg_name, B)["c"]
    D, P = len(shape), int(np.prod(shape))
    zs = np.stack([_quad_fields(shape, h, rng) for _ in range(B)])
    b = (c.astype(np.float64) * zs).sum(axis=1).astype(np.float32)
    om = zs[:, 0].astype(np.float32)
    omn = np.stack([zs[:, field_index(d, 1)] for d in range(D)], axis=1).astype(np.float32)
    s = mpde.Solver(shape, h, _dev(c), bc=bc)
    z = s.forward(_dev(b), _dev(om), omega_n=_dev(omn))
    torch.cuda.synchronize()
    st = s.stats_list()
    s.close()
    for i in range(B):
        assert st[i]["status"] == "converged", st[i]
        assert _rel(z[i].cpu().numpy(), zs[i]) <= E_Z


def _oracle_lambda_structured(pr, lam, info):
    """Map the oracle's dual vector (rows in assemble's order) onto the structured layout of
    mpde_solve_fwd_bc's lambda_opt: [2 + 5D][P] (mpde.h)."""
    shape, D, P = tuple(pr.shape), pr.D, pr.P
    out = np.zeros((2 + 5 * D, P))
    out[0] = lam[info["eq_rows"]]
    out[1][info["bnd_points"]] = lam[info["bnd_rows"]]
    r0 = P + info["bnd_rows"].size
    for d, side, fp, rr in info["neu"]:
        out[2 + d][fp] = lam[rr]
        r0 += rr.size
    for d in range(D):
        for k in (1, 2):
            out[2 + D + 2 * d + (k - 1)] = lam[r0:r0 + P]
            r0 += P
    idx = np.unravel_index(np.arange(P), shape)
    for d in range(D):
        for j, sel in enumerate((idx[d] <= shape[d] - 2, idx[d] >= 1)):
            pts = np.flatnonzero(sel)
            out[2 + 3 * D + 2 * d + j][pts] = lam[r0:r0 + pts.size]
            r0 += pts.size
    assert r0 == lam.size
    return out


@pytest.mark.parametrize("shape,h,bc", [((16, 16), (1 / 15, 1 / 15), None), ((12, 14), (0.1, 0.07), MIXED2),
                                        ((8, 9, 10), (0.1, 0.07, 0.05), MIXED3)])
def test_duals_match_oracle(shape, h, bc):
    """lambda* = d - A z* (Eq. 10 first block row) exported by the forward, against
    the oracle's lambda* mapped onto the structured layout; judged in absolute terms relative
    to ||d|| (lambda* -> 0 on consistent systems)."""
    from paper_2502_18377_b200 import mpde
    B = 2
    c, b, om, omn, _ = _problem(shape, B, 6)
    s = mpde.Solver(shape, h, _dev(c), weights=W, bc=bc)
    z, lam = s.forward(_dev(b), _dev(om), omega_n=_dev(omn), want_lambda=True)
    torch.cuda.synchronize()
    s.close()
    pr = Problem(shape, h, *W, bc=bc)
    for i in range(B):
        f = solve_forward(pr, c[i], b[i], om[i], method="dense" if pr.n_v <= 5000 else "lu",
                          omega_n=omn[i] if bc is not None else None)
        ref = _oracle_lambda_structured(pr, f["lam"], f["info"])
        got = lam[i].cpu().numpy().astype(np.float64)
        assert np.linalg.norm(got - ref) <= 1e-4 * np.linalg.norm(f["d"]), \
            (np.linalg.norm(got - ref), np.linalg.norm(f["d"]))


@pytest.mark.parametrize("shape,h,bc", [((16, 16), (1 / 15, 1 / 15), None), ((12, 14), (0.1, 0.07), MIXED2),
                                        ((8, 9, 10), (0.1, 0.07, 0.05), MIXED3)])
def test_step_gradient_matches_oracle(shape, h, bc):
    """dl/dh_d (differentiable step sizes) through mpde_step_gradient against the
    oracle's P:240 contraction with dA/dh_d (itself pinned by central differences,
    tests/test_oracle_bc.py)."""
    from oracle import step_gradient
    from paper_2502_18377_b200 import mpde
    B = 2
    c, b, om, omn, g = _problem(shape, B, 8)
    s = mpde.Solver(shape, h, _dev(c), weights=W, bc=bc, opts=mpde.mpde_default_options(grad_steps=1))
    bd = _dev(b)
    z = s.forward(bd, _dev(om), omega_n=_dev(omn))
    s.backward(bd, z, _dev(g))
    gh = s.step_gradient(z)
    torch.cuda.synchronize()
    s.close()
    pr = Problem(shape, h, *W, bc=bc)
    meth = "dense" if pr.n_v <= 5000 else "lu"
    for i in range(B):
        f = solve_forward(pr, c[i], b[i], om[i], method=meth, omega_n=omn[i] if bc is not None else None)
        bw = solve_backward(pr, f, g[i].reshape(-1).astype(np.float64), method=meth)
        ref = step_gradient(pr, f, bw)
        assert _rel(gh[i].cpu().numpy(), ref) <= E_G, (gh[i].cpu().numpy(), ref)


def test_step_gradient_requires_option():
    from paper_2502_18377_b200 import mpde
    c, b, om, _, g = _problem((12, 14), 1, 9)
    s = mpde.Solver((12, 14), (0.1, 0.07), _dev(c))
    z = s.forward(_dev(b), _dev(om))
    s.backward(_dev(b), z, _dev(g))
    with pytest.raises(RuntimeError):
        s.step_gradient(z)
    s.close()
