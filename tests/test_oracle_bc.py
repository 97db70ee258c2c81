"""Oracle pins for the boundary-type extension ("Dirichlet
(i.e., boundary conditions on u), Neumann (i.e., boundary conditions on partial derivatives)
or mixed types").  Reading B1: per face (dim d, low / high side) a type 'D'
(u_phi = omega), 'N' (the first derivative along d = omega_n[d]) or '-' (no row); every point
on a Dirichlet face gets one Dirichlet row, every point of a Neumann face one Neumann row.

Pinned by: row counts, manufactured per-dim-quadratic solutions (exact: the Neumann data is the
analytic derivative), central finite differences of the Neumann-data gradient, full column rank,
and the analytic Neumann heat solution u = exp(-nu pi^2 t) cos(pi x) within discretisation error."""
import numpy as np
import pytest

from oracle import Problem, assemble, counts, solve_backward, solve_forward
from oracle.neurlp import boundary_mask, face_points, field_index

MIXED2 = (("D", "-"), ("N", "N"))                 # initial value, no final condition, Neumann in x
MIXED3 = (("D", "-"), ("N", "D"), ("D", "N"))


def _rand_c(shape, rng):
    D = len(shape)
    M, P = 1 + 2 * D, int(np.prod(shape))
    c = rng.normal(0.0, 0.5, (M, P))
    c[1] += 1.0
    return c


def _quad_u(shape, h, rng):
    """u = sum_e a_e prod_d x_d^e_d (degree <= 2 per dim) and its pure derivatives [M][P]."""
    D = len(shape)
    axes = [np.arange(n) * h[d] for d, n in enumerate(shape)]
    X = np.meshgrid(*axes, indexing="ij")
    a = rng.normal(size=(3,) * D)
    fields = []
    for which in [None] + [(d, k) for d in range(D) for k in (1, 2)]:
        out = np.zeros(shape)
        for e in np.ndindex(*(3,) * D):
            term = np.full(shape, a[e])
            for d in range(D):
                x, p = X[d], e[d]
                if which is not None and which[0] == d:
                    if which[1] == 1:
                        f = p * x ** (p - 1) if p >= 1 else 0 * x
                    else:
                        f = p * (p - 1) * x ** (p - 2) if p >= 2 else 0 * x
                else:
                    f = x ** p
                term = term * f
            out = out + term
        fields.append(out.reshape(-1))
    return np.stack(fields)


@pytest.mark.parametrize("shape,bc", [((7, 8), MIXED2), ((6, 7, 8), MIXED3),
                                      ((6, 7), (("N", "N"), ("N", "N")))])
def test_row_counts(shape, bc):
    pr = Problem(shape, (0.1,) * len(shape), bc=bc)
    rng = np.random.default_rng(0)
    A, d, info = assemble(pr, _rand_c(shape, rng), np.zeros(pr.P), np.zeros(pr.P))
    n_v, n_c = counts(shape, bc)
    assert A.shape == (n_c, n_v)
    nd = int(boundary_mask(shape, bc, "D").sum())
    nn = sum(face_points(shape, dd, s).size for dd in range(len(shape)) for s in (0, 1)
             if bc[dd][s] == "N")
    P = pr.P
    smooth = sum(2 * (n - 1) * (P // n) for n in shape)
    assert n_c == P + nd + nn + 2 * len(shape) * P + smooth
    assert len(info["neu"]) == sum(bc[dd][s] == "N" for dd in range(len(shape)) for s in (0, 1))


@pytest.mark.parametrize("shape,h,bc", [((8, 9), (0.1, 0.12), MIXED2),
                                        ((6, 7, 8), (0.1, 0.2, 0.15), MIXED3)])
def test_manufactured_solution_exact(shape, h, bc):
    """P2 with Neumann data omega_n = du/dx_d: A z_exact = d exactly and the least-squares
    solution is z_exact (the 5-point stencils and Taylor rows are exact on quadratics)."""
    rng = np.random.default_rng(1)
    pr = Problem(shape, h, 1.3, 2.0, 0.7, 0.9, bc=bc)
    c = _rand_c(shape, rng)
    z = _quad_u(shape, h, rng)
    D = len(shape)
    b = (c * z).sum(axis=0)
    om = z[0].copy()
    om_n = np.stack([z[field_index(d, 1)] for d in range(D)])
    A, dvec, _ = assemble(pr, c, b, om, om_n)
    zz = z.reshape(-1)
    assert np.linalg.norm(A @ zz - dvec) <= 1e-11 * np.linalg.norm(dvec)
    f = solve_forward(pr, c, b, om, method="dense", omega_n=om_n)
    assert np.linalg.norm(f["z"] - zz) <= 1e-9 * np.linalg.norm(zz)


def test_full_column_rank_mixed():
    """Generic c with the mixed types: A has full column rank (unique z*)."""
    rng = np.random.default_rng(2)
    for shape, bc in (((7, 8), MIXED2), ((6, 6, 7), MIXED3), ((6, 7), (("N", "N"), ("N", "N")))):
        pr = Problem(shape, (0.1,) * len(shape), bc=bc)
        A, _, _ = assemble(pr, _rand_c(shape, rng), np.zeros(pr.P), np.zeros(pr.P))
        s = np.linalg.svd(A.toarray(), compute_uv=False)
        assert s[-1] > 1e-8 * s[0]


def test_neumann_gradient_matches_central_differences():
    """P7 for the Neumann data: dl/domega_n[d][p] of l = <g, z*> matches central finite
    differences; it vanishes off the Neumann faces of dim d."""
    shape, h, bc = (8, 9), (0.1, 0.2), MIXED2
    rng = np.random.default_rng(3)
    pr = Problem(shape, h, 1.3, 2.0, 0.7, 0.9, bc=bc)
    c = _rand_c(shape, rng)
    b = rng.normal(size=pr.P)
    om = rng.normal(size=pr.P)
    om_n = rng.normal(size=(2, pr.P))
    g = rng.normal(size=pr.n_v)
    f = solve_forward(pr, c, b, om, method="dense", omega_n=om_n)
    bw = solve_backward(pr, f, g, method="dense")
    gn = bw["grad_omega_n"]
    on_face = np.zeros((2, pr.P), bool)
    on_face[1][face_points(shape, 1, 0)] = True
    on_face[1][face_points(shape, 1, 1)] = True
    assert np.all(gn[~on_face] == 0.0)
    eps = 1e-6
    scale = np.abs(gn).max()
    for d, p in [(1, int(face_points(shape, 1, 0)[3])), (1, int(face_points(shape, 1, 1)[5]))]:
        lp, lm = [], []
        for sgn, acc in ((1, lp), (-1, lm)):
            o2 = om_n.copy()
            o2[d][p] += sgn * eps
            acc.append(g @ solve_forward(pr, c, b, om, method="dense", omega_n=o2)["z"])
        fd = (lp[0] - lm[0]) / (2 * eps)
        assert abs(fd - gn[d][p]) <= 1e-6 * scale
    # the other gradients still match their finite differences with Neumann rows present
    p = 20
    lp = g @ solve_forward(pr, c, b + eps * (np.arange(pr.P) == p), om, method="dense", omega_n=om_n)["z"]
    lm = g @ solve_forward(pr, c, b - eps * (np.arange(pr.P) == p), om, method="dense", omega_n=om_n)["z"]
    assert abs((lp - lm) / (2 * eps) - bw["grad_b"][p]) <= 1e-6 * np.abs(bw["grad_b"]).max()


def test_neumann_heat_converges_to_analytic():
    """u_t = nu u_xx on [0,1]^2 with u(0,x) = cos(pi x) (Dirichlet at t = 0), u_x = 0 on both x
    faces (Neumann) and no final-time row: u = exp(-nu pi^2 t) cos(pi x).  The converged
    least-squares solution approaches it at second order (measured error ratios 3.2 and 4.1
    for 16 -> 32 -> 64; the same problem with Dirichlet x faces and no final-time row gives
    4.8 / 4.2, so the order comes from the open final face, not from the Neumann rows).  The
    all-Dirichlet heat case of pin P8 converges faster (order 4-5)."""
    nu = 0.1
    errs = []
    for n in (16, 32, 64):
        h = 1.0 / (n - 1)
        shape = (n, n)
        pr = Problem(shape, (h, h), bc=(("D", "-"), ("N", "N")))
        t, x = np.meshgrid(np.arange(n) * h, np.arange(n) * h, indexing="ij")
        u = np.exp(-nu * np.pi ** 2 * t) * np.cos(np.pi * x)
        c = np.zeros((5, pr.P))
        c[1] = 1.0
        c[4] = -nu
        f = solve_forward(pr, c, np.zeros(pr.P), u.reshape(-1), method="lu",
                          omega_n=np.zeros((2, pr.P)))
        up = f["z"][:pr.P]
        errs.append(np.linalg.norm(up - u.reshape(-1)) / np.linalg.norm(u))
    assert errs[0] < 1e-3 and errs[1] < errs[0] / 3 and errs[2] < errs[1] / 3.5, errs


@pytest.mark.parametrize("shape,h,bc", [((8, 9), (0.1, 0.2), None), ((8, 9), (0.1, 0.2), MIXED2),
                                        ((6, 7, 8), (0.1, 0.15, 0.12), MIXED3)])
def test_step_gradient_matches_central_differences(shape, h, bc):
    """dl/dh_d of l = <g, z*> ("step sizes ... are differentiable"): the P:240 matrix
    gradient contracted with dA/dh_d (oracle.step_gradient) against central finite differences
    of the forward solve in h_d; and dA/dh_d itself against the difference quotient of the
    assembly (its entries are polynomials of degree <= 2 in h_d, so the central quotient is
    exact up to rounding)."""
    from oracle import assemble_dh, step_gradient
    rng = np.random.default_rng(11)
    pr = Problem(shape, h, 1.3, 2.0, 0.7, 0.9, bc=bc)
    D = len(shape)
    c = _rand_c(shape, rng)
    b = rng.normal(size=pr.P)
    om = rng.normal(size=pr.P)
    om_n = rng.normal(size=(D, pr.P)) if bc is not None else None
    g = rng.normal(size=pr.n_v)
    meth = "dense" if D == 2 else "lu"  # SuperLU + fp64 refinement: same accuracy, 3D in seconds
    f = solve_forward(pr, c, b, om, method=meth, omega_n=om_n)
    bw = solve_backward(pr, f, g, method=meth)
    gh = step_gradient(pr, f, bw)
    for d in range(D):
        eps = 1e-5 * h[d]
        hp, hm = list(h), list(h)
        hp[d] += eps
        hm[d] -= eps
        prp = Problem(shape, tuple(hp), 1.3, 2.0, 0.7, 0.9, bc=bc)
        prm = Problem(shape, tuple(hm), 1.3, 2.0, 0.7, 0.9, bc=bc)
        Ap, _, _ = assemble(prp, c, b, om, om_n)
        Am, _, _ = assemble(prm, c, b, om, om_n)
        J = assemble_dh(pr, d, f["info"])
        assert abs((Ap - Am) / (2 * eps) - J).max() <= 1e-6 * abs(J).max()
        lp = g @ solve_forward(prp, c, b, om, method=meth, omega_n=om_n)["z"]
        lm = g @ solve_forward(prm, c, b, om, method=meth, omega_n=om_n)["z"]
        fd = (lp - lm) / (2 * eps)
        assert abs(fd - gh[d]) <= 1e-5 * max(abs(fd), abs(gh[d])), (d, fd, gh[d])
