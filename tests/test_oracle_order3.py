"""Oracle pins for third-order derivative variables ("partial
derivatives of arbitrary order"; the u_xxx term of the KdV half of BASELINE configs[1]).
Reading O3: Problem(order=(..)) keeps derivatives up to order 3 along a dim as
variables; their derivative rows use 5-point rules (central (-1, 2, 0, -2, 1)/2, one-sided
(-5, 18, -24, 14, -3)/2, mirrored with sign (-1)^3 at the far edge) with coefficient h^3 on
the variable (literal Eq. 5, reading Q5), and that dim's Taylor rows run to third order
(+- h^3/6 u_ddd).

Pinned by: the stencils on quartics, row counts, manufactured solutions cubic in the
third-order dim (exact), and central finite differences of the field and step gradients.  The
GPU path is not built for order 3."""
import numpy as np
import pytest

from oracle import Problem, assemble, counts, solve_backward, solve_forward, step_gradient
from oracle.neurlp import fd_stencil


@pytest.mark.parametrize("i", [0, 1, 2, 5, 7, 8, 9])
def test_third_derivative_stencils_exact_on_quartics(i):
    n = 10
    f = lambda x: 0.3 * x ** 4 - x ** 3 + 2 * x ** 2 - x + 1
    f3 = lambda x: 7.2 * x - 6.0
    offs, w = fd_stencil(3, i, n)
    assert abs(sum(wj * f(i + o) for o, wj in zip(offs, w)) - f3(i)) <= 1e-10


@pytest.mark.parametrize("shape,order", [((7, 9), (2, 3)), ((6, 7, 8), (2, 3, 2)), ((6, 7, 8), (2, 3, 3))])
def test_row_counts_order3(shape, order):
    pr = Problem(shape, (0.1,) * len(shape), order=order)
    rng = np.random.default_rng(0)
    c = rng.normal(size=(pr.M, pr.P))
    A, _, _ = assemble(pr, c, np.zeros(pr.P), np.zeros(pr.P))
    n_v, n_c = counts(shape, order=order)
    assert pr.M == 1 + sum(order) and A.shape == (n_c, n_v)


def _poly_fields(pr, coefs):
    """u = sum a_(e) prod_d x_d^e_d (e_d <= ord(d)) and its pure derivatives, field order of pr."""
    D = pr.D
    axes = [np.arange(n) * pr.h[d] for d, n in enumerate(pr.shape)]
    X = np.meshgrid(*axes, indexing="ij")

    def deriv(p, x, k):
        if k > p:
            return 0 * x
        fac = 1.0
        for j in range(k):
            fac *= (p - j)
        return fac * x ** (p - k)

    out = np.zeros((pr.M, pr.P))
    for e, a in coefs.items():
        base = [X[d] ** e[d] for d in range(D)]
        out[0] += a * np.prod(base, axis=0).reshape(-1)
        for d in range(D):
            for k in range(1, pr.ord(d) + 1):
                term = [base[e2] if e2 != d else deriv(e[d], X[d], k) for e2 in range(D)]
                out[pr.field(d, k)] += a * np.prod(term, axis=0).reshape(-1)
    return out


@pytest.mark.parametrize("shape,h,order", [((10, 12), (0.1, 0.08), (2, 3)), ((6, 8, 7), (0.1, 0.12, 0.09), (2, 3, 2))])
def test_manufactured_cubic_solution_exact(shape, h, order):
    """P2 for order 3: degree <= 2 in the order-2 dims and <= 3 in the order-3 dims; b := sum c z,
    omega := u: A z_exact = d and the least-squares solution is z_exact."""
    rng = np.random.default_rng(1)
    pr = Problem(shape, h, 1.3, 2.0, 0.7, 0.9, order=order)
    coefs = {e: rng.normal() for e in np.ndindex(*[pr.ord(d) + 1 for d in range(pr.D)])}
    z = _poly_fields(pr, coefs)
    c = rng.normal(size=(pr.M, pr.P))
    c[1] += 1.0
    b = (c * z).sum(axis=0)
    A, d, _ = assemble(pr, c, b, z[0])
    zz = z.reshape(-1)
    assert np.linalg.norm(A @ zz - d) <= 1e-11 * np.linalg.norm(d)
    f = solve_forward(pr, c, b, z[0], method="dense")
    assert np.linalg.norm(f["z"] - zz) <= 1e-8 * np.linalg.norm(zz)


def test_gradients_order3_match_central_differences():
    """P7 with a third-order dim: dl/dc (all 6 fields), dl/db and dl/dh against central
    differences of l = <g, z*>."""
    shape, h = (8, 9), (0.1, 0.2)
    rng = np.random.default_rng(4)
    pr = Problem(shape, h, 1.3, 2.0, 0.7, 0.9, order=(2, 3))
    c = rng.normal(0.0, 0.5, (pr.M, pr.P))
    c[1] += 1.0
    b = rng.normal(size=pr.P)
    om = rng.normal(size=pr.P)
    g = rng.normal(size=pr.n_v)
    f = solve_forward(pr, c, b, om, method="dense")
    bw = solve_backward(pr, f, g, method="dense")
    eps = 1e-6
    for m, p in ((pr.field(1, 3), 17), (0, 30), (pr.field(0, 1), 44)):
        cp, cm = c.copy(), c.copy()
        cp[m, p] += eps
        cm[m, p] -= eps
        fd = (g @ solve_forward(pr, cp, b, om, method="dense")["z"]
              - g @ solve_forward(pr, cm, b, om, method="dense")["z"]) / (2 * eps)
        assert abs(fd - bw["grad_c"][m, p]) <= 1e-6 * np.abs(bw["grad_c"]).max()
    gh = step_gradient(pr, f, bw)
    for d in range(2):
        e = 1e-5 * h[d]
        hp, hm = list(h), list(h)
        hp[d] += e
        hm[d] -= e
        lp = g @ solve_forward(Problem(shape, tuple(hp), 1.3, 2.0, 0.7, 0.9, order=(2, 3)), c, b, om, method="dense")["z"]
        lm = g @ solve_forward(Problem(shape, tuple(hm), 1.3, 2.0, 0.7, 0.9, order=(2, 3)), c, b, om, method="dense")["z"]
        fd = (lp - lm) / (2 * e)
        assert abs(fd - gh[d]) <= 1e-5 * max(abs(fd), abs(gh[d]))
