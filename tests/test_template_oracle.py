"""Pins of the polynomial-template oracle (oracle/template.py).

Each test checks the oracle against something other than itself: the paper's printed
expressions, the monomial count C(F+G, G), a closed-form polynomial, and
central finite differences of the full least-squares solve (P:240 chained through the
template)."""
from math import comb

import numpy as np
import pytest

from oracle import Problem, boundary_mask, solve_backward, solve_forward
from oracle.template import features, monomials, template_coeff, template_grad


@pytest.mark.parametrize("F,G", [(1, 0), (1, 2), (1, 4), (2, 1), (2, 3), (3, 2), (3, 4)])
def test_monomial_count_and_order(F, G):
    mons = monomials(F, G)
    assert len(mons) == comb(F + G, G) == len(set(mons))
    degs = [sum(e) for e in mons]
    assert degs == sorted(degs)
    assert mons[0] == (0,) * F


def test_paper_burgers_expressions():
    """p_1(u~) = theta_0 + theta_1 u~ + theta_2 u~^2 (degree two, one field);
    P:339: the true Burgers equation u_t = u u_x + 0.1 u_xx has theta_1 = 1, phi_0 = 0.1,
    all other parameters 0.  In the form sum_m c_m u_m = b with fields (phi, t, tt, x, xx):
    c_t = 1, c_x = -p_1, c_xx = -p_2."""
    assert monomials(1, 2) == [(0,), (1,), (2,)]
    rng = np.random.default_rng(3)
    u = rng.normal(size=(1, 50))
    th = np.zeros((6, 3))
    th[1, 0] = 1.0             # c_t = 1
    th[3, 1] = -1.0            # c_x = -(theta_1 u~), theta_1 = 1
    th[4, 0] = -0.1            # c_xx = -(phi_0),    phi_0 = 0.1
    c, b = template_coeff(th, u, 2)
    np.testing.assert_array_equal(c[1], 1.0)
    np.testing.assert_allclose(c[3], -u[0], rtol=0, atol=0)
    np.testing.assert_array_equal(c[4], -0.1)
    np.testing.assert_array_equal(c[[0, 2]], 0.0)
    np.testing.assert_array_equal(b, 0.0)
    # a general theta reproduces the printed quadratic for every point
    th2 = rng.normal(size=(6, 3))
    c2, _ = template_coeff(th2, u, 2)
    np.testing.assert_allclose(c2[3], th2[3, 0] + th2[3, 1] * u[0] + th2[3, 2] * u[0] ** 2,
                               rtol=1e-14)


def test_two_field_cubic_closed_form():
    """third-degree polynomials of (u~, v~); Phi evaluated against numpy.polynomial's
    2-D power-series evaluation (an independent routine)."""
    rng = np.random.default_rng(4)
    uv = rng.normal(size=(2, 40))
    mons = monomials(2, 3)
    coef = rng.normal(size=len(mons))
    cgrid = np.zeros((4, 4))
    for a, e in zip(coef, mons):
        cgrid[e[0], e[1]] += a
    ref = np.polynomial.polynomial.polyval2d(uv[0], uv[1], cgrid)
    np.testing.assert_allclose(coef @ features(uv, 3), ref, rtol=1e-12)


def test_template_gradients_match_central_differences():
    """dl/dtheta and dl/du~ of l = <g, z*(c(theta, u~), b(theta, u~), omega)> through the
    full dense least-squares solve and P:240, against central finite differences."""
    shape, h = (8, 9), (0.1, 0.2)
    pr = Problem(shape, h, w_eq=1.2, w_bnd=1.5, w_der=0.8, w_sm=1.1)
    rng = np.random.default_rng(11)
    F, G = 2, 2
    K = comb(F + G, G)
    u = 0.5 * rng.normal(size=(F, pr.P))
    th = 0.3 * rng.normal(size=(pr.M + 1, K))
    th[1, 0] = 1.0  # c_t = 1 keeps A full rank
    om = rng.normal(size=pr.P)
    g = rng.normal(size=pr.n_v)

    def loss(th_, u_):
        c, b = template_coeff(th_, u_, G)
        return g @ solve_forward(pr, c, b, om, method="dense")["z"]

    c, b = template_coeff(th, u, G)
    f = solve_forward(pr, c, b, om, method="dense")
    bw = solve_backward(pr, f, g, method="dense")
    gth, gu = template_grad(th, u[None], G, bw["grad_c"][None], bw["grad_b"][None])
    eps = 1e-6
    for m, k in [(0, 0), (1, 2), (3, 1), (4, 5), (pr.M, 0), (pr.M, 3), (2, 4)]:
        tp, tm = th.copy(), th.copy()
        tp[m, k] += eps
        tm[m, k] -= eps
        fd = (loss(tp, u) - loss(tm, u)) / (2 * eps)
        assert abs(fd - gth[m, k]) <= 1e-6 * max(1.0, np.abs(gth).max())
    for f_, p in [(0, 10), (1, 33), (0, 50), (1, 71)]:
        up, um = u.copy(), u.copy()
        up[f_, p] += eps
        um[f_, p] -= eps
        fd = (loss(th, up) - loss(th, um)) / (2 * eps)
        assert abs(fd - gu[0, f_, p]) <= 1e-6 * max(1.0, np.abs(gu).max())
    assert not boundary_mask(shape).all()


def test_template_grad_batch_sums():
    """theta is shared over the batch: dl/dtheta of a batch is the sum of the per-PDE
    gradients, grad_feat is per PDE."""
    rng = np.random.default_rng(5)
    th = rng.normal(size=(6, 5))
    u = rng.normal(size=(3, 1, 20))
    gc = rng.normal(size=(3, 5, 20))
    gb = rng.normal(size=(3, 20))
    gth, gu = template_grad(th, u, 4, gc, gb)
    parts = [template_grad(th, u[i:i + 1], 4, gc[i:i + 1], gb[i:i + 1]) for i in range(3)]
    np.testing.assert_allclose(gth, sum(p[0] for p in parts), rtol=1e-12)
    np.testing.assert_allclose(gu, np.concatenate([p[1] for p in parts]), rtol=1e-12)
