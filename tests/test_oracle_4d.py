"""Oracle pins in 4D (t + three space dims; the grid, the derivative variables and the
Taylor rows are defined per dim for any D).  The oracle's assembly is dimension-generic; these
pins fix it at D = 4 before the GPU parity tests (tests/test_gpu_4d.py) lean on it:
  - row counts group by group (Eqs. 3-7 with mixed face types);
  - manufactured per-dim-quadratic fields satisfy A z = d exactly (every stencil and Taylor row
    along all four axes is exact on quadratics), with Dirichlet and Neumann data;
  - reduction to 2D: data constant along two space dims whose faces carry no rows make the
    broadcast 2D least-squares solution (with zero derivative fields along those dims) a
    stationary point of the 4D least-squares objective, A^T (A z - d) = 0."""
import numpy as np
import pytest

from oracle import Problem, assemble, counts, solve_forward
from oracle.neurlp import boundary_mask, face_points, field_index

MIXED4 = (("D", "-"), ("N", "D"), ("D", "N"), ("N", "N"))


def _quad4(shape, h, rng):
    D = len(shape)
    L = [(n - 1) * h[d] for d, n in enumerate(shape)]
    X = np.meshgrid(*[np.arange(n) * h[d] / L[d] for d, n in enumerate(shape)], indexing="ij")
    a = rng.normal(size=(3,) * D)
    out = []
    for which in [None] + [(d, k) for d in range(D) for k in (1, 2)]:
        f = np.zeros(shape)
        for e in np.ndindex(*(3,) * D):
            t = np.full(shape, a[e])
            for d in range(D):
                s, p = X[d], e[d]
                if which is not None and which[0] == d:
                    if which[1] == 1:
                        v = p * s ** (p - 1) / L[d] if p >= 1 else 0 * s
                    else:
                        v = p * (p - 1) * s ** (p - 2) / L[d] ** 2 if p >= 2 else 0 * s
                else:
                    v = s ** p
                t = t * v
            f = f + t
        out.append(f.reshape(-1))
    return np.stack(out)


@pytest.mark.parametrize("shape,bc", [((6, 7, 6, 8), None), ((7, 6, 9, 6), MIXED4)])
def test_row_counts_4d(shape, bc):
    pr = Problem(shape, (0.1,) * 4, bc=bc)
    rng = np.random.default_rng(0)
    c = rng.normal(size=(pr.M, pr.P))
    A, _, info = assemble(pr, c, np.zeros(pr.P), np.zeros(pr.P))
    n_v, n_c = counts(shape, bc)
    P = pr.P
    nd = int(boundary_mask(shape, bc, "D").sum())
    nn = sum(face_points(shape, d, s).size for d in range(4) for s in (0, 1)
             if bc is not None and bc[d][s] == "N")
    assert pr.M == 9 and n_v == 9 * P and A.shape == (n_c, n_v)
    assert n_c == P + nd + nn + 8 * P + sum(2 * (n - 1) * (P // n) for n in shape)
    if bc is None:  # every point with an index on a face of the 4-cube
        inner = int(np.prod([n - 2 for n in shape]))
        assert nd == P - inner


@pytest.mark.parametrize("shape,h,bc", [((6, 7, 6, 8), (0.1, 0.12, 0.09, 0.11), None),
                                        ((7, 6, 9, 6), (0.2, 0.1, 0.15, 0.3), MIXED4)])
def test_manufactured_fields_satisfy_constraints_4d(shape, h, bc):
    rng = np.random.default_rng(1)
    pr = Problem(shape, h, 1.3, 2.0, 0.7, 0.9, bc=bc)
    c = rng.normal(0.0, 0.5, (pr.M, pr.P))
    c[1] += 1.0
    z = _quad4(shape, h, rng)
    b = (c * z).sum(axis=0)
    omn = np.stack([z[field_index(d, 1)] for d in range(4)])
    A, d, _ = assemble(pr, c, b, z[0], omn)
    r = A @ z.reshape(-1) - d
    assert np.linalg.norm(r) <= 1e-11 * np.linalg.norm(d)
    # a wrong sign anywhere breaks it: perturbing one derivative field leaves a residual
    z2 = z.copy()
    z2[field_index(3, 2)] *= 1.01
    assert np.linalg.norm(A @ z2.reshape(-1) - d) > 1e-6 * np.linalg.norm(d)


def test_reduces_to_2d_when_constant_along_two_dims():
    n0, n1, n2, n3 = 7, 8, 6, 6
    h = (0.1, 0.12, 0.2, 0.25)
    rng = np.random.default_rng(2)
    pr2 = Problem((n0, n1), h[:2], 1.3, 2.0, 0.7, 0.9)
    c2 = rng.normal(0.0, 0.5, (5, n0 * n1))
    c2[1] += 1.0
    b2 = rng.normal(size=n0 * n1)
    om2 = rng.normal(size=n0 * n1)
    z2 = solve_forward(pr2, c2, b2, om2, method="dense")["z"].reshape(5, n0, n1)
    bc4 = (("D", "D"), ("D", "D"), ("-", "-"), ("-", "-"))
    pr4 = Problem((n0, n1, n2, n3), h, 1.3, 2.0, 0.7, 0.9, bc=bc4)
    bcast = lambda a: np.broadcast_to(a.reshape(n0, n1, 1, 1), (n0, n1, n2, n3)).reshape(-1)
    c4 = np.zeros((9, pr4.P))
    for m in range(5):  # fields phi, (0,1), (0,2), (1,1), (1,2) keep their indices in 4D
        c4[m] = bcast(c2[m])
    A, d, _ = assemble(pr4, c4, bcast(b2), bcast(om2))
    z4 = np.zeros((9, pr4.P))
    for m in range(5):
        z4[m] = bcast(z2[m])
    g = A.T @ (A @ z4.reshape(-1) - d)
    assert np.linalg.norm(g) <= 1e-9 * np.linalg.norm(A.T @ d)
    # and it is not trivially stationary: shifting phi off the 2D solution is not
    z4[0] += 1e-3
    assert np.linalg.norm(A.T @ (A @ z4.reshape(-1) - d)) > 1e-6 * np.linalg.norm(A.T @ d)
