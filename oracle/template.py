"""Plain float64 oracle of the polynomial PDE-expression template.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.

The paper builds the PDE coefficients from learned polynomial expressions of
transformed data fields:
  * P:332-337 (§4 "Discovery Example", Eq. burgers-example): "Choosing degree two
    polynomials as the expression functions we obtain the coefficients for u_x and u_xx
    respectively as p_1(u~) = theta_0 + theta_1 u~ + theta_2 u~^2 and
    p_2(u~) = phi_0 + phi_1 u~ + phi_2 u~^2";
  * P:520-521 (reaction-diffusion): "third degree polynomial functions built from the
    parameterized inputs u~, v~ ... four separate polynomial expressions in the PDE: one
    serving as the coefficients of the u term, another two for the u_xx and u_yy terms,
    and one as the right hand side b";
  * P:552 (Navier-Stokes): "degree 1 polynomials".

Definition used by this oracle and by the CUDA path (reading T1):
every coefficient field and the right-hand side is a polynomial of total degree <= G in
the F feature fields u~_0..u~_{F-1} of the same grid point,
    c_m(p) = sum_k theta[m][k] Phi_k(u~(p)),    b(p) = sum_k theta[M][k] Phi_k(u~(p)),
with Phi_k the monomials prod_f u~_f^{e_f}, ordered by total degree, and within one degree
by exponent tuple in descending lexicographic order (F = 1: 1, u, u^2, ...; F = 2, G = 2:
1, u0, u1, u0^2, u0 u1, u1^2).  A coefficient the paper fixes (c_t = 1 in Eq.
burgers-example) is the constant monomial of its row.  theta is shared by the whole batch
(the discovered equation).  The gradient of a loss l through this map is the chain rule
written out point by point:
    dl/dtheta[m][k] = sum_b sum_p dl/dc_m(p) Phi_k(u~_b(p))   (row M: dl/db)
    dl/du~_f(p)     = sum_m dl/dc_m(p) sum_k theta[m][k] dPhi_k/du~_f + (same for b).
Pinned (tests/test_template_oracle.py) by the paper's printed p_1/p_2,
monomial counts C(F+G, G), and central finite differences through the full oracle solve.
"""
from __future__ import annotations

from itertools import product
from math import comb

import numpy as np


def monomials(n_feat: int, degree: int):
    """Exponent tuples of all monomials of total degree <= degree in n_feat variables, in
    the order stated in the module docstring."""
    out = []
    for t in range(degree + 1):
        same = [e for e in product(range(t, -1, -1), repeat=n_feat) if sum(e) == t]
        same.sort(reverse=True)
        out.extend(same)
    assert len(out) == comb(n_feat + degree, degree)
    return out


def features(feat: np.ndarray, degree: int) -> np.ndarray:
    """Phi [K][P] from feat [F][P]: each monomial evaluated literally, in fp64."""
    feat = np.asarray(feat, dtype=np.float64)
    F, P = feat.shape
    mons = monomials(F, degree)
    phi = np.ones((len(mons), P))
    for k, e in enumerate(mons):
        for f in range(F):
            for _ in range(e[f]):
                phi[k] *= feat[f]
    return phi


def template_coeff(theta: np.ndarray, feat: np.ndarray, degree: int):
    """(c [M][P], b [P]) of one PDE: theta [(M+1)][K], feat [F][P]."""
    theta = np.asarray(theta, dtype=np.float64)
    phi = features(feat, degree)
    K = phi.shape[0]
    assert theta.shape[1] == K
    rows = np.zeros((theta.shape[0], phi.shape[1]))
    for m in range(theta.shape[0]):
        for k in range(K):
            rows[m] += theta[m, k] * phi[k]
    return rows[:-1], rows[-1]


def template_grad(theta: np.ndarray, feat_batch: np.ndarray, degree: int,
                  grad_c_batch: np.ndarray, grad_b_batch: np.ndarray):
    """Chain rule through the template for a batch.

    feat_batch [B][F][P], grad_c_batch [B][M][P], grad_b_batch [B][P] ->
    (grad_theta [(M+1)][K] summed over the batch, grad_feat [B][F][P])."""
    theta = np.asarray(theta, dtype=np.float64)
    feat_batch = np.asarray(feat_batch, dtype=np.float64)
    Bn, F, P = feat_batch.shape
    mons = monomials(F, degree)
    K = len(mons)
    R = theta.shape[0]
    gth = np.zeros((R, K))
    gfeat = np.zeros((Bn, F, P))
    for b in range(Bn):
        g_rows = np.concatenate([np.asarray(grad_c_batch[b], np.float64),
                                 np.asarray(grad_b_batch[b], np.float64)[None]], axis=0)
        phi = features(feat_batch[b], degree)
        for m in range(R):
            for k in range(K):
                gth[m, k] += np.dot(g_rows[m], phi[k])
        # d Phi_k / d u_f = e_f u_f^(e_f - 1) prod_{f' != f} u_f'^e_f'
        for f in range(F):
            for k, e in enumerate(mons):
                if e[f] == 0:
                    continue
                dphi = np.full(P, float(e[f]))
                for f2 in range(F):
                    for _ in range(e[f2] - (1 if f2 == f else 0)):
                        dphi *= feat_batch[b, f2]
                for m in range(R):
                    gfeat[b, f] += g_rows[m] * theta[m, k] * dphi
    return gth, gfeat
