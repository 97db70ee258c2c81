"""Plain float64 CPU oracle of the NeuRLP-PDE solve (arXiv 2502.18377, §3).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Nothing here is blocked,
fused or reordered beyond what the paper's definitions state: the constraint
matrix A and vector d are assembled explicitly row by row (Eqs. 3-8), the least
squares problem is solved through its normal equations (Eq. 9), the duals are the
first block row of the saddle system (Eq. 10) and the backward pass is Eq. 11
followed by the gradient formulas of P:240.

Conventions:
  * points are row-major with dim 0 = time slowest; variables are field-major
    z[m*P + p] with fields ordered (phi, d0, d00, d1, d11, ...)             (Q2)
  * the boundary set B is every point on any face of the space-time box       (Q1)
  * boundary types per face ("Dirichlet ..., Neumann ... or mixed types"):
    'D' (default) u_phi = omega on the face, 'N' the first derivative along the face's
    axis = omega_n[d] on the face, '-' no boundary row (reading B1)
  * derivative rows: h_d^k z[(d,k),p] - sum_j a^k_j z[phi, p + o_j e_d] = 0
    with 5-point central weights for 2 <= i_d <= n_d-3 and fully one-sided
    5-point weights at the two points nearest each edge                 (Q4, Q5)
  * smoothness rows in both directions wherever the neighbour exists         (Q7)
  * duals lambda = d - A z                                                   (Q8)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


# ----------------------------------------------------------------------------
# Problem description
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Problem:
    """One grid + weights.  P:89 (§2 Cartesian grid), P:114-117 (uniform steps).

    ``shape`` = points per dim (dim 0 = t), ``h`` = step per dim, weights are the
    row-group weights (Q6; the paper's Eqs. 8-9 are unweighted = all 1).
    """
    shape: tuple
    h: tuple
    w_eq: float = 1.0
    w_bnd: float = 1.0
    w_der: float = 1.0
    w_sm: float = 1.0
    bc: tuple | None = None  # per dim (low face, high face) in {'D', 'N', '-'}; None = all 'D'
    order: tuple | None = None  # per dim highest derivative variable, 2 or 3; None = all 2

    def face_type(self, d: int, side: int) -> str:
        return "D" if self.bc is None else self.bc[d][side]

    def ord(self, d: int) -> int:
        """Highest derivative order kept as a variable along dim d ("partial derivatives
        of arbitrary order"; reading O3: 2 by default, 3 for the KdV u_xxx term)."""
        return 2 if self.order is None else int(self.order[d])

    def field(self, d: int, k: int) -> int:
        """Field index of the k-th derivative along dim d: phi first, then per dim its
        derivatives of orders 1 .. ord(d) (= field_index for the default order 2)."""
        return 1 + sum(self.ord(e) for e in range(d)) + (k - 1)

    @property
    def D(self) -> int:
        return len(self.shape)

    @property
    def P(self) -> int:
        return int(np.prod(self.shape))

    @property
    def M(self) -> int:
        return 1 + sum(self.ord(d) for d in range(self.D))

    @property
    def n_v(self) -> int:
        return self.M * self.P


def n_fields(D: int) -> int:
    """|M| = 1 + 2D: phi plus first and second pure derivative per dim (Q2)."""
    return 1 + 2 * D


def field_index(d: int, k: int) -> int:
    """Index of the field holding the k-th derivative (k = 1, 2) along dim d."""
    return 1 + 2 * d + (k - 1)


def boundary_mask(shape, bc=None, kind: str = "D") -> np.ndarray:
    """B = points with i_d in {0, n_d-1} for some d (reading Q1).

    With per-face types `bc` (Problem.bc), the points on at least one face of type `kind`."""
    mask = np.zeros(shape, dtype=bool)
    for d, n in enumerate(shape):
        for side, i in ((0, 0), (1, n - 1)):
            if bc is not None and bc[d][side] != kind:
                continue
            sl = [slice(None)] * len(shape)
            sl[d] = i
            mask[tuple(sl)] = True
    return mask.reshape(-1)


def face_points(shape, d: int, side: int) -> np.ndarray:
    """Flat indices of the points on face (d, side), ascending."""
    idx = np.unravel_index(np.arange(int(np.prod(shape))), shape)
    return np.flatnonzero(idx[d] == (0 if side == 0 else shape[d] - 1))


# 5-point finite-difference weights on a unit-spaced grid ("5 point central
# differences and ... forward, backward finite differences at the edges").
_A_CENTRAL = {1: np.array([1.0, -8.0, 0.0, 8.0, -1.0]) / 12.0,
              2: np.array([-1.0, 16.0, -30.0, 16.0, -1.0]) / 12.0}
_A_FORWARD = {1: np.array([-25.0, 48.0, -36.0, 16.0, -3.0]) / 12.0,
              2: np.array([35.0, -104.0, 114.0, -56.0, 11.0]) / 12.0}
# third derivative (reading O3, "arbitrary order"; the KdV term u_xxx of BASELINE C2): the
# 5-point central and one-sided rules, exact for polynomials of degree <= 4 like the others
_A_CENTRAL[3] = np.array([-1.0, 2.0, 0.0, -2.0, 1.0]) / 2.0
_A_FORWARD[3] = np.array([-5.0, 18.0, -24.0, 14.0, -3.0]) / 2.0


def fd_stencil(k: int, i: int, n: int):
    """(offsets, weights) of the k-th derivative stencil at index i of an n-point axis.

    Central for 2 <= i <= n-3, forward (offsets 0..4) for i < 2, backward
    (offsets 0..-4, a_bwd(-j) = (-1)^k a_fwd(j)) for i > n-3.  P:169-174 (Eq. 5);
    edge width/order is reading Q4.
    """
    if n < 6:
        raise ValueError("each dim needs >= 6 points for the 5-point edge stencils (Q4)")
    if 2 <= i <= n - 3:
        return np.arange(-2, 3), _A_CENTRAL[k]
    if i < 2:
        return np.arange(0, 5), _A_FORWARD[k]
    return -np.arange(0, 5), ((-1.0) ** k) * _A_FORWARD[k]


def counts(shape, bc=None, order=None):
    """(n_v, n_c) of the constraint system, counted row group by row group.

    n_c = P (Eq. 3) + |B| (Eq. 4) + 2D P (Eq. 5, one row per derivative variable)
          + sum_d 2 (n_d - 1) P / n_d (Eqs. 6-7 where the neighbour exists).
    With per-face types: |B| -> |B_D| (points on a Dirichlet face) + sum over Neumann faces
    of the face's point count.
    """
    D = len(shape)
    P = int(np.prod(shape))
    nb = int(boundary_mask(shape, bc, "D").sum())
    if bc is not None:
        nb += sum(P // shape[d] for d in range(D) for side in (0, 1) if bc[d][side] == "N")
    smooth = sum(2 * (n - 1) * (P // n) for n in shape)
    nder = 2 * D if order is None else int(sum(order))
    return (1 + nder) * P, P + nb + nder * P + smooth


# ----------------------------------------------------------------------------
# Assembly: Eqs. 3-8
# ----------------------------------------------------------------------------
def assemble(prob: Problem, c: np.ndarray, b: np.ndarray, omega: np.ndarray, omega_n=None):
    """Explicit sparse A (n_c x n_v, CSR, fp64) and d for one PDE.  P:186-191 (Eq. 8).

    c: [M][P] coefficient fields (Eq. 1); b: [P] right-hand side; omega: [P]
    (only entries on B are read, Eq. 4); omega_n: [D][P] Neumann data (only entries on the
    Neumann faces of dim d are read; None = 0).  Rows, in order:
      equation rows  (Eq. 3)      w_eq * sum_m c_m[p] z[m,p]       = w_eq b[p]
      boundary rows  (Eq. 4)      w_bnd * z[phi,p]                 = w_bnd omega[p]
                     (points on a Dirichlet face, p ascending)
      Neumann rows         w_bnd * z[(d,1),p]               = w_bnd omega_n[d][p]
                     (per Neumann face: d ascending, low then high, p ascending)
      derivative rows(Eq. 5)  w_der*(h^k z[(d,k),p] - sum_j a_j z[phi,p+o_j e_d]) = 0
      smoothness rows(Eqs. 6-7)
                      w_sm*(z[phi,p] +- h z[(d,1),p] + h^2/2 z[(d,2),p] - z[phi,p +- e_d]) = 0
    Returns (A, d, info) with info = {eq_rows, bnd_points, bnd_rows, neu}; neu lists
    (d, side, points, rows) per Neumann face.
    """
    shape, D, P, M = tuple(prob.shape), prob.D, prob.P, prob.M
    c = np.asarray(c, dtype=np.float64).reshape(M, P)
    b = np.asarray(b, dtype=np.float64).reshape(P)
    omega = np.asarray(omega, dtype=np.float64).reshape(P)
    for n in shape:
        if n < 6:
            raise ValueError("each dim needs >= 6 points (Q4)")
    pts = np.arange(P)
    idx = np.unravel_index(pts, shape)
    strides = [int(np.prod(shape[d + 1:])) for d in range(D)]
    rows, cols, vals, dvec = [], [], [], []
    r0 = 0

    # Equation rows (Eq. 3).  Structural entries are kept even where c_m[p] = 0,
    # because c is a parameter and its gradient lives on these entries.
    for m in range(M):
        rows.append(r0 + pts)
        cols.append(m * P + pts)
        vals.append(prob.w_eq * c[m])
    dvec.append(prob.w_eq * b)
    eq_rows = r0 + pts
    r0 += P

    # Boundary rows (Eq. 4): Dirichlet on u_phi.
    bpts = np.flatnonzero(boundary_mask(shape, prob.bc, "D"))
    rows.append(r0 + np.arange(bpts.size))
    cols.append(0 * P + bpts)
    vals.append(np.full(bpts.size, prob.w_bnd))
    dvec.append(prob.w_bnd * omega[bpts])
    bnd_rows = r0 + np.arange(bpts.size)
    r0 += bpts.size

    # Neumann rows: the first derivative along the face's axis.
    on = None if omega_n is None else np.asarray(omega_n, dtype=np.float64).reshape(D, P)
    neu = []
    for d in range(D):
        for side in (0, 1):
            if prob.face_type(d, side) != "N":
                continue
            fp = face_points(shape, d, side)
            rows.append(r0 + np.arange(fp.size))
            cols.append(prob.field(d, 1) * P + fp)
            vals.append(np.full(fp.size, prob.w_bnd))
            dvec.append(prob.w_bnd * (on[d][fp] if on is not None else np.zeros(fp.size)))
            neu.append((d, side, fp, r0 + np.arange(fp.size)))
            r0 += fp.size

    # Derivative rows (Eq. 5), one per (d, k, p), k = 1 .. ord(d).
    for d in range(D):
        n, hd, i_d = shape[d], prob.h[d], idx[d]
        for k in range(1, prob.ord(d) + 1):
            f = prob.field(d, k)
            rows.append(r0 + pts)
            cols.append(f * P + pts)
            vals.append(np.full(P, prob.w_der * hd ** k))
            for i in range(n):
                sel = pts[i_d == i]
                offs, wts = fd_stencil(k, i, n)
                for o, a in zip(offs, wts):
                    if a == 0.0:
                        continue
                    rows.append(r0 + sel)
                    cols.append(0 * P + sel + o * strides[d])
                    vals.append(np.full(sel.size, -prob.w_der * a))
            dvec.append(np.zeros(P))
            r0 += P

    # Smoothness rows (Eqs. 6-7), forward then backward, where the neighbour exists; the Taylor
    # expansion runs to the dim's highest derivative variable (+-h^3/6 u_ddd when ord = 3).
    for d in range(D):
        n, hd, i_d = shape[d], prob.h[d], idx[d]
        f1, f2 = prob.field(d, 1), prob.field(d, 2)
        for sgn in (+1, -1):
            sel = pts[(i_d <= n - 2) if sgn > 0 else (i_d >= 1)]
            rr = r0 + np.arange(sel.size)
            w = prob.w_sm
            terms = [(0 * P + sel, w), (f1 * P + sel, sgn * w * hd),
                     (f2 * P + sel, 0.5 * w * hd * hd)]
            if prob.ord(d) >= 3:
                terms.append((prob.field(d, 3) * P + sel, sgn * w * hd ** 3 / 6.0))
            terms.append((0 * P + sel + sgn * strides[d], -w))
            for col, val in terms:
                rows.append(rr)
                cols.append(col)
                vals.append(np.full(sel.size, val) if np.isscalar(val) else val)
            dvec.append(np.zeros(sel.size))
            r0 += sel.size

    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(r0, M * P))
    d_out = np.concatenate(dvec)
    return A, d_out, {"eq_rows": eq_rows, "bnd_points": bpts, "bnd_rows": bnd_rows, "neu": neu}


def normal_apply(A: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """A^T (A x): the normal operator of Eq. 9 applied to x."""
    return A.T @ (A @ x)


# ----------------------------------------------------------------------------
# Least squares on an arbitrary A: Eqs. 9-11 and P:240
# ----------------------------------------------------------------------------
def _svd_normal_solve(A, rhs):
    """(A^T A)^{-1} rhs via the SVD A = U S V^T: V S^-2 V^T rhs (plain definition)."""
    Ad = A.toarray() if sp.issparse(A) else np.asarray(A, dtype=np.float64)
    _, s, vt = np.linalg.svd(Ad, full_matrices=False)
    if s[-1] <= s[0] * 1e-13:
        raise np.linalg.LinAlgError("A is column-rank-deficient (P:109 assumes uniqueness)")
    return vt.T @ ((vt @ rhs) / (s * s))


def _equilibration(N):
    """S = diag(A^T A)^(-1/2): column equilibration (a change of variables)."""
    dg = N.diagonal()
    if np.any(dg <= 0):
        raise np.linalg.LinAlgError("zero column in A")
    return 1.0 / np.sqrt(dg)


STRICT_REL_RES = 1e-10  # largest normal residual an iterative oracle answer may have (strict)


def _slab_blocks(shape, M, T):
    """Index sets of the block-Jacobi blocks of method 'slab': all unknowns (every field m)
    of T consecutive planes along dim 0 (time), in the field-major z[m*P + p] order."""
    P = int(np.prod(shape))
    pl = P // shape[0]
    out = []
    for t in range(0, shape[0], T):
        te = min(shape[0], t + T)
        out.append(np.concatenate([m * P + np.arange(t * pl, te * pl) for m in range(M)]))
    return out


def solve_normal(A, rhs, method: str = "auto", tol: float = 1e-12, maxiter: int = 200000,
                 info: dict | None = None, strict: bool = True, shape=None, slab: int = 2,
                 log=None):
    """Solve A^T A x = rhs (Eq. 9).

    method: 'dense' (SVD), 'lu' (SuperLU on S A^T A S + 2 fp64 refinement steps with
    r = rhs - A^T A x), 'cg' (textbook CG on S A^T A S, i.e. Jacobi-preconditioned
    CG, stopping at ||rhs - A^T A x|| / ||rhs|| <= tol, true residual every 500 its) or
    'slab' (textbook preconditioned CG on S A^T A S whose preconditioner is block Jacobi
    with one block per `slab` consecutive t-planes -- every unknown of those planes -- each
    block factorised by SuperLU; `shape` = grid shape).  'slab' converges where 'cg' needs
    10^5 iterations (3D, transport-dominated C4 backward); the preconditioner only changes
    the speed: the stop test is the same true normal residual.  Iterative methods stop at
    rel_res <= tol, or when the true residual stagnates at the fp64 rounding floor (no halving
    within 150 iterations); with strict=True an answer whose rel_res exceeds STRICT_REL_RES
    raises.  log: optional callable receiving (iteration, rel_res) every 25 iterations.
    """
    n_v = A.shape[1]
    if method == "auto":
        method = "dense" if n_v <= 5000 else "cg"
    info = {} if info is None else info
    info["method"] = method
    rhs = np.asarray(rhs, dtype=np.float64)
    if not np.any(rhs):
        info["iters"] = 0
        return np.zeros(n_v)
    if method == "dense":
        return _svd_normal_solve(A, rhs)
    N = (A.T @ A).tocsr()
    s = _equilibration(N)
    if method == "lu":
        Ns = sp.diags(s) @ N @ sp.diags(s)
        lu = spla.splu(Ns.tocsc())
        x = s * lu.solve(s * rhs)
        for _ in range(2):
            r = rhs - N @ x
            x = x + s * lu.solve(s * r)
        return x
    if method == "slab":
        if shape is None:
            raise ValueError("method 'slab' needs the grid shape")
        M = n_v // int(np.prod(shape))
        Ns = (sp.diags(s) @ N @ sp.diags(s)).tocsr()
        blocks = [(idx, spla.splu(Ns[idx][:, idx].tocsc())) for idx in _slab_blocks(shape, M, slab)]

        def prec(r):
            out = np.empty_like(r)
            for idx, lu in blocks:
                out[idx] = lu.solve(r[idx])
            return out

        nrm = np.linalg.norm(rhs)
        bs = s * rhs
        y = np.zeros(n_v)  # unknowns of the scaled system: x = s * y
        r = bs.copy()
        zv = prec(r)
        p = zv.copy()
        rz = r @ zv
        it, best, since = 0, np.inf, 0
        hist = []
        while it < maxiter:
            q = Ns @ p
            alpha = rz / (p @ q)
            y += alpha * p
            r -= alpha * q
            it += 1
            if it % 25 == 0:
                rel = np.linalg.norm(rhs - N @ (s * y)) / nrm
                hist.append((it, float(rel)))
                if log is not None:
                    log(it, float(rel))
                if rel <= tol:
                    break
                if rel < 0.5 * best:
                    best, since = rel, 0
                else:
                    since += 25
                    if since >= 150:  # the true residual stopped halving: fp64 rounding floor
                        break
            zv = prec(r)
            rz_new = r @ zv
            p = zv + (rz_new / rz) * p
            rz = rz_new
        x = s * y
        info["iters"] = it
        info["rel_res"] = float(np.linalg.norm(rhs - N @ x) / nrm)
        info["history"] = hist
        if strict and not (info["rel_res"] <= STRICT_REL_RES):
            raise RuntimeError(f"oracle slab-PCG did not converge: rel_res {info['rel_res']:.3e} after "
                               f"{it} iterations")
        return x
    if method == "cg":
        minv = s * s
        x = np.zeros(n_v)
        r = rhs.copy()
        zv = minv * r
        p = zv.copy()
        rz = r @ zv
        nrm = np.linalg.norm(rhs)
        it = 0
        while it < maxiter:
            q = N @ p
            alpha = rz / (p @ q)
            x += alpha * p
            r -= alpha * q
            it += 1
            if it % 500 == 0:
                r = rhs - N @ x
            if np.linalg.norm(r) <= tol * nrm:
                r = rhs - N @ x
                if np.linalg.norm(r) <= tol * nrm:
                    break
            zv = minv * r
            rz_new = r @ zv
            p = zv + (rz_new / rz) * p
            rz = rz_new
        info["iters"] = it
        info["rel_res"] = float(np.linalg.norm(rhs - N @ x) / nrm)
        if strict and not (info["rel_res"] <= STRICT_REL_RES):
            raise RuntimeError(f"oracle CG did not converge: rel_res {info['rel_res']:.3e} after "
                               f"{it} iterations (ill-conditioned system; use method='lu')")
        return x
    raise ValueError(method)


def lstsq_forward(A, d, method: str = "auto", tol: float = 1e-12, info=None, shape=None, slab=2):
    """Forward pass: z* from A^T A z = A^T d (Eq. 9); lambda* = d - A z* (Eq. 10
    first block row, reading Q8).  'dense' solves min ||Az - d|| by SVD directly."""
    d = np.asarray(d, dtype=np.float64)
    if method == "dense" or (method == "auto" and A.shape[1] <= 5000):
        Ad = A.toarray() if sp.issparse(A) else np.asarray(A, dtype=np.float64)
        z = np.linalg.lstsq(Ad, d, rcond=None)[0]
        if info is not None:
            info["method"] = "dense"
    else:
        z = solve_normal(A, A.T @ d, method=method, tol=tol, info=info, shape=shape, slab=slab)
    lam = d - A @ z
    return z, lam


def lstsq_backward(A, z, lam, g, method: str = "auto", tol: float = 1e-12, info=None, shape=None,
                   slab=2):
    """Backward pass (Eq. 11).

    [[I, A], [A^T, 0]] [d_lam; d_z] = [0; -g]  =>  A^T A d_z = g,  d_lam = -A d_z.
    dA = d_lam z*^T + lambda* d_z^T on A's pattern, dd = -d_lam.
    Returns (d_z, d_lam, dA as a sparse matrix on A's pattern, dd).
    """
    dz = solve_normal(A, g, method=method, tol=tol, info=info, shape=shape, slab=slab)
    dlam = -(A @ dz)
    Acoo = sp.coo_matrix(A)
    gv = dlam[Acoo.row] * z[Acoo.col] + lam[Acoo.row] * dz[Acoo.col]
    dA = sp.csr_matrix((gv, (Acoo.row, Acoo.col)), shape=A.shape)
    return dz, dlam, dA, -dlam


# ----------------------------------------------------------------------------
# PDE-level forward / backward
# ----------------------------------------------------------------------------
def solve_forward(prob: Problem, c, b, omega, method: str = "auto", tol: float = 1e-12, slab=2,
                  omega_n=None):
    """Forward NeuRLP-PDE solve of one PDE.  Returns dict(z, lam, A, d, info)."""
    A, d, info = assemble(prob, c, b, omega, omega_n)
    sinfo = {}
    z, lam = lstsq_forward(A, d, method=method, tol=tol, info=sinfo, shape=tuple(prob.shape),
                           slab=slab)
    info.update(solve=sinfo)
    return {"z": z, "lam": lam, "A": A, "d": d, "info": info}


def field_gradients(prob: Problem, info, z, lam, dz, dlam):
    """Chain dA, dd through the assembly of Eqs. 3-4 to the encoder outputs.

    A[eq(p), (m,p)] = w_eq c_m[p]    =>  dl/dc_m[p] = w_eq * dA[eq(p), (m,p)]
    d[eq(p)]        = w_eq b[p]      =>  dl/db[p]   = w_eq * dd[eq(p)]
    d[bnd(p)]       = w_bnd omega[p] =>  dl/domega[p] = w_bnd * dd[bnd(p)], 0 off B
    with dA[i,j] = d_lam[i] z[j] + lam[i] d_z[j] and dd = -d_lam evaluated at the entries.
    """
    P, M = prob.P, prob.M
    er = info["eq_rows"]
    grad_c = np.empty((M, P))
    for m in range(M):
        j = m * P + np.arange(P)
        grad_c[m] = prob.w_eq * (dlam[er] * z[j] + lam[er] * dz[j])
    grad_b = prob.w_eq * (-dlam[er])
    grad_omega = np.zeros(P)
    grad_omega[info["bnd_points"]] = prob.w_bnd * (-dlam[info["bnd_rows"]])
    if info.get("neu"):  # d[neu(d,p)] = w_bnd omega_n[d][p]  =>  dl/domega_n = w_bnd dd[neu]
        grad_omega_n = np.zeros((prob.D, P))
        for d, side, fp, rr in info["neu"]:
            grad_omega_n[d][fp] += prob.w_bnd * (-dlam[rr])
        return grad_c, grad_b, grad_omega, grad_omega_n
    return grad_c, grad_b, grad_omega


def assemble_dh(prob: Problem, d: int, info) -> sp.csr_matrix:
    """dA/dh_d: the derivative of the assembly (Eqs. 5-7) with respect to the uniform step of
    dim d ("step sizes ... are differentiable").  Same row order as `assemble`
    (info from it); only the derivative rows of dim d (coefficient w_der h^k on z[(d,k),p] ->
    w_der k h^(k-1)) and the Taylor rows of dim d (+-w_sm h on z[(d,1),p] -> +-w_sm,
    w_sm h^2/2 on z[(d,2),p] -> w_sm h) depend on h_d."""
    shape, D, P = tuple(prob.shape), prob.D, prob.P
    pts = np.arange(P)
    idx = np.unravel_index(pts, shape)
    r0 = P + info["bnd_rows"].size + sum(rr.size for _, _, _, rr in info.get("neu", []))
    rows, cols, vals = [], [], []
    for dd in range(D):
        for k in range(1, prob.ord(dd) + 1):
            if dd == d:
                rows.append(r0 + pts)
                cols.append(prob.field(dd, k) * P + pts)
                vals.append(np.full(P, prob.w_der * k * prob.h[dd] ** (k - 1)))
            r0 += P
    for dd in range(D):
        n = shape[dd]
        for sgn in (+1, -1):
            sel = pts[(idx[dd] <= n - 2) if sgn > 0 else (idx[dd] >= 1)]
            if dd == d:
                rr = r0 + np.arange(sel.size)
                rows += [rr, rr]
                cols += [prob.field(dd, 1) * P + sel, prob.field(dd, 2) * P + sel]
                vals += [np.full(sel.size, sgn * prob.w_sm), np.full(sel.size, prob.w_sm * prob.h[dd])]
                if prob.ord(dd) >= 3:
                    rows.append(rr)
                    cols.append(prob.field(dd, 3) * P + sel)
                    vals.append(np.full(sel.size, sgn * prob.w_sm * 0.5 * prob.h[dd] ** 2))
            r0 += sel.size
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(r0, prob.n_v))


def step_gradient(prob: Problem, fwd: dict, bwd: dict) -> np.ndarray:
    """dl/dh_d for every dim: the P:240 matrix gradient dA = d_lambda z*^T + lambda* d_z^T
    contracted with dA/dh_d over A's entries: sum_(r,c) dA_rc (dA/dh_d)_rc."""
    z, lam, dz, dlam = fwd["z"], fwd["lam"], bwd["dz"], bwd["dlam"]
    out = np.zeros(prob.D)
    for d in range(prob.D):
        J = sp.coo_matrix(assemble_dh(prob, d, fwd["info"]))
        out[d] = float(np.sum(J.data * (dlam[J.row] * z[J.col] + lam[J.row] * dz[J.col])))
    return out


def solve_backward(prob: Problem, fwd: dict, g, method: str = "auto", tol: float = 1e-12, slab=2):
    """Backward NeuRLP-PDE solve for g = dl/dz* (Eq. 11) and field gradients."""
    sinfo = {}
    dz, dlam, dA, dd = lstsq_backward(fwd["A"], fwd["z"], fwd["lam"], g, method=method,
                                      tol=tol, info=sinfo, shape=tuple(prob.shape), slab=slab)
    grads = field_gradients(prob, fwd["info"], fwd["z"], fwd["lam"], dz, dlam)
    out = {"dz": dz, "dlam": dlam, "dA": dA, "dd": dd, "grad_c": grads[0], "grad_b": grads[1],
           "grad_omega": grads[2], "info": sinfo}
    if len(grads) == 4:
        out["grad_omega_n"] = grads[3]
    return out
