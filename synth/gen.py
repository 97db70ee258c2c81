"""Seeded generators for configs C1-C5 (BASELINE.json ``configs``).

Field order of c: (phi, d0, d00, d1, d11, d2, d22), dim 0 = time (slowest).  All
fields are built in float64 and rounded to float32 once; both the oracle and the
CUDA path consume the rounded values.  ``rng = default_rng(1000*k + b)`` for config
Ck and batch index b.

Workload shapes (the paper's PDE families, Table 1):
  C1 heat 1D                     (t,x)   = (16,16)    batch 1
  C2 Burgers 1D template         (t,x)   = (101,256)  batch 64
  C3 lambda-omega RD, two fields (t,x,y) = (32,32,32) 8 samples x 2 solves
  C4 NS vorticity (the metric)   (t,x,y) = (32,64,64) batch 32
  C5 scaling sweep               (t,x,y) = (64,128,128) batch 256 (C4 generator)

MMS twin (``make_mms``): same grid and c, u a random polynomial of degree <= 2 in each
dim, b := sum_m c_m d_m u and omega := u, so the exact solution z* = (u, du) is known in
closed form.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    k: int              # seed block: rng seed = 1000*k + b
    shape: tuple        # points per dim, dim 0 = time
    h: tuple            # uniform step per dim
    origin: tuple       # coordinate of index 0 per dim
    batch: int
    kind: str


CONFIGS = {
    "C1": Config("C1", 1, (16, 16), (1 / 15, 1 / 15), (0.0, 0.0), 1, "heat1d"),
    "C2": Config("C2", 2, (101, 256), (0.1, 1 / 16), (0.0, -8.0), 64, "burgers1d"),
    "C3": Config("C3", 3, (32, 32, 32), (0.05, 0.3125, 0.3125), (0.0, 0.0, 0.0), 16, "rd2d"),
    "C4": Config("C4", 4, (32, 64, 64), (0.01, 1 / 64, 1 / 64), (0.0, 0.0, 0.0), 32, "ns2d"),
    "C5": Config("C5", 5, (64, 128, 128), (0.005, 1 / 128, 1 / 128), (0.0, 0.0, 0.0), 256, "ns2d"),
}


def field_names(D: int):
    names = ["phi"]
    for d in range(D):
        names += [f"d{d}", f"d{d}{d}"]
    return names


def _coords(cfg: Config):
    axes = [cfg.origin[d] + cfg.h[d] * np.arange(n) for d, n in enumerate(cfg.shape)]
    return np.meshgrid(*axes, indexing="ij")


def _heat1d(cfg, rng):
    t, x = _coords(cfg)
    nu = 0.1
    c = np.zeros((5,) + cfg.shape)
    c[1] = 1.0            # u_t
    c[4] = -nu            # -nu u_xx
    b = np.zeros(cfg.shape)
    omega = np.exp(-nu * np.pi ** 2 * t) * np.sin(np.pi * x)
    return c, b, omega


def _burgers1d(cfg, rng):
    t, x = _coords(cfg)
    ut = np.zeros(cfg.shape)
    for k in range(1, 5):
        a = rng.normal(0.0, 1.0 / k)
        ph = rng.uniform(0.0, 2 * np.pi)
        ut += a * np.exp(-0.1 * (k * np.pi / 8) ** 2 * t) * np.sin(k * np.pi * (x + 8) / 16 + ph)
    ut /= np.abs(ut).max()
    theta = np.array([0.0, 1.0, 0.0, 0.0, 0.0]) + rng.normal(0.0, 0.05, 5)
    phi = np.array([0.1, 0.0, 0.0, 0.0, 0.0]) + rng.normal(0.0, 0.01, 5)
    p1 = sum(theta[j] * ut ** j for j in range(5))
    p2 = sum(phi[j] * ut ** j for j in range(5))
    c = np.zeros((5,) + cfg.shape)
    c[1] = 1.0
    c[3] = -p1
    c[4] = -np.maximum(p2, 0.02)
    return c, np.zeros(cfg.shape), ut


def _rd2d(cfg, rng, which):
    t, x, y = _coords(cfg)
    cx, cy = rng.uniform(3.0, 7.0, 2)
    r = np.hypot(x - cx, y - cy)
    th = np.arctan2(y - cy, x - cx)
    amp = np.tanh(r / 2) * np.exp(1j * (th - 0.8 * r - t))
    u, v = amp.real, amp.imag
    gam = rng.normal(0.0, 1.0, 10)
    mons = [u ** i * v ** j for i in range(4) for j in range(4 - i)]
    q = sum(g * mm for g, mm in zip(gam, mons))
    D1, beta = 0.1, 1.0
    a2 = u * u + v * v
    c = np.zeros((7,) + cfg.shape)
    c[0] = -(1.0 - a2)
    c[1] = 1.0
    c[4] = c[6] = -D1 * (1.0 + 0.01 * q)
    if which == 0:
        return c, beta * a2 * v, u
    return c, -beta * a2 * u, v


def _ns2d(cfg, rng):
    nt, nx, ny = cfg.shape
    t = cfg.origin[0] + cfg.h[0] * np.arange(nt)
    xs = cfg.origin[1] + cfg.h[1] * np.arange(nx)
    ys = cfg.origin[2] + cfg.h[2] * np.arange(ny)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    U1 = np.zeros(cfg.shape)
    U2 = np.zeros(cfg.shape)
    zeta = np.zeros(cfg.shape)
    for k1 in range(-4, 5):
        for k2 in range(-4, 5):
            if k1 == 0 and k2 == 0:
                continue
            kk = k1 * k1 + k2 * k2
            a = rng.normal(0.0, 1.0 / kk)
            ph = rng.uniform(0.0, 2 * np.pi)
            arg = 2 * np.pi * (k1 * X + k2 * Y) + ph
            decay = a * np.exp(-0.5 * kk * t)[:, None, None]
            s, cs = np.sin(arg)[None], np.cos(arg)[None]
            U1 += decay * (-2 * np.pi * k2) * s        # d psi / dy
            U2 += decay * (2 * np.pi * k1) * s         # -d psi / dx
            zeta += decay * (4 * np.pi ** 2 * kk) * cs  # -lap psi
    scale = np.sqrt(U1 ** 2 + U2 ** 2).max()
    U1 /= scale
    U2 /= scale
    zeta /= scale
    nu = 1e-3
    c = np.zeros((7,) + cfg.shape)
    c[1] = 1.0
    c[3] = U1
    c[5] = U2
    c[4] = c[6] = -nu
    return c, np.zeros(cfg.shape), zeta


def make_pde(cfg_name: str, index: int):
    """One PDE of config ``cfg_name`` at batch index ``index`` (float64 fields)."""
    cfg = CONFIGS[cfg_name]
    if cfg.kind == "rd2d":
        rng = np.random.default_rng(1000 * cfg.k + index // 2)
        return _rd2d(cfg, rng, index % 2)
    rng = np.random.default_rng(1000 * cfg.k + index)
    return {"heat1d": _heat1d, "burgers1d": _burgers1d, "ns2d": _ns2d}[cfg.kind](cfg, rng)


def make_batch(cfg_name: str, batch: int | None = None, start: int = 0):
    """Batch of PDEs, float32: c [B][M][P], b [B][P], omega [B][P]."""
    cfg = CONFIGS[cfg_name]
    B = cfg.batch if batch is None else batch
    D = len(cfg.shape)
    P = int(np.prod(cfg.shape))
    c = np.empty((B, 1 + 2 * D, P), np.float32)
    b = np.empty((B, P), np.float32)
    om = np.empty((B, P), np.float32)
    for i in range(B):
        ci, bi, oi = make_pde(cfg_name, start + i)
        c[i] = ci.reshape(1 + 2 * D, P)
        b[i] = bi.reshape(P)
        om[i] = oi.reshape(P)
    return {"cfg": cfg, "c": c, "b": b, "omega": om}


def _mms_poly(cfg: Config, rng):
    """u = sum_{e in {0,1,2}^D} alpha_e prod_d s_d^{e_d}, s_d = (x_d - x0_d)/L_d, with its
    pure first/second derivatives per dim (closed form)."""
    D = len(cfg.shape)
    axes = [np.arange(n) * cfg.h[d] for d, n in enumerate(cfg.shape)]
    L = [(n - 1) * cfg.h[d] for d, n in enumerate(cfg.shape)]
    s = [a / l for a, l in zip(axes, L)]
    alpha = rng.normal(0.0, 1.0, (3,) * D)
    # per-dim basis values and derivatives: s^e, d/dx s^e, d2/dx2 s^e
    basis = []
    for d in range(D):
        sd, l = s[d], L[d]
        val = np.stack([np.ones_like(sd), sd, sd * sd])
        d1 = np.stack([np.zeros_like(sd), np.ones_like(sd) / l, 2 * sd / l])
        d2 = np.stack([np.zeros_like(sd), np.zeros_like(sd), np.full_like(sd, 2 / l ** 2)])
        basis.append((val, d1, d2))
    fields = []
    for which in [None] + [(d, k) for d in range(D) for k in (1, 2)]:
        out = np.zeros(cfg.shape)
        for e in np.ndindex(*(3,) * D):
            term = alpha[e]
            for d in range(D):
                tbl = basis[d][0] if which is None or which[0] != d else basis[d][which[1]]
                sh = [1] * D
                sh[d] = -1
                term = term * tbl[e[d]].reshape(sh)
            out = out + term
        fields.append(out)
    return np.stack(fields)


def make_mms(cfg_name: str, batch: int | None = None, start: int = 0):
    """MMS twin of ``make_batch``: same c; b := sum_m c_m d_m u, omega := u (float32);
    ``z_exact`` [B][M][P] float64 is the closed-form solution."""
    base = make_batch(cfg_name, batch, start)
    cfg = base["cfg"]
    B, M, P = base["c"].shape
    z = np.empty((B, M, P))
    b = np.empty((B, P), np.float32)
    om = np.empty((B, P), np.float32)
    for i in range(B):
        rng = np.random.default_rng(10_000_000 + 1000 * cfg.k + start + i)
        zi = _mms_poly(cfg, rng).reshape(M, P)
        z[i] = zi
        b[i] = (base["c"][i].astype(np.float64) * zi).sum(axis=0)
        om[i] = zi[0]
    return {"cfg": cfg, "c": base["c"], "b": b, "omega": om, "z_exact": z}


def make_g(cfg_name: str, batch: int | None = None, start: int = 0, seed: int = 77):
    """Loss direction g = dl/dz*, N(0,1) float32 [B][M][P] (SURVEY.md §8(c) parity dir. 1)."""
    cfg = CONFIGS[cfg_name]
    B = cfg.batch if batch is None else batch
    D = len(cfg.shape)
    P = int(np.prod(cfg.shape))
    out = np.empty((B, 1 + 2 * D, P), np.float32)
    for i in range(B):
        rng = np.random.default_rng(seed * 100_000 + 1000 * cfg.k + start + i)
        out[i] = rng.standard_normal((1 + 2 * D, P))
    return out


def make_template_batch(cfg_name: str, batch: int | None = None, start: int = 0):
    """Template twin of the C4 Navier-Stokes workload (SURVEY.md §8(f) N2, P:551-553:
    "degree 1 polynomials"): feature fields u~ = (U1, U2) [B][2][P] and the parameters
    theta [|M|+1][3] (monomials 1, U1, U2) of the vorticity-transport equation the C4
    generator draws: c_t = 1, c_x = U1, c_y = U2, c_xx = c_yy = -nu, b = 0.  Only draws
    inputs; evaluating the template is the method's job."""
    if CONFIGS[cfg_name].kind != "ns2d":
        raise ValueError("template twin defined for the NS-vorticity configs (C4, C5)")
    bt = make_batch(cfg_name, batch, start)
    feat = np.ascontiguousarray(bt["c"][:, [3, 5]])
    return {"cfg": bt["cfg"], "feat": feat, "theta": ns_template_theta(), "omega": bt["omega"],
            "c": bt["c"]}


def ns_template_theta():
    """theta [8][3] of the NS template twin (monomials 1, U1, U2; rows phi, t, tt, x, xx, y,
    yy, b): c_t = 1, c_x = U1, c_y = U2, c_xx = c_yy = -nu (nu = 1e-3), b = 0."""
    nu = np.float32(1e-3)
    theta = np.zeros((8, 3), np.float32)
    theta[1, 0] = 1.0
    theta[3, 1] = 1.0
    theta[5, 2] = 1.0
    theta[4, 0] = theta[6, 0] = -nu
    return theta
