"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mpde.h
declares, and its host logic (validation, sizes, level plan) agrees with the oracle's
counts -- no compute calls (no GPU here)."""
import ctypes as C
import os
import re

import pytest

from oracle import counts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mp():
    from paper_2502_18377_b200 import build, mpde
    build.build()
    return mpde


def test_exports_every_declared_symbol(mp):
    hdr = open(os.path.join(ROOT, "include", "mpde.h")).read()
    declared = set(re.findall(r"\b(mpde_[a-z_0-9]+)\s*\(", hdr))
    assert declared >= {"mpde_build_hierarchy", "mpde_solve_fwd", "mpde_solve_bwd"}
    lib = C.CDLL(mp.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(mp.EXPORTS)


@pytest.mark.parametrize("shape", [(16, 16), (32, 32), (101, 256), (32, 32, 32), (32, 64, 64), (6, 7, 6, 8),
                                   (12, 16, 16, 20)])
def test_sizes_match_oracle_counts(mp, shape):
    prob = mp.make_problem(shape, [0.1] * len(shape), 4)
    n_v, n_c, _ = mp.mpde_sizes(prob)
    assert (n_v, n_c) == counts(shape)


def test_level_plan(mp):
    """halve each dim (ceil, keeping >= 6 points) down to size 8."""
    cases = {(32, 64, 64): 4, (101, 256): 6, (16, 16): 2, (32, 32, 32): 3, (64, 128, 128): 5}
    for shape, L in cases.items():
        prob = mp.make_problem(shape, [0.1] * len(shape), 1)
        assert mp.mpde_sizes(prob)[2] == L, shape
    prob = mp.make_problem((32, 64, 64), [0.1] * 3, 1)
    assert mp.mpde_sizes(prob, mp.mpde_default_options(levels_max=2))[2] == 2


def test_validation_errors(mp):
    lib = mp.lib()
    bad = [mp.make_problem((5, 16), (0.1, 0.1), 1),            # n < 6 (Q4)
           mp.make_problem((16, 16), (0.0, 0.1), 1),           # h = 0
           mp.make_problem((16, 16), (0.1, 0.1), 0)]           # batch 0
    codes = []
    for pr in bad:
        codes.append(lib.mpde_sizes(C.byref(pr), None, None, None, None))
    assert codes == [2, 1, 1]
    assert "6" in lib.mpde_last_error().decode() or lib.mpde_last_error()
    pr = mp.make_problem((16, 16), (0.1, 0.1), 1)
    pr.deriv_order = 3
    assert lib.mpde_sizes(C.byref(pr), None, None, None, None) == 3
    opts = mp.mpde_default_options(smoother=7)
    assert lib.mpde_workspace_bytes(C.byref(mp.make_problem((16, 16), (0.1, 0.1), 1)),
                                    C.byref(opts)) == 0


def test_workspace_scales_linearly_in_batch(mp):
    o = mp.mpde_default_options()
    w1 = mp.mpde_workspace_bytes(mp.make_problem((32, 64, 64), (0.01, 1 / 64, 1 / 64), 1), o)
    w32 = mp.mpde_workspace_bytes(mp.make_problem((32, 64, 64), (0.01, 1 / 64, 1 / 64), 32), o)
    assert 30 * w1 < w32 < 33 * w1
    # ~ tens of bytes per unknown (matrix-free), far below a CSR A^T A
    assert w32 / (32 * 7 * 131072) < 80


def test_template_terms_and_validation(mp):
    """mpde_template_terms = C(F+G, G) (the oracle's monomial count); unsupported templates
    are refused synchronously."""
    from math import comb

    from oracle.template import monomials
    for F in (1, 2, 3):
        for G in range(5):
            assert mp.mpde_template_terms(mp.make_template(F, G)) == comb(F + G, G) \
                == len(monomials(F, G))
    assert mp.mpde_template_terms(mp.make_template(4, 1)) == -1
    assert mp.mpde_template_terms(mp.make_template(1, 5)) == -1
    pr = mp.make_problem((32, 64, 64), (0.01, 1 / 64, 1 / 64), 32)
    # fp64 partials of grad_theta: one per (PDE, CTA of 1024 points) and (|M|+1) K entries
    assert mp.mpde_template_workspace_bytes(pr, mp.make_template(2, 1)) == 8 * 32 * 128 * 8 * 3
    assert mp.lib().mpde_template_workspace_bytes(C.byref(pr), C.byref(mp.make_template(2, 7))) == 0


def test_fgmres_options_and_workspace(mp):
    """krylov = 1 (FGMRES(m), §8(f) N1): default off, restart 30; the workspace grows by
    (2m+1) scalar fields per PDE plus the per-PDE Arnoldi state; restart outside 1..32 and an
    unknown Krylov method are rejected (workspace 0)."""
    import ctypes as C
    o = mp.mpde_default_options()
    assert o.krylov == 0 and o.restart == 30
    pr = mp.make_problem((32, 64, 64), (0.01, 1 / 64, 1 / 64), 4)
    w0 = mp.mpde_workspace_bytes(pr, o)
    for m in (1, 20, 32):
        w = mp.mpde_workspace_bytes(pr, mp.mpde_default_options(krylov=1, restart=m))
        assert w - w0 >= (2 * m + 1) * 4 * 32 * 64 * 64 * 4
    lib = mp.lib()
    for kw in ({"krylov": 1, "restart": 0}, {"krylov": 1, "restart": 33}, {"krylov": 2}):
        assert lib.mpde_workspace_bytes(C.byref(pr), C.byref(mp.mpde_default_options(**kw))) == 0


def test_adaptive_pass_tolerance_option(mp):
    """options.tol_adapt (Q14): default 0.1, 0 disables, values outside [0, 1)
    are rejected (workspace 0); ndim 4 is accepted and ndim 5 rejected."""
    import ctypes as C
    lib = mp.lib()
    assert abs(mp.mpde_default_options().tol_adapt - 0.1) < 1e-7
    pr = mp.make_problem((16, 16), (0.1, 0.1), 1)
    assert mp.mpde_workspace_bytes(pr, mp.mpde_default_options(tol_adapt=0.0)) > 0
    for bad in (-0.1, 1.0, float("nan")):
        assert lib.mpde_workspace_bytes(C.byref(pr), C.byref(mp.mpde_default_options(tol_adapt=bad))) == 0
    p4 = mp.make_problem((6, 7, 6, 8), (0.1,) * 4, 2)
    n_v, n_c, L = mp.mpde_sizes(p4)
    assert n_v == 9 * 6 * 7 * 6 * 8 and L == 1
    p5 = mp.make_problem((6, 6, 6, 6), (0.1,) * 4, 1)
    p5.ndim = 5
    assert lib.mpde_sizes(C.byref(p5), None, None, None, None) == 2
