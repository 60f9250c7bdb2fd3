"""Config 4 on its production kernels against the oracle: 64^2 cells on the
full 2888-patch cone mesh (tests/golden/make_golden_c4n64.py).

At 64^2 the kernels the 256^2 solve runs are the ones engaged -- padded
8-direction sweep groups, the row-walk apply_L (nx >= 38) and the row-mode
coarse Gauss-Seidel (nx >= 64) -- unlike the 8^2 fixture, which exercises the
4-direction small-grid variants. Each operator output is compared through its
two projections (sums over directions per (cell, dof), sums over cells per
(direction, dof)), a strided sample and its norm. Solve: GMRES(12) + V(1,1)
angular MG, equal-k flux <= 1e-10 relative L2 and the iteration count at tol
1e-8 within +-1 (BASELINE.json north_star). References: sweeps.cpp:20-104,
transport.cpp:66-101, scatter.cpp:110-135, multigrid.cpp:138-176.
"""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden_c4n64 as G  # noqa: E402

pytestmark = pytest.mark.gpu
FIX = os.path.join(HERE, "golden", "c4n64.npz")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def ctx(stamg):
    if not os.path.exists(FIX):
        pytest.fail("tests/golden/c4n64.npz missing: run tests/golden/make_golden_c4n64.py")
    g = np.load(FIX)
    c = stamg.Context(G.spec())
    yield c, g
    c.close()


def check(g, name, v, P, tol):
    n_el = int(g["n_el"][0])
    cs, ds = G.projections(v, n_el, P)
    assert rel(cs, g[f"{name}_cellsum"]) <= tol, (name, "cellsum", rel(cs, g[f"{name}_cellsum"]))
    assert rel(ds, g[f"{name}_dirsum"]) <= tol, (name, "dirsum", rel(ds, g[f"{name}_dirsum"]))
    st = int(g["stride"][0])
    assert rel(v[::st], g[f"{name}_sample"]) <= tol, (name, "sample")
    assert abs(np.linalg.norm(v) - g[f"{name}_norm"][0]) <= tol * g[f"{name}_norm"][0]


def test_production_kernels_engaged(ctx):
    c, g = ctx
    n_el, P, _, _ = c.layout()
    assert (n_el, P) == (int(g["n_el"][0]), int(g["n_patch"][0])) == (4096, 2888)
    assert c.levels()[0] == int(g["n_levels"][0])
    assert c.layout(0)[1] == int(g["coarse_patches"][0])
    mw, cluster, rows, _, _ = c.table("gs_mode", 0)[:5]
    assert mw == 1 or rows > 0  # row-CTA (multi-warp) or row-mode coarse GS, not the segment kernel


def test_operators(ctx):
    c, g = ctx
    n_el, P, _, _ = c.layout()
    x, xc = G.inputs(n_el * P * 4, c.layout(0)[0] * c.layout(0)[1] * 4)
    xv = c.vec(data=x)
    y = c.vec()
    c.apply_L_into(xv, y)
    check(g, "apply_L", y.numpy(), P, 1e-13)
    c.standard_sweep(xv, y)
    check(g, "sweep", y.numpy(), P, 1e-12)
    c.apply_A_into(xv, c.spec.N, y)
    check(g, "apply_A", y.numpy(), P, 1e-13)
    if "coarse_gs_cellsum" in g:
        phi = c.vec(level=0)
        c.coarse_scatter_sweep(c.vec(level=0, data=xc), 1, phi, level=0)
        check(g, "coarse_gs", phi.numpy(), c.layout(0)[1], 1e-11)
    if "mg_apply_cellsum" in g:
        z = c.mg_apply(xv)
        check(g, "mg_apply", z.numpy(), P, 1e-11)


def test_solve(ctx):
    c, g = ctx
    if "fixed_k" not in g:
        pytest.fail("fixture has no solve stage yet")
    b = c.rhs()
    kfix = int(g["fixed_k"][0])
    xk, repk = c.solve(b, "gmres", "mg", tol=1e-300, max_iter=kfix)
    assert repk["iterations"] == kfix
    assert rel(c.scalar_flux(xk), g["fixed_scalar_flux"]) <= 1e-10
    a = xk.numpy()
    assert rel(a[::int(g["stride"][0])], g["fixed_angular_sample"]) <= 1e-10
    assert abs(np.linalg.norm(a) - g["fixed_angular_norm"][0]) <= 1e-10 * g["fixed_angular_norm"][0]
    if "solve_iterations" in g:
        xs, rep = c.solve(b, "gmres", "mg")
        assert rep["converged"]
        assert abs(rep["iterations"] - int(g["solve_iterations"][0])) <= 1, (rep["iterations"], g["solve_iterations"])
        assert rel(c.scalar_flux(xs), g["solve_scalar_flux"]) < 1e-7
