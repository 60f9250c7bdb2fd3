"""The B200 path against the REFERENCE ITSELF on the reference's own kind of problems.

tests/golden/ref_*.npz hold outputs of the reference's unmodified solver sources
(tests/golden/make_golden_ref.py: 3D hexahedra, uniform and banded angular meshes, Const
and Lin angular bases, p = 0 / 1, Fokker-Planck-equivalent moments, uniform and +z beam
sources). These discretisations run on the library's reference-shape path
(csrc/generic*.{hpp,cpp,cu}; angular_disc.cpp:40-59,
spatial_disc.cpp:45-88). Every hot-path operator is compared on the same seeded inputs
through the C ABI; BiCGSTAB must take the reference's iteration count (+-1) and reach the
same solution. Tolerances: operators 1e-12 relative L2 (the library applies precomputed
block inverses where the reference solves with a pivoted LU), solves 1e-9.
"""
import os
import sys

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden_ref as MGR  # noqa: E402

pytestmark = pytest.mark.gpu
OP_TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def spec_for(name):
    n, box, level, basis, p, N, alpha, sa, banded, beam = MGR.CASES[name]
    m, st = MGR.fp_moments(N, alpha, sa)
    kw = dict(n_levels=0)
    if beam is not None:
        kw.update(beam=cf.BEAM_PENCIL_Z, x0=beam[0], x1=beam[1], y0=beam[2], y1=beam[3])
    else:
        kw.update(q_el=np.ones(n ** 3))
    spec = cf.reference_test_problem(n, box, level, basis, p, N, m, st, dim=3, **kw)
    if banded:
        spec.angular_kind = cf.ANGULAR_BANDED
    return spec, N


@pytest.fixture(scope="module", params=sorted(MGR.CASES))
def case(request, stamg):
    name = request.param
    g = dict(np.load(os.path.join(HERE, "golden", f"{name}.npz")))
    spec, N = spec_for(name)
    c = stamg.Context(spec)
    yield name, c, g, N
    c.close()


def test_layout_and_tables(case):
    name, c, g, N = case
    assert tuple(c.layout()) == tuple(g["layout"])
    nlev, nr = c.levels()
    assert (nlev, nr) == tuple(g["levels"])
    n_el, P, S, D = c.layout()
    assert rel(c.table("X").reshape(P * D, -1), g["X"]) <= 1e-13
    assert rel(c.rhs().numpy(), g["rhs"]) <= 1e-13


def test_operators(case):
    name, c, g, N = case
    nlev, nr = c.levels()
    x, y0, xc = MGR.inputs(c.vec().n, c.vec(0).n)
    xv = c.vec(data=x)
    y = c.vec()
    c.apply_L_into(xv, y)
    assert rel(y.numpy(), g["apply_L"]) <= OP_TOL
    c.apply_A_into(xv, N, y)
    assert rel(y.numpy(), g["apply_A"]) <= OP_TOL
    c.apply_A_into(xv, nr, y)
    assert rel(y.numpy(), g["apply_A_nr"]) <= OP_TOL
    y.upload(y0)
    c.apply_scatter_into(xv, N, -0.5, y)
    assert rel(y.numpy(), g["scatter"]) <= OP_TOL
    c.standard_sweep(xv, y)
    assert rel(y.numpy(), g["sweep"]) <= OP_TOL
    z = c.vec(data=x)
    c.standard_sweep(z, z)  # aliasing allowed (sweeps.hpp:24)
    assert np.array_equal(z.numpy(), y.numpy())


def test_multigrid_components(case):
    name, c, g, N = case
    nlev, nr = c.levels()
    x, y0, xc = MGR.inputs(c.vec().n, c.vec(0).n)
    phi = c.vec(0)
    c.coarse_scatter_sweep(c.vec(0, xc), 2, phi, level=0)
    assert rel(phi.numpy(), g["coarse_gs"]) <= 1e-11
    top = nlev - 1
    ph = c.vec(top, y0)
    c.smoother_step(c.vec(top, x), nr, ph, level=top)
    assert rel(ph.numpy(), g["smoother"]) <= OP_TOL
    r = c.restrict_residual(top, c.vec(top, x))
    assert rel(r.numpy(), g["restrict"]) <= 1e-14
    pc = c.prolongate(top, c.vec(top - 1, MGR.coarse_input(c.vec(top - 1).n)))
    assert rel(pc.numpy(), g["prolong"]) <= 1e-14
    z = c.mg_apply(c.vec(top, x))
    assert rel(z.numpy(), g["mg_apply"]) <= 1e-11
    z2 = c.mg_apply(c.vec(top, x))
    assert np.array_equal(z.numpy(), z2.numpy())


@pytest.mark.parametrize("pc", ["mg", "sweep"])
def test_bicgstab(case, pc):
    name, c, g, N = case
    b = c.rhs()
    xs, rep = c.solve(b, "bicgstab", pc, tol=1e-10, max_iter=100)
    assert rep["converged"]
    assert abs(rep["iterations"] - int(g[f"bicgstab_{pc}_iterations"][0])) <= 1, (pc, rep["iterations"])
    assert rel(xs.numpy(), g[f"bicgstab_{pc}_x"]) <= 1e-9
    k = min(len(rep["residual_history"]), len(g[f"bicgstab_{pc}_history"]), 5)
    assert rel(rep["residual_history"][:k], g[f"bicgstab_{pc}_history"][:k]) <= 1e-6


def test_gmres_matches_bicgstab_solution(case):
    name, c, g, N = case
    xs, rep = c.solve(c.rhs(), "gmres", "mg", tol=1e-10, max_iter=100, restart=30)
    assert rep["converged"]
    assert rel(xs.numpy(), g["bicgstab_mg_x"]) <= 1e-8
    sf = c.scalar_flux(xs)
    assert np.all(np.isfinite(sf)) and sf.shape == (c.layout()[0],)


def test_host_buffer_entry_points(case, stamg):
    """The FFI boundary a reference maintainer binds: host buffers in, host buffers
    out, for the reference's own discretisations too."""
    name, c, g, N = case
    x, _, _ = MGR.inputs(c.vec().n, c.vec(0).n)
    z = np.empty_like(x)
    c.sweep_host(np.ascontiguousarray(x), z)
    assert rel(z, g["sweep"]) <= OP_TOL
    b = c.rhs().numpy()
    xs = np.zeros_like(b)
    rep = c.solve_host(np.ascontiguousarray(b), xs, method="bicgstab", precond="mg", tol=1e-10, max_iter=100)
    assert rep["converged"]
    assert abs(rep["iterations"] - int(g["bicgstab_mg_iterations"][0])) <= 1
    assert rel(xs, g["bicgstab_mg_x"]) <= 1e-9
