"""The oracle restatement pinned to the REFERENCE ITSELF.

tests/golden/ref_*.npz hold outputs of the reference's own solver sources
(/root/reference/proj/src, unmodified, compiled against the Eigen-subset shim
into oracle/_ref/; tests/golden/make_golden_ref.py) on the reference's kind of
problems: 3D hexahedra, uniform and banded angular meshes, Const and Lin
bases, p = 0 / 1, FP moments, uniform and beam sources. The oracle
(oracle/stamg_oracle.cpp) recomputes every operator on the same seeded inputs
and must agree to rounding; BiCGSTAB must take exactly the reference's
iterations. The GPU path is pinned to the oracle (tests/test_gpu_*.py), so
this closes the chain GPU -> oracle -> reference.

When the reference sources are present (this container), the live reference
is also rebuilt and checked against the committed fixtures, so the fixtures
are shown to be the reference's output.
"""
import os
import sys

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden_ref as MGR  # noqa: E402

OP_TOL = 1e-13
SOLVE_TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def oracle_for(orc, name):
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
    return orc.Oracle(spec), N


def load(name):
    return dict(np.load(os.path.join(HERE, "golden", f"{name}.npz")))


@pytest.mark.parametrize("name", sorted(MGR.CASES))
def test_oracle_matches_reference(orc, name):
    g = load(name)
    o, N = oracle_for(orc, name)
    assert tuple(o.layout()) == tuple(g["layout"])
    nlev, nr = o.levels()
    assert (nlev, nr) == tuple(g["levels"])
    x, y0, xc = MGR.inputs(o.size(), o.size(0))
    assert rel(o.X(), g["X"]) <= OP_TOL
    assert rel(o.rhs(), g["rhs"]) <= OP_TOL
    assert rel(o.apply_L(x), g["apply_L"]) <= OP_TOL
    assert rel(o.apply_A(x, N), g["apply_A"]) <= OP_TOL
    assert rel(o.apply_A(x, nr), g["apply_A_nr"]) <= OP_TOL
    assert rel(o.apply_scatter(x, N, -0.5, y=y0), g["scatter"]) <= OP_TOL
    assert rel(o.sweep(x), g["sweep"]) <= OP_TOL
    assert rel(o.coarse_gs(xc, 2, np.zeros_like(xc)), g["coarse_gs"]) <= OP_TOL
    assert rel(o.smoother(x, nr, y0, level=nlev - 1), g["smoother"]) <= OP_TOL
    assert rel(o.restrict(x, nlev - 1), g["restrict"]) <= OP_TOL
    assert rel(o.prolong(MGR.coarse_input(o.size(nlev - 2)), nlev - 1), g["prolong"]) <= OP_TOL
    assert rel(o.mg_apply(x), g["mg_apply"]) <= OP_TOL
    for pc in ("mg", "sweep"):
        xs, rep = o.solve("bicgstab", pc, tol=1e-10, max_iter=100)
        assert rep["iterations"] == int(g[f"bicgstab_{pc}_iterations"][0]), (pc, rep["iterations"])
        assert rel(xs, g[f"bicgstab_{pc}_x"]) <= SOLVE_TOL
        assert rel(rep["residual_history"], g[f"bicgstab_{pc}_history"]) <= 1e-6


def _live_reference_ok():
    try:
        import pyref
        return pyref.available()
    except Exception:  # noqa: BLE001
        return False


@pytest.mark.skipif(not _live_reference_ok(), reason="reference sources / oracle/_ref not present")
@pytest.mark.parametrize("name", sorted(MGR.CASES)[:2])
def test_fixtures_are_the_reference_output(name):
    """Rebuild the reference (oracle/_ref) and regenerate the fixture values:
    the committed vectors are the reference's own output."""
    g = load(name)
    live = MGR.run_reference(name)
    for key in ("X", "rhs", "apply_L", "apply_A", "sweep", "coarse_gs", "mg_apply", "bicgstab_mg_x"):
        assert rel(live[key], g[key]) <= 1e-15, key
    assert int(live["bicgstab_mg_iterations"][0]) == int(g["bicgstab_mg_iterations"][0])
