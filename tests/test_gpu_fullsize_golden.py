"""Solve parity at the full BASELINE.json sizes of configs 1-3 against committed
oracle fixtures (tests/golden/make_golden_full.py): GMRES + V(1,1) angular MG
to tol 1e-8 within +-1 iteration of the oracle, and after a fixed number of
iterations the scalar flux and the angular flux at <= 1e-10 relative L2
(SURVEY.md §8(d) parity (ii), (iii))."""
import os
import sys

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden_full as MGF  # noqa: E402

CASES = [(name, k) for name, k in sorted(MGF.CASES.items())
         if os.path.exists(os.path.join(HERE, "golden", f"{name}.npz"))]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_fixtures_present():
    assert len(CASES) == len(MGF.CASES), "run tests/golden/make_golden_full.py"


def test_oracle_reproduces_c1_full(orc):
    """The CPU side of the pin: the oracle regenerates the config-1 fixture
    (configs 2-3 take minutes; their fixtures come from the same script)."""
    g = np.load(os.path.join(HERE, "golden", "c1full.npz"))
    o = orc.Oracle(cf.baseline_config(1))
    xk, rep = o.solve("gmres", "mg", tol=1e-300, max_iter=int(g["fixed_k"][0]))
    assert rel(o.scalar_flux(xk), g["fixed_scalar_flux"]) <= 1e-13
    assert rel(xk[::int(g["sample_stride"][0])], g["fixed_angular_sample"]) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("name,k", CASES)
def test_gpu_solve_matches_full_size_oracle(stamg, name, k):
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    spec = cf.baseline_config(k)
    c = stamg.Context(spec)
    try:
        b = c.rhs()
        xs, rep = c.solve(b, "gmres", "mg")
        assert rep["converged"]
        assert abs(rep["iterations"] - int(g["solve_iterations"][0])) <= 1, (rep["iterations"], g["solve_iterations"])
        assert rel(c.scalar_flux(xs), g["solve_scalar_flux"]) < 1e-7
        kfix = int(g["fixed_k"][0])
        xk, repk = c.solve(b, "gmres", "mg", tol=1e-300, max_iter=kfix)
        assert repk["iterations"] == kfix
        assert rel(c.scalar_flux(xk), g["fixed_scalar_flux"]) <= 1e-10
        a = xk.numpy()
        assert rel(a[::int(g["sample_stride"][0])], g["fixed_angular_sample"]) <= 1e-10
        assert abs(np.linalg.norm(a) - g["fixed_angular_norm"][0]) <= 1e-10 * g["fixed_angular_norm"][0]
    finally:
        c.close()
