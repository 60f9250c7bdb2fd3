"""Committed golden fixtures (tests/golden/, made by make_golden.py from the
oracle): the oracle must reproduce them (CPU), and the GPU path must match them
(-m gpu) without needing the oracle at run time."""
import os
import sys

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden as MG  # noqa: E402

CASES = sorted(MG.CASES.items())


def compare(g, key, v, rtol):
    if key in g:
        ref = g[key]
        assert np.linalg.norm(v - ref) <= rtol * max(np.linalg.norm(ref), 1e-300), key
    else:
        s, nrm = g[key + "_sample"], g[key + "_norm"][0]
        assert np.linalg.norm(v[::MG.SAMPLE] - s) <= rtol * max(np.linalg.norm(s), 1e-300), key
        assert abs(np.linalg.norm(v) - nrm) <= rtol * nrm, key


@pytest.mark.parametrize("name,case", CASES)
def test_oracle_reproduces_golden(orc, name, case):
    k, n = case
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    spec = cf.baseline_config(k, n)
    o = orc.Oracle(spec)
    x = MG.seeded_input(k, o.size())
    compare(g, "sweep", o.sweep(x), 1e-13)
    compare(g, "apply_A", o.apply_A(x, spec.N), 1e-13)
    compare(g, "rhs", o.rhs(), 1e-15)
    if name in MG.THROUGHPUT:
        compare(g, "source_iteration", o.sweep(o.rhs() + o.apply_scatter(np.abs(x), spec.N, 1.0)), 1e-13)
    else:
        compare(g, "mg_apply", o.mg_apply(x), 1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", CASES)
def test_gpu_matches_golden(stamg, name, case):
    k, n = case
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    spec = cf.baseline_config(k, n)
    throughput = name in MG.THROUGHPUT
    c = stamg.Context(spec, build_hierarchy=not throughput)
    size = c.vec().n
    x = MG.seeded_input(k, size)
    xv = c.vec(data=x)
    y = c.vec()
    c.apply_L_into(xv, y)
    compare(g, "apply_L", y.numpy(), 1e-13)
    c.apply_A_into(xv, spec.N, y)
    compare(g, "apply_A", y.numpy(), 1e-13)
    y.fill(0.0)
    c.apply_scatter_into(xv, spec.N, 1.0, y)
    compare(g, "scatter_full", y.numpy(), 1e-12)
    c.standard_sweep(xv, y)
    compare(g, "sweep", y.numpy(), 1e-12)
    compare(g, "rhs", c.rhs().numpy(), 1e-14)
    if throughput:  # hierarchy-free context: wavefront layout, folded scatter
        psi = c.vec(data=np.abs(x))
        c.source_iteration(psi, 1)
        compare(g, "source_iteration", psi.numpy(), 1e-12)
        return
    compare(g, "mg_apply", c.mg_apply(xv).numpy(), 1e-11)
    phi0 = c.vec(0)
    c.coarse_scatter_sweep(c.vec(0, MG.seeded_coarse(k, phi0.n)), 1, phi0, level=0)
    compare(g, "coarse_gs_nu1", phi0.numpy(), 1e-11)
    xs, rep = c.solve(c.rhs(), "gmres", "mg")
    assert abs(rep["iterations"] - int(g["solve_iterations"][0])) <= 1
    compare(g, "solve_scalar_flux", c.scalar_flux(xs), 1e-7)
