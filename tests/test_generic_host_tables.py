"""Host setup of the reference-shape path (csrc/generic_setup.cpp: 3D hexahedra, p0 / trilinear
cells, Const / Lin angular bases) against tables produced by the REFERENCE ITSELF
(tests/golden/ref_*.npz, made by tests/golden/make_golden_ref.py from the reference's unmodified
sources). Host only: runs without a GPU through stamg_host_table.
References: scatter.cpp:74-99 (X), transport.cpp:23-64 (blocks), transport.cpp:110-179 (rhs).
"""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden_ref as MGR  # noqa: E402
from test_gpu_reference_parity import spec_for, rel  # noqa: E402


@pytest.mark.parametrize("name", sorted(MGR.CASES))
def test_host_tables_match_the_reference(stamg, name):
    g = dict(np.load(os.path.join(HERE, "golden", f"{name}.npz")))
    spec, N = spec_for(name)
    n_el, P, S, D = (int(v) for v in stamg.host_table(spec, "layout"))
    assert (n_el, P, S, D) == tuple(g["layout"])
    X = stamg.host_table(spec, "X").reshape(P * D, -1)
    assert rel(X, g["X"]) <= 1e-13
    assert rel(stamg.host_table(spec, "rhs"), g["rhs"]) <= 1e-13


@pytest.mark.parametrize("name", sorted(MGR.CASES))
def test_host_blocks_reproduce_apply_L(stamg, name):
    """y = B x + sum C x_up assembled in numpy from the host blocks equals the reference's apply_L."""
    g = dict(np.load(os.path.join(HERE, "golden", f"{name}.npz")))
    spec, N = spec_for(name)
    n_el, P, S, D = (int(v) for v in stamg.host_table(spec, "layout"))
    bs = S * D
    B = stamg.host_table(spec, "B").reshape(P, bs, bs)
    C = stamg.host_table(spec, "C").reshape(P, 3, bs, bs)
    x, _, _ = MGR.inputs(n_el * P * bs, 1)
    xv = x.reshape(n_el, P, bs)
    y = np.einsum("qab,eqb->eqa", B, xv)
    octant = stamg.host_table(spec, "octant").astype(int)
    n = spec.nx
    ref = g["apply_L"].reshape(n_el, P, bs)
    idx = np.arange(n_el).reshape(n, n, n)  # [iz][iy][ix]
    for q in range(P):
        for xi in range(3):
            # positive cosine: inflow through the low face, i.e. from the neighbour at -1
            direction = 1 if (octant[q] >> xi) & 1 else -1
            up = np.roll(idx, -direction, axis=2 - xi)
            valid = np.ones((n, n, n), dtype=bool)
            sl = [slice(None)] * 3
            sl[2 - xi] = 0 if direction == -1 else n - 1
            valid[tuple(sl)] = False
            y[idx[valid], q, :] += xv[up[valid], q, :] @ C[q, xi].T
    assert rel(y, ref) <= 1e-12
