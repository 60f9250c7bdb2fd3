"""Device-side setup: build_couplings (scatter.cpp:74-99) and
build_operators (transport.cpp:43-57: patch mass / Jacobians by quadrature, fused blocks,
their inverses, inflow blocks) run on the GPU (csrc/couplings.cu). The tables must match
the host loops (STAMG_HOST_SETUP=1, the same quadrature, recurrence and block algebra on
one core) at the full BASELINE angular meshes, including config 4's mixed-level cone mesh,
config 3's two materials and every MG level, and the device path must be much faster."""
import os
import time

import numpy as np
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu


def make(stamg, spec, host, mg):
    if host:
        os.environ["STAMG_HOST_SETUP"] = "1"
    try:
        t0 = time.perf_counter()
        c = stamg.Context(spec, build_hierarchy=mg)
        return c, time.perf_counter() - t0
    finally:
        os.environ.pop("STAMG_HOST_SETUP", None)


@pytest.mark.parametrize("k,mg", [(5, False), (4, True), (3, True)], ids=["c5", "c4", "c3"])
def test_device_couplings_match_host(stamg, k, mg):
    spec = cf.baseline_config(k, 16 if k != 5 else 8)  # the grid does not enter X; keep vectors small
    d, td = make(stamg, spec, False, mg)
    h, th = make(stamg, spec, True, mg)
    try:
        levels = [stamg.OUTER] + (list(range(d.levels()[0])) if mg else [])
        for l in levels:
            a, b = d.table("X", l), h.table("X", l)
            assert a.shape == b.shape
            assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max(), l
            for name in ("B", "Binv", "C", "area"):  # build_operators on the device
                a, b = d.table(name, l), h.table(name, l)
                assert a.shape == b.shape
                assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max(), (name, l)
        print(f"c{k}: setup device {td:.3f} s, host {th:.3f} s")
        if k == 5:
            assert td < th
    finally:
        d.close()
        h.close()
