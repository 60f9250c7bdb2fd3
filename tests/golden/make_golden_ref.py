"""Golden vectors from the REFERENCE ITSELF (not the oracle).

The reference's solver sources (/root/reference/proj/src/*.cpp, unmodified)
are compiled against the Eigen-subset shim into oracle/_ref/libstamgref.so
(`make -C oracle ref`, oracle/ref_capi.cpp) and run on the reference's own
kind of problems: 3D hexahedral grids, uniform and banded angular meshes,
Const and Lin angular bases, p = 0 / 1, Fokker-Planck-equivalent moments
(scatter.cpp:9-21), uniform and +z beam sources. For seeded inputs the script
records every hot-path operator's output and the BiCGSTAB solves
(harness.cpp:211-231 closures, sweep and MG preconditioners).
tests/test_oracle_vs_reference.py re-runs the oracle restatement on the same
inputs and compares -- this pins the oracle (and through it the GPU path, which
is pinned to the oracle) to the reference.

Run (in the container that has /root/reference):  python tests/golden/make_golden_ref.py
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

# name: (n, box, level, basis, p, N, alpha, sigma_a, banded, beam)
CASES = {
    "ref_const_p0_l1": (3, 3.0, 1, 0, 0, 4, 1.0, 0.3, False, None),
    "ref_lin_p1_l1": (2, 2.0, 1, 1, 1, 4, 1.0, 0.3, False, None),
    "ref_const_p1_l2": (2, 1.0, 2, 0, 1, 8, 0.5, 0.1, False, None),
    "ref_lin_p1_banded3_beam": (2, 1.0, 3, 1, 1, 8, 0.5, 0.1, True, (0.2, 0.7, 0.3, 0.8)),
}
SEED = 2010


def fp_moments(N, alpha, sigma_a):
    """scatter.cpp:9-21 (the reference computes the same inside ref_create's caller)."""
    n = np.arange(N + 1, dtype=np.float64)
    m = 0.5 * alpha * (N * (N + 1.0) - n * (n + 1.0))
    return m, sigma_a + m[0]


def inputs(size_fine, size_coarse, seed=SEED):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size_fine), rng.uniform(-1.0, 1.0, size_fine), rng.uniform(-1.0, 1.0, size_coarse)


def coarse_input(size):
    return np.random.default_rng(SEED + 7).uniform(-1.0, 1.0, size)


def run_reference(name):
    import pyref
    n, box, level, basis, p, N, alpha, sa, banded, beam = CASES[name]
    m, st = fp_moments(N, alpha, sa)
    r = pyref.Reference(n, box, level, basis, p, N, m, st, sa, banded=banded, beam=beam)
    nlev, nr = r.levels()
    x, y0, xc = inputs(r.size(), r.size(0))
    out = {"layout": np.array(r.layout()), "levels": np.array([nlev, nr]), "X": r.X(), "rhs": r.rhs(),
           "apply_L": r.apply_L(x), "apply_A": r.apply_A(x, N), "apply_A_nr": r.apply_A(x, nr),
           "scatter": r.apply_scatter(x, N, -0.5, y=y0), "sweep": r.sweep(x),
           "coarse_gs": r.coarse_gs(xc, 2, np.zeros_like(xc)),
           "smoother": r.smoother(x, nr, y0, level=nlev - 1),
           "restrict": r.restrict(x, nlev - 1), "prolong": r.prolong(coarse_input(r.size(nlev - 2)), nlev - 1),
           "mg_apply": r.mg_apply(x)}
    for pc in ("mg", "sweep"):
        xs, rep = r.bicgstab(pc, tol=1e-10, max_iter=100)
        out[f"bicgstab_{pc}_x"] = xs
        out[f"bicgstab_{pc}_iterations"] = np.array([rep["iterations"]])
        out[f"bicgstab_{pc}_history"] = rep["residual_history"]
    return out


def main(which):
    for name in CASES:
        if which and name not in which:
            continue
        t0 = time.time()
        out = run_reference(name)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, tuple(out["layout"]), int(out["bicgstab_mg_iterations"][0]), f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
