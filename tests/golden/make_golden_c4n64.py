"""Config-4 oracle fixture at 64^2 cells on the full 2888-patch cone mesh.

At 64^2 the production config-4 kernels engage (padded 8-direction sweep
groups and the row-walk apply_L need nx >= 38, the row-mode coarse
Gauss-Seidel needs nx >= 64), so this fixture pins the kernels the 256^2
solve runs, not the 4-direction small-grid variants the 8^2 fixture sees.

Recorded (ORACLE output, CPU restatement of the reference; see oracle/):
  * operator level, on x = default_rng(SEED).uniform(-1, 1, n) (and a
    coarsest-level vector from SEED+1): apply_L, standard_sweep, outer
    apply_A at full order N = 32, one coarse_scatter_sweep pass (nu = 1, phi
    from zero) on the coarsest level, mg_apply.  Each output is stored as two
    projections that together touch every entry -- per (cell, dof) sums over
    the directions and per (direction, dof) sums over the cells -- plus a
    strided sample and the 2-norm (the full vectors are 378 MB each).
  * solve level: GMRES(12) + V(1,1) angular MG for exactly K_FIXED
    iterations (scalar flux, angular sample, norm) and to tol 1e-8
    (iteration count, scalar flux).  References: sweeps.cpp:20-104,
    transport.cpp:66-101, scatter.cpp:110-135, multigrid.cpp:138-176.

Run: OMP_NUM_THREADS=8 python tests/golden/make_golden_c4n64.py   (~1 h)
The npz is rewritten after every stage, so a partial run still pins the
finished stages (the GPU test checks whichever keys are present);
`--solve-only` keeps the stages already in the npz and adds the solve to 1e-8.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2010_04559_b200 import configs as cf  # noqa: E402

NAME = "c4n64"
N_CELLS = 64
SEED = 4064
K_FIXED = 6
STRIDE = 9697
OUT = os.path.join(HERE, f"{NAME}.npz")


def spec():
    return cf.baseline_config(4, N_CELLS)


def inputs(n_fine, n_coarse):
    x = np.random.default_rng(SEED).uniform(-1.0, 1.0, n_fine)
    xc = np.random.default_rng(SEED + 1).uniform(-1.0, 1.0, n_coarse)
    return x, xc


def projections(v, n_el, P):
    """(cell, dof) sums over directions, (direction, dof) sums over cells."""
    a = np.asarray(v).reshape(n_el, P, 4)
    return a.sum(axis=1), a.sum(axis=0)


def main():
    import pyoracle
    s = spec()
    t00 = time.time()
    o = pyoracle.Oracle(s)
    n_el, P, _, _ = o.layout()
    nlev, _ = o.levels()
    Pc = o.layout(0)[1]
    x, xc = inputs(o.size(), o.size(0))
    out = {"n_el": np.array([n_el]), "n_patch": np.array([P]), "n_levels": np.array([nlev]),
           "coarse_patches": np.array([Pc]), "seed": np.array([SEED]), "stride": np.array([STRIDE])}
    solve_only = "--solve-only" in sys.argv and os.path.exists(OUT)
    if solve_only:
        out = dict(np.load(OUT))

    def put(name, v, layout_P):
        cs, ds = projections(v, n_el, layout_P)
        out[f"{name}_cellsum"] = cs
        out[f"{name}_dirsum"] = ds
        out[f"{name}_sample"] = np.asarray(v)[::STRIDE].copy()
        out[f"{name}_norm"] = np.array([np.linalg.norm(v)])
        np.savez_compressed(OUT, **out)
        print(f"{name}: {time.time() - t00:.0f}s", flush=True)

    if not solve_only:
        operator_and_fixed_k_stages(o, s, x, xc, out, put, P, Pc)
    xs, rep = o.solve("gmres", "mg")
    out["solve_iterations"] = np.array([rep["iterations"]])
    out["solve_final_residual"] = np.array([rep["final_residual"]])
    out["solve_scalar_flux"] = o.scalar_flux(xs)
    np.savez_compressed(OUT, **out)
    print(f"solve: {rep['iterations']} iterations, residual {rep['final_residual']:.3e}, "
          f"{time.time() - t00:.0f}s", flush=True)


def operator_and_fixed_k_stages(o, s, x, xc, out, put, P, Pc):
    t00 = time.time()
    put("apply_L", o.apply_L(x), P)
    put("sweep", o.sweep(x), P)
    put("apply_A", o.apply_A(x, s.N), P)
    put("coarse_gs", o.coarse_gs(xc, 1, np.zeros_like(xc), level=0), Pc)
    put("mg_apply", o.mg_apply(x), P)
    b = o.rhs()
    xk, repk = o.solve("gmres", "mg", tol=1e-300, max_iter=K_FIXED)
    out["fixed_k"] = np.array([K_FIXED])
    out["fixed_scalar_flux"] = o.scalar_flux(xk)
    out["fixed_angular_sample"] = xk[::STRIDE].copy()
    out["fixed_angular_norm"] = np.array([np.linalg.norm(xk)])
    out["rhs_norm"] = np.array([np.linalg.norm(b)])
    np.savez_compressed(OUT, **out)
    print(f"fixed-k solve: {time.time() - t00:.0f}s", flush=True)


if __name__ == "__main__":
    main()
