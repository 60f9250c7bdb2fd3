"""Generate the committed golden fixtures from the CPU oracle (oracle/).

The reference cannot be built here (Eigen3 absent), so these vectors come from
the restated oracle, itself pinned by the reference's own unit-test identities
(tests/test_oracle_reference.py). They freeze small, seeded cases of every hot
operator so a regression in either the oracle or the GPU path is caught without
re-deriving anything. Run: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402
from paper_2010_04559_b200 import configs as cf  # noqa: E402

CASES = {"c1n8": (1, 8), "c2n8": (2, 8), "c3n8": (3, 8), "c4n8": (4, 8), "c5n8": (5, 8)}
# configs whose BASELINE entry is a throughput workload (no MG hierarchy, no
# solve): frozen operators plus one source iteration at the full angular mesh
THROUGHPUT = {"c5n8"}
SAMPLE = 61  # larger cases keep every 61st entry plus the L2 norm of each vector


def seeded_input(k, size):
    return np.random.default_rng(1000 + k).uniform(-1, 1, size)


def seeded_coarse(k, size):
    return np.random.default_rng(2000 + k).uniform(-1, 1, size)


def throughput_case(o, spec, x):
    """Operators of a hierarchy-free context and one source iteration
    psi <- L^-1 (q + S psi) (sweeps.cpp:106-113 with the full-order kernel)."""
    return dict(
        apply_L=o.apply_L(x),
        apply_A=o.apply_A(x, spec.N),
        scatter_full=o.apply_scatter(x, spec.N, 1.0),
        sweep=o.sweep(x),
        rhs=o.rhs(),
        source_iteration=o.sweep(o.rhs() + o.apply_scatter(np.abs(x), spec.N, 1.0)),
    )


def main(only=None):
    for name, (k, n) in CASES.items():
        if only and name not in only:
            continue
        spec = cf.baseline_config(k, n)
        o = pyoracle.Oracle(spec)
        size = o.size()
        x = seeded_input(k, size)
        if name in THROUGHPUT:
            full, rep = throughput_case(o, spec, x), {"iterations": "-"}
        else:
            full, rep = solve_case(o, spec, k, x)
        out = {}
        for key, v in full.items():
            v = np.asarray(v, dtype=np.float64)
            if key.startswith("solve"):
                out[key] = v
            elif name == "c1n8" and key in ("sweep", "apply_A"):
                out[key] = v
            else:
                out[key + "_sample"] = v[::SAMPLE]
                out[key + "_norm"] = np.array([np.linalg.norm(v)])
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, size, rep["iterations"])


def solve_case(o, spec, k, x):
    xs, rep = o.solve("gmres", "mg")
    return dict(
        apply_L=o.apply_L(x),
        apply_A=o.apply_A(x, spec.N),
        scatter_full=o.apply_scatter(x, spec.N, 1.0),
        sweep=o.sweep(x),
        mg_apply=o.mg_apply(x),
        rhs=o.rhs(),
        solve_scalar_flux=o.scalar_flux(xs),
        solve_iterations=np.array([rep["iterations"]]),
        coarse_gs_nu1=o.coarse_gs(seeded_coarse(k, o.size(0)), 1, np.zeros(o.size(0)), level=0),
    ), rep


if __name__ == "__main__":
    main(sys.argv[1:] or None)
