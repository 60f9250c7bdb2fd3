"""Timing probe of the reference-shape path (3D, trilinear cells, Lin angular basis: 24 dofs per
(cell, patch)): per-operator time and the HBM bandwidth the algorithmic bytes correspond to."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04559_b200 import configs as cf, stamg
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import make_golden_ref as MGR

n = int(os.environ.get("GN", "24"))
level = int(os.environ.get("GLEVEL", "2"))
basis = int(os.environ.get("GBASIS", "1"))
p = int(os.environ.get("GP", "1"))
N = 8
m, st = MGR.fp_moments(N, 0.5, 0.1)
spec = cf.reference_test_problem(n, 1.0 * n / 8, level, basis, p, N, m, st, dim=3, q_el=np.ones(n ** 3), n_levels=0, nr=4)
t0 = time.perf_counter()
g = stamg.Context(spec)
setup = time.perf_counter() - t0
n_el, P, S, D = g.layout()
vec_bytes = n_el * P * S * D * 8


def timeit(fn, reps=5):
    fn(); g.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    g.synchronize()
    return (time.perf_counter() - t) / reps


x = g.vec().fill(1.0)
y = g.vec()
out = {"problem": f"{n}^3 cells, level {level} ({P} patches), S={S}, D={D}", "setup_s": setup, "vector_MB": vec_bytes / 1e6}
t = timeit(lambda: g.apply_L_into(x, y)); out["apply_L"] = {"ms": t * 1e3, "GBs": 2 * vec_bytes / t / 1e9}
t = timeit(lambda: g.standard_sweep(x, y)); out["sweep"] = {"ms": t * 1e3, "GBs": 2 * vec_bytes / t / 1e9, "updates_per_s": n_el * P / t}
t = timeit(lambda: g.apply_scatter_into(x, N, 1.0, y)); out["scatter_N8"] = {"ms": t * 1e3, "GBs": 3 * vec_bytes / t / 1e9,
                                                                             "gflops": 4 * (N + 1) ** 2 * P * D * S * n_el / t / 1e9}
f0 = g.vec(0).fill(1e-3); p0 = g.vec(0)
t = timeit(lambda: g.coarse_scatter_sweep(f0, 10, p0, level=0), reps=2); out["coarse_gs_10"] = {"ms": t * 1e3}
t = timeit(lambda: g.mg_apply(x, y), reps=2); out["mg_apply"] = {"ms": t * 1e3}
b = g.rhs()
t0 = time.perf_counter(); xs, rep = g.solve(b, "bicgstab", "mg", tol=1e-8, max_iter=100); g.synchronize()
out["bicgstab_mg"] = {"s": time.perf_counter() - t0, "iterations": rep["iterations"], "converged": rep["converged"]}
print(json.dumps(out))
