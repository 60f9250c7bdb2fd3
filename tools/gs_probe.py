"""Run the config-4 coarse Gauss-Seidel (one call, nu passes) for profiling."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04559_b200 import configs as cf, stamg
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nu = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
spec = cf.baseline_config(k, n)
g = stamg.Context(spec)
print("gs_mode (mw, cluster, rows, slots, credit, blocked chain):", [int(v) for v in g.table("gs_mode", 0)], flush=True)
f = g.vec(0).fill(1e-3)
phi = g.vec(0)
for rep in range(2):
    g.synchronize(); t = time.perf_counter()
    g.coarse_scatter_sweep(f, nu, phi, level=0)
    g.synchronize(); dt = time.perf_counter() - t
    nx = spec.nx
    print(f"c{k} n={nx} coarse_gs nu={nu}: {dt:.4f} s  ({dt / (nu * 12 * nx) * 1e6:.2f} us per critical-path item, 8 nx + 4 ny per pass)", flush=True)
g.close()
