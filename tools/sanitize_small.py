"""Small end-to-end run for compute-sanitizer: every kernel family once on c1 (16^2)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04559_b200 import configs as cf, stamg
spec = cf.baseline_config(1, 16)
g = stamg.Context(spec)
x = g.vec(data=np.random.default_rng(0).uniform(-1, 1, g.vec().n))
y = g.vec()
g.apply_L_into(x, y); g.apply_A_into(x, spec.N, y); g.standard_sweep(x, y)
g.apply_scatter_into(x, spec.N, 1.0, y)
z = g.mg_apply(x)
xs, rep = g.solve(g.rhs(), "gmres", "mg", max_iter=3, tol=1e-300)
xs, rep = g.solve(g.rhs(), "bicgstab", "sweep", max_iter=2, tol=1e-300)
spec5 = cf.baseline_config(5, 40); spec5.angular_level = 3; spec5.N = 11
spec5.moments = np.asarray(spec5.moments)[:, :12]
h = stamg.Context(spec5, build_hierarchy=False)  # folded scatter + source iteration
psi = h.vec().fill(1.0)
h.source_iteration(psi, 1)
g.synchronize(); h.synchronize()
print("sanitize run ok", rep["iterations"])
# coarse GS in its clustered multi-warp row kernel (DSMEM mailboxes, spin flags): c2 physics at 32^2
c2 = cf.baseline_config(2, 32)
g2 = stamg.Context(c2)
print("c2 32^2 coarse GS mode [mw, cluster, rows, slots, credit]:", g2.table("gs_mode", 0)[:5].tolist())
f0 = g2.vec(0).fill(1e-3)
phi0 = g2.vec(0)
g2.coarse_scatter_sweep(f0, 2, phi0, level=0)
g2.synchronize()
# sweep with two column blocks per group (XBLK: strip flags + L2 trace scratch): rank 0 of 8, 80^2
c5 = cf.baseline_config(5, 80)
g5 = stamg.Context(c5, build_hierarchy=False, rank=0, world=8, shard_probe=True)
v5 = g5.vec().fill(1.0)
g5.standard_sweep(v5, v5)
g5.standard_sweep(v5, v5)
g5.synchronize()
print("sanitize run (coarse GS cluster + XBLK sweep) ok")
