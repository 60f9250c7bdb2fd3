"""One config-5 context (512^2 x 8192, wavefront layout) and N in-place sweeps:
the target of the full-size ncu --set full capture (DRAM bytes per launch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04559_b200 import configs as cf, stamg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = stamg.Context(cf.baseline_config(5), build_hierarchy=False)
psi = g.vec().fill(1.0)
for _ in range(n):
    g.standard_sweep(psi, psi)
g.synchronize()
print("sweeps done", g.layout())
