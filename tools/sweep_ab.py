"""Time the config-5 in-place sweep (512^2 x 8192, wavefront layout) for A/B runs of
build or environment variants: prints ms per sweep (best and mean of `reps`)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_04559_b200 import configs as cf, stamg
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(os.environ.get("C5N", "512"))
g = stamg.Context(cf.baseline_config(5, n), build_hierarchy=False)
psi = g.vec().fill(1.0)
for _ in range(3):
    g.standard_sweep(psi, psi)
g.synchronize()
ts = []
for _ in range(reps):
    g.synchronize(); t = time.perf_counter()
    g.standard_sweep(psi, psi)
    g.synchronize(); ts.append(time.perf_counter() - t)
n_el, P, _, _ = g.layout()
best, mean = min(ts), sum(ts) / len(ts)
print(f"sweep n={n} xb={os.environ.get('STAMG_SWEEP_XB', 'auto')} lib={os.environ.get('STAMG_LIB', 'default')}: "
      f"best {best*1e3:.3f} ms mean {mean*1e3:.3f} ms  {n_el*P*64/best/1e9:.0f} GB/s best")
