"""Full-BASELINE-size solve fixtures from the CPU oracle (oracle/).

For configs 1-3 at their BASELINE.json grids (32^2, 64^2, 128^2) the oracle
runs GMRES + V(1,1) angular MG (a) to tol 1e-8, recording the iteration count
and the scalar flux, and (b) for exactly K_FIXED iterations (tol 0), recording
the scalar flux and a strided sample of the angular flux. The GPU test
(tests/test_gpu_fullsize_golden.py) compares (a) within +-1 iteration and (b)
at <= 1e-10 relative L2 (SURVEY §8(d) parity (ii)/(iii)) without the oracle
at run time. Configs 4 and 5 are beyond the oracle's reach in minutes (c4:
~3 TFLOP per outer apply_A on the host; c5 has no solve) and are covered by
size-independent properties instead (tests/test_gpu_fullsize.py).

Run: python tests/golden/make_golden_full.py [config ...]   (c3 takes minutes)
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402
from paper_2010_04559_b200 import configs as cf  # noqa: E402

CASES = {"c1full": 1, "c2full": 2, "c3full": 3}
K_FIXED = 6
STRIDE = {1: 97, 2: 97, 3: 970}  # angular-flux sample stride (keeps each fixture under 1 MB)


def main(which):
    for name, k in CASES.items():
        if which and str(k) not in which:
            continue
        spec = cf.baseline_config(k)
        t0 = time.time()
        o = pyoracle.Oracle(spec)
        xs, rep = o.solve("gmres", "mg")
        xk, repk = o.solve("gmres", "mg", tol=1e-300, max_iter=K_FIXED)
        out = dict(
            solve_iterations=np.array([rep["iterations"]]),
            solve_final_residual=np.array([rep["final_residual"]]),
            solve_scalar_flux=o.scalar_flux(xs),
            fixed_k=np.array([K_FIXED]),
            fixed_scalar_flux=o.scalar_flux(xk),
            fixed_angular_sample=xk[::STRIDE[k]].copy(),
            sample_stride=np.array([STRIDE[k]]),
            fixed_angular_norm=np.array([np.linalg.norm(xk)]),
        )
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, o.size(), rep["iterations"], rep["final_residual"], f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
