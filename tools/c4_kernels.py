"""Config-4 kernel rooflines alone (the bench's `kernels` section without the rest of the bench):
apply_L, sweep, scatter GEMMs, transfers. Usage: python tools/c4_kernels.py [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2010_04559_b200 import configs as cf  # noqa: E402
from paper_2010_04559_b200 import stamg  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    peak = 37.1
    for _ in range(reps):
        out = bench.kernel_rooflines(stamg, cf, peak)
        row = {k: (round(v["ms"], 3), round(v["frac"], 3)) for k, v in out.items() if isinstance(v, dict) and "ms" in v}
        print(json.dumps(row))
    # one smoother step on the finest MG level: per-class kernel time (apply_L here is the
    # y = f - L x form, the sweep the accumulating one)
    spec = cf.baseline_config(4)
    g = stamg.Context(spec)
    try:
        nlev, nr = g.levels()
        lf = nlev - 1
        f, phi = g.vec(lf).fill(1.0), g.vec(lf).fill(0.5)
        g.smoother_step(f, nr, phi, level=lf)
        g.synchronize()
        g.timing(True)
        g.smoother_step(f, nr, phi, level=lf)
        g.synchronize()
        print(json.dumps({"smoother_step_lf": {k: round(g.timed(k)[0], 3) for k in ("apply_L", "sweep", "d2m", "m2d")}}))
        g.timing(False)
    finally:
        g.close()


if __name__ == "__main__":
    main()
