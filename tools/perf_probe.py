"""Quick per-kernel timing probe on the GPU (development aid, not the bench)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2010_04559_b200 import configs as cf  # noqa: E402
from paper_2010_04559_b200 import stamg  # noqa: E402

HBM = 6455.3e9


def timeit(ctx, fn, reps=5):
    fn()
    ctx.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    ctx.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    out = {}
    which = sys.argv[1:] or ["c5s", "c2", "c3"]
    if "c5s" in which:
        spec = cf.baseline_config(5, int(os.environ.get("C5N", "128")))
        g = stamg.Context(spec, build_hierarchy=False)
        n_el, P, _, _ = g.layout()
        x = g.vec().fill(1.0)
        y = g.vec()
        upd = n_el * P
        t = timeit(g, lambda: g.standard_sweep(x, x))
        out["c5s_sweep"] = {"s": t, "upd_per_s": upd / t, "hbm_frac": upd * 64 / t / HBM}
        t = timeit(g, lambda: g.apply_L_into(x, y))
        out["c5s_apply_L"] = {"s": t, "hbm_frac": upd * 64 / t / HBM}
        g.timing(True)
        g.apply_scatter_into(x, spec.N, 1.0, y)
        g.synchronize()
        for k in ("d2m", "m2d"):
            ms, nl = g.timed(k)
            H = (spec.N + 1) ** 2
            fl = 2.0 * H * P * 4 * n_el
            out[f"c5s_{k}"] = {"s": ms * 1e-3, "tflops": fl / (ms * 1e-3) * 1e-12}
        g.timing(False)
        a, b = g.fp64_peaks()
        out["fp64_peaks_tflops"] = {"dmma": a, "dfma": b}
        del x, y
        g.close()
    if "si" in which:  # one source iteration at config-5 physics on an n^2 grid, per kernel
        spec = cf.baseline_config(5, int(os.environ.get("C5N", "256")))
        t0 = time.perf_counter()
        g = stamg.Context(spec, build_hierarchy=False)
        setup = time.perf_counter() - t0
        n_el, P, _, _ = g.layout()
        psi = g.vec().fill(1.0)
        g.source_iteration(psi, 1)
        g.synchronize()
        g.timing(True)
        t0 = time.perf_counter()
        g.source_iteration(psi, 2)
        g.synchronize()
        wall = (time.perf_counter() - t0) / 2
        kt = {kk: g.timed(kk)[0] / 2 for kk in ("fold", "d2m", "m2d", "unfold", "sweep")}
        g.timing(False)
        H = (spec.N + 1) ** 2
        fold = max(1, int(g.table("fold")[0]))
        exe = 2.0 * H * P * 4 * n_el / fold
        out["si"] = {"n": spec.nx, "setup_s": setup, "ms_per_iter": wall * 1e3, "kernels_ms": kt,
                     "d2m_tflops_exec": exe / (kt["d2m"] * 1e-3) * 1e-12,
                     "m2d_tflops_exec": exe / (kt["m2d"] * 1e-3) * 1e-12,
                     "fold_gbs": 2 * n_el * P * 32 / (kt["fold"] * 1e-3) * 1e-9,
                     "unfold_gbs": 2 * n_el * P * 32 / (kt["unfold"] * 1e-3) * 1e-9,
                     "fp64_peaks": g.fp64_peaks()}
        g.close()
    for k in (2, 3, 1):
        if f"c{k}" not in which:
            continue
        spec = cf.baseline_config(k)
        t0 = time.perf_counter()
        g = stamg.Context(spec)
        setup = time.perf_counter() - t0
        b = g.rhs()
        g.solve(b, "gmres", "mg")
        g.synchronize()
        g.timing(True)
        t0 = time.perf_counter()
        x, rep = g.solve(b, "gmres", "mg")
        g.synchronize()
        wall = time.perf_counter() - t0
        kt = {kk: g.timed(kk) for kk in ("sweep", "apply_L", "d2m", "m2d", "coarse_gs", "prolong", "restrict")}
        g.timing(False)
        out[f"c{k}_solve"] = {"setup_s": setup, "wall_s": wall, "iters": rep["iterations"],
                              "final_residual": rep["final_residual"], "kernels_ms": kt}
        g.close()
    if "c4v" in which:  # one V-cycle and one outer apply_A at full config-4 size
        spec = cf.baseline_config(4)
        t0 = time.perf_counter()
        g = stamg.Context(spec)
        setup = time.perf_counter() - t0
        b = g.rhs()
        z = g.mg_apply(b)
        y = g.vec()
        g.synchronize()
        g.timing(True)
        t0 = time.perf_counter()
        g.mg_apply(b, z)
        g.synchronize()
        tv = time.perf_counter() - t0
        t0 = time.perf_counter()
        g.apply_A_into(b, spec.N, y)
        g.synchronize()
        ta = time.perf_counter() - t0
        kt = {kk: g.timed(kk) for kk in ("sweep", "apply_L", "d2m", "m2d", "coarse_gs", "prolong", "restrict")}
        g.timing(False)
        out["c4_vcycle"] = {"setup_s": setup, "mg_apply_s": tv, "apply_A_outer_s": ta, "kernels_ms": kt,
                            "levels": g.levels(), "layout": g.layout()}
        g.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
