cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python - > gpurun_out/r3g_ab.log 2>&1 <<'PY'
import os, sys, time
sys.path.insert(0, '.')
from paper_2010_04559_b200 import configs as cf, stamg
g = stamg.Context(cf.baseline_config(4))
b = g.rhs()
g.solve(b, "gmres", "mg", tol=1e-300, max_iter=2); g.synchronize()
for rep in range(2):
    for fused in ("1", "0"):
        os.environ["STAMG_GMRES_FUSED"] = fused
        t = time.perf_counter(); x, r = g.solve(b, "gmres", "mg"); g.synchronize()
        print(f"c4 fused={fused}: {time.perf_counter() - t:.3f} s, {r['iterations']} iterations, residual {r['final_residual']:.6e}", flush=True)
PY
