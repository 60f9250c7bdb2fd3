cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export STAMG_SETUP_TRACE=1
python - > gpurun_out/r3b_setup.log 2>&1 <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2010_04559_b200 import configs as cf, stamg
for k, mg in ((5, False), (4, True), (3, True)):
    for rep in range(2):
        t = time.perf_counter()
        g = stamg.Context(cf.baseline_config(k), build_hierarchy=mg)
        print(f"c{k} create: {time.perf_counter() - t:.3f} s", flush=True)
        sys.stderr.flush()
        g.close()
PY
