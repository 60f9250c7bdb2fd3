cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_reference_identities.py -m gpu -q -x > gpurun_out/r3l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3l_tests.log
STAMG_SETUP_TRACE=1 python - > gpurun_out/r3l_setup.log 2>&1 <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2010_04559_b200 import configs as cf, stamg
for k, mg in ((5, False), (5, False), (4, True), (4, True)):
    t = time.perf_counter()
    g = stamg.Context(cf.baseline_config(k), build_hierarchy=mg)
    print(f"c{k} create: {time.perf_counter() - t:.3f} s", flush=True)
    g.close()
PY
