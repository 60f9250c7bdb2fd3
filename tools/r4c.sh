cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_shard_sweep.py tests/test_gpu_graphs.py -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
