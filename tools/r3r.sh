cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_c4n64_golden.py tests/test_gpu_graphs.py tests/test_gpu_sharded_emulation.py tests/test_gpu_fullsize_golden.py tests/test_gpu_reference_parity.py -m gpu -q -x > gpurun_out/r3r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3r_tests.log
tail -3 gpurun_out/r3r_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-si --no-e2e --no-kernels --no-cpu --no-generic > gpurun_out/r3r_bench.json 2> gpurun_out/r3r_bench.err; echo "bench rc=$?"
STAMG_MG_ZERO_GUESS=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-si --no-e2e --no-kernels --no-cpu --no-generic --solve-configs 2 3 4 > gpurun_out/r3r_bench_full_seq.json 2> gpurun_out/r3r_bench_full_seq.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/r3r_bench.json", "gpurun_out/r3r_bench_full_seq.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, {k: (round(v["wall_s"], 3), v["iterations"]) for k, v in d["solve"].items() if isinstance(v, dict) and "wall_s" in v})
PY
