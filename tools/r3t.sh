cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graphs.py -m gpu -q > gpurun_out/r3t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3t_tests.log
tail -15 gpurun_out/r3t_tests.log
timeout 600 python bench.py --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3t_bench.json 2> gpurun_out/r3t_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r3t_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['clocks'])"
timeout 600 python bench.py --steps 40 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3t_bench40.json 2>> gpurun_out/r3t_bench.err
python -c "
import json
d=json.loads(open('gpurun_out/r3t_bench40.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['clocks'])"
