cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_shard_sweep.py -m gpu -q -x > gpurun_out/r3w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3w_tests.log
tail -3 gpurun_out/r3w_tests.log
for steps in 10 40; do
for v in default u1 bulk1 default u1 bulk1; do
  if [ "$v" = default ]; then timeout 600 python bench.py --steps $steps --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3w_$v.json 2>> gpurun_out/r3w.err
  else STAMG_LIB=abl/$v.so timeout 600 python bench.py --steps $steps --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3w_$v.json 2>> gpurun_out/r3w.err; fi
  python -c "
import json,sys
d=json.loads(open('gpurun_out/r3w_$v.json').read().strip().splitlines()[-1])
c=d['clocks']
print('$v steps=$steps', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), c['sm_mhz'], c.get('sm_mhz_min'), c.get('power_w'), c['reasons'])"
done; done
STAMG_LIB=abl/bulk1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard_sweep.py -m gpu -q -x 2>&1 | tail -2
