cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/c4_kernels.py 2>&1 | tail -2
for steps in 10 40 10 40; do
  timeout 600 python bench.py --steps $steps --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3z_b.json 2>> gpurun_out/r3z.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/r3z_b.json').read().strip().splitlines()[-1])
c=d['clocks']
print('steps=$steps', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), c['sm_mhz'], c.get('sm_mhz_min'), c.get('power_w'), c['reasons'])"
done
timeout 600 python tools/shard_probe.py 1 8 2>&1 | cut -c1-200
