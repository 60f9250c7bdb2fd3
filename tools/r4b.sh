cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for steps in 10 40; do
for v in default nst4 nst8 default nst4 nst8; do
  if [ "$v" = default ]; then timeout 600 python bench.py --steps $steps --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r4b_$v.json 2>> gpurun_out/r4b.err
  else STAMG_LIB=abl/$v.so timeout 600 python bench.py --steps $steps --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r4b_$v.json 2>> gpurun_out/r4b.err; fi
  python -c "
import json,sys
d=json.loads(open('gpurun_out/r4b_$v.json').read().strip().splitlines()[-1])
c=d['clocks']
print('$v steps=$steps', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), c['sm_mhz'], c.get('sm_mhz_min'), c.get('power_w'), c['reasons'])"
done; done
