cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in default bulk1 default bulk1; do
  if [ "$v" = default ]; then timeout 600 python bench.py --steps 40 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3v_$v.json 2>> gpurun_out/r3v.err
  else STAMG_LIB=abl/$v.so timeout 600 python bench.py --steps 40 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3v_$v.json 2>> gpurun_out/r3v.err; fi
  python -c "
import json,sys
d=json.loads(open('gpurun_out/r3v_$v.json').read().strip().splitlines()[-1])
c=d['clocks']
print('$v', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), c['sm_mhz'], c.get('sm_mhz_min'), c.get('power_w'), c['reasons'])"
done
