cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do for v in default gsw2 gsw3; do for k in 1 2 3; do
  if [ $v = default ]; then timeout 120 python tools/gs_probe.py $k 10 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r2x_gsw.log
  else STAMG_LIB=abl/$v.so timeout 120 python tools/gs_probe.py $k 10 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r2x_gsw.log; fi
done; done; done
