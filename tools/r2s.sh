cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
GN=24 timeout 600 ncu --set full --clock-control none --import-source on -k regex:coarse_gs_kernel -s 1 -c 1 -o gpurun_out/r2s_ggs python tools/generic_probe.py > gpurun_out/r2s_ncu.log 2>&1
ncu -i gpurun_out/r2s_ggs.ncu-rep --page source --csv --print-source sass > gpurun_out/r2s_ggs_source.csv 2>/dev/null
rm -f gpurun_out/r2s_ggs.ncu-rep
