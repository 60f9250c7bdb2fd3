cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for k in 2 3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/r2w_gs_c$k python tools/gs_probe.py $k 2 > gpurun_out/r2w_ncu_$k.log 2>&1
ncu -i gpurun_out/r2w_gs_c$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r2w_gs_c${k}_source.csv 2>/dev/null
ncu -i gpurun_out/r2w_gs_c$k.ncu-rep --page details > gpurun_out/r2w_gs_c${k}_details.txt 2>/dev/null
rm -f gpurun_out/r2w_gs_c$k.ncu-rep
done
