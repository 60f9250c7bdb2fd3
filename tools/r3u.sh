cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
C5N=256 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -f -o gpurun_out/r3u_sweep python tools/sweep_c5_once.py 3 > gpurun_out/r3u_ncu.log 2>&1
ncu -i gpurun_out/r3u_sweep.ncu-rep --page source --csv > gpurun_out/r3u_sweep_source.csv 2>/dev/null
ncu -i gpurun_out/r3u_sweep.ncu-rep --page details > gpurun_out/r3u_sweep_details.txt 2>/dev/null
rm -f gpurun_out/r3u_sweep.ncu-rep
ls -la gpurun_out | tail -5
