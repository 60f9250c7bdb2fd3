cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2b_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2b_memcheck.log
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2b_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r2b_racecheck.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/r2b_gs_c4 python tools/gs_probe.py 4 1 > gpurun_out/r2b_ncu_gs4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/r2b_gs_c2 python tools/gs_probe.py 2 2 > gpurun_out/r2b_ncu_gs2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/r2b_sweep_c5 python tools/sweep_c5_once.py 3 > gpurun_out/r2b_ncu_sweep.log 2>&1
for k in 1 2 3 4; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/r2b_gs.log 2>&1; done
