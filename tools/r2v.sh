cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-solve --no-generic > gpurun_out/r2v_kern_default_$i.json 2>/dev/null
STAMG_LIB=abl/swap1.so timeout 600 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-solve --no-generic > gpurun_out/r2v_kern_swap_$i.json 2>/dev/null
done
C5N=512 timeout 600 python tools/perf_probe.py si > gpurun_out/r2v_si_default.json 2>&1
STAMG_LIB=abl/swap1.so C5N=512 timeout 600 python tools/perf_probe.py si > gpurun_out/r2v_si_swap.json 2>&1
