cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
( time timeout 1500 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err ) 2> gpurun_out/r2z_time.txt; echo "bench rc=$?" >> gpurun_out/r2z_bench.err
