cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2d_smi.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2d_tests.log
timeout 900 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?" >> gpurun_out/r2d_bench.err
timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 4 > gpurun_out/r2d_bench_c4.json 2> gpurun_out/r2d_bench_c4.err
for k in 1 2 3 4; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/r2d_gs.log 2>&1; done
