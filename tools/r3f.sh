cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_krylov_workspace.py tests/test_gpu_graphs.py tests/test_gpu_fullsize_golden.py -m gpu -q -x -k "gmres or bicgstab or solve or krylov or poison or graph or fullsize" > gpurun_out/r3f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_tests.log
timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --no-generic --solve-configs 2 3 4 > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err
