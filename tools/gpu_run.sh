set -x
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_setup.py tests/test_gpu_fullsize.py -m gpu -x -q -s > gpurun_out/v2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v2_tests.log
C5N=512 timeout 300 python tools/perf_probe.py si > gpurun_out/v2_si512.json 2>&1
C5N=256 timeout 300 python tools/perf_probe.py si > gpurun_out/v2_si256.json 2>&1
C5N=256 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fold|d2m|unfold" -c 6 -o gpurun_out/v2_si256 python tools/perf_probe.py si > gpurun_out/v2_ncu.log 2>&1
echo done
