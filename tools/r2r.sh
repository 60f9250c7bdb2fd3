cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_reference_parity.py tests/test_gpu_reference_identities.py -m gpu -q > gpurun_out/r2r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_tests.log
GN=8 timeout 600 python tools/generic_probe.py > gpurun_out/r2r_gen8.json 2>&1
GN=24 timeout 600 python tools/generic_probe.py > gpurun_out/r2r_gen24.json 2>&1
