cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reference_parity.py -m gpu -q > gpurun_out/r3h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3h_tests.log
