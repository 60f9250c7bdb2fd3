cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -m gpu -q > gpurun_out/r2h_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_ref.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c1 or cfg0 or 16" > gpurun_out/r2h_par.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_par.log
