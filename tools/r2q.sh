cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_reference_identities.py -m gpu -q > gpurun_out/r2q_ident.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_ident.log
