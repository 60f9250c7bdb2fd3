cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nccl_selftest.py -m gpu -q > gpurun_out/r2p_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_nccl.log
