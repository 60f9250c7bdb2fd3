cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_shard_sweep.py -m gpu -q > gpurun_out/r3j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3j_tests.log
timeout 1500 python tools/shard_probe.py 1 2 4 8 > gpurun_out/r3j_shard.jsonl 2> gpurun_out/r3j_shard.err
