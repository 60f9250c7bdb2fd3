cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python tools/shard_probe.py 1 2 4 8 > gpurun_out/r3i_shard.jsonl 2> gpurun_out/r3i_shard.err
