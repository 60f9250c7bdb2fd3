cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_coarse_chain.py tests/test_gpu_coarse_cluster.py tests/test_gpu_shard_sweep.py -m gpu -q -x > gpurun_out/r2e_chain_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_chain_tests.log
for k in 1 2 3 4; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/r2e_gs_blk.log 2>&1; done
for k in 1 2 3 4; do STAMG_GS_CHAIN_BLOCKS=0 timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/r2e_gs_seq.log 2>&1; done
for xb in 1 2 4 2 1; do STAMG_SWEEP_XB=$xb C5N=512 timeout 600 python tools/perf_probe.py c5s > gpurun_out/r2e_sweep_xb${xb}_$RANDOM.json 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_c4n64_golden.py tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
