cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard_sweep.py -m gpu -q -x > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
for i in 1 2 3; do
timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2k_sweep_ab.log 2>&1
STAMG_SWEEP_TAIL=0 timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2k_sweep_ab_notail.log 2>&1
done
