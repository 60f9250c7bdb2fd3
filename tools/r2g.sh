cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse_chain.py tests/test_gpu_coarse_cluster.py tests/test_gpu_shard_sweep.py -m gpu -q > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
for i in 1 2 3; do
timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2g_sweep_ab.log 2>&1
STAMG_LIB=abl/bulk0.so timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2g_sweep_ab.log 2>&1
done
for k in 1 2 3 4; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/r2g_gs.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "sweep or apply_L or wavefront or smoother or source" > gpurun_out/r2g_sweeptests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_sweeptests.log
